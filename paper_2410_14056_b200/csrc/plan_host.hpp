#pragma once
#include <cstdint>
#include <functional>
#include <vector>

namespace saba_cu {

struct HostCsr {
    uint32_t n;
    uint64_t m;
    const uint32_t* off;
    const uint32_t* adj;
};

// TruncationPlan (aesc.hpp:55-61) + bipartiteness.
struct Plan {
    std::vector<uint32_t> tau;  // per edge id
    double lambda_hat = 0.0;
    bool clamped = false;
    bool bipartite = false;
    bool uniform = true;
    uint32_t max_tau = 0;
};

bool host_is_connected(const HostCsr& g);
uint32_t host_bfs_parity(const HostCsr& g, std::vector<uint8_t>& parity);
bool host_bipartition(const HostCsr& g, std::vector<char>& side);
// y[u] = (sum over neighbours a of u, in slot order, of x[a] * isd[a]) * isd[u]
// -- the power iteration's SpMV; a device implementation can be plugged in
// (it must round exactly like the host loop: one multiply, then the add).
using SpmvFn = std::function<void(const std::vector<double>& x, const std::vector<double>& isd,
                                  std::vector<double>& y)>;
double host_estimate_decay(const HostCsr& g, uint32_t iters, bool bip, const std::vector<char>& side,
                           const SpmvFn* spmv = nullptr);
Plan host_truncated_lengths(const HostCsr& g, const uint32_t* slot_edge, double eps,
                            uint32_t omega, uint32_t max_truncation, bool per_edge,
                            const SpmvFn* spmv = nullptr);
double walks_needed_raw(int64_t tau_eff, double eps, double delta, uint32_t degree, uint64_t m);
uint64_t walk_budget(uint32_t tau_eff, double eps, double delta, uint32_t degree, uint64_t m);

}  // namespace saba_cu
