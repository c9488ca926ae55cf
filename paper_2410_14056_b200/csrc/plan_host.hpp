#pragma once
#include <cstdint>
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
double host_estimate_decay(const HostCsr& g, uint32_t iters, bool bip, const std::vector<char>& side);
Plan host_truncated_lengths(const HostCsr& g, const std::vector<uint32_t>& slot_edge, double eps,
                            uint32_t omega, uint32_t max_truncation, bool per_edge);
double walks_needed_raw(int64_t tau_eff, double eps, double delta, uint32_t degree, uint64_t m);
uint64_t walk_budget(uint32_t tau_eff, double eps, double delta, uint32_t degree, uint64_t m);

}  // namespace saba_cu
