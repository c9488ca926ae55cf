// TGT+ AESC on sm_100a (placeholder until the estimator kernels land).
#include "device_graph.cuh"
#include "plan_host.hpp"

namespace saba_cu {
struct AescState {};
void release_aesc_state(saba_cu_graph* g) {
    delete g->aesc;
    g->aesc = nullptr;
}
}  // namespace saba_cu

using namespace saba_cu;

extern "C" {

int saba_cu_truncated_lengths(saba_cu_graph* g, double epsilon, uint32_t power_iterations,
                              uint32_t max_truncation, int per_edge, uint32_t* tau_out,
                              double* lambda_hat, int* clamped) {
    return guard([&] {
        check_arg(g && tau_out && lambda_hat && clamped, "null argument");
        const HostCsr h{g->n, g->m, g->h_off.data(), g->h_adj.data()};
        const Plan p = host_truncated_lengths(h, slot_edges(g), epsilon, power_iterations,
                                              max_truncation, per_edge != 0);
        std::copy(p.tau.begin(), p.tau.end(), tau_out);
        *lambda_hat = p.lambda_hat;
        *clamped = p.clamped ? 1 : 0;
    });
}

int saba_cu_aesc(saba_cu_graph*, const saba_cu_aesc_config*, const uint32_t*, uint64_t, uint32_t,
                 uint32_t, double*, double*, uint32_t*, uint32_t*, saba_cu_aesc_report*) {
    return guard([&] { throw ArgError("aesc: not implemented yet"); });
}

int saba_cu_propagate(saba_cu_graph*, uint32_t, const uint32_t*, double, double, int64_t, double*,
                      uint32_t*) {
    return guard([&] { throw ArgError("propagate: not implemented yet"); });
}

int saba_cu_estimate_edge(saba_cu_graph*, uint32_t, uint32_t, const double*, uint32_t, uint64_t, int,
                          uint64_t, uint32_t, uint64_t, double*) {
    return guard([&] { throw ArgError("estimate_edge: not implemented yet"); });
}

}  // extern "C"
