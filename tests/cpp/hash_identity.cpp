// hash_state_fast (the walk kernels' per-step split of HashSpec::state, rng.hpp:20-31)
// equals hash_state bit for bit: random vertices, steps and multipliers.
#include "saba_hash.cuh"
#include <cstdio>
#include <random>
using namespace saba_cu;
int main() {
    std::mt19937_64 r(1);
    uint64_t bad = 0;
    for (int i = 0; i < 20000000; ++i) {
        uint64_t m = (i % 3 == 0) ? 0xc6a4a7935bd1e995ull : r();
        uint32_t v = uint32_t(r()), l = uint32_t(r() % 4096);
        if (i % 5 == 0) l = uint32_t(r());
        if (hash_state(m, v, l) != hash_state_fast(step_hash(m, l), v)) ++bad;
    }
    printf("mismatches %llu\n", (unsigned long long)bad);
    return bad != 0;
}
