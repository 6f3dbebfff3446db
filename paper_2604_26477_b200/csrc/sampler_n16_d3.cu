// Instantiation unit for the register-resident SB kernel, NMAX = 16, DMAX = 3 (parallel build).
#include "sampler_impl.cuh"

namespace momc_b200 {
int launch_small_n16_d3(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    return sbimpl::launch_variant<16, 4, 3>(p, nblocks, st);
}
}  // namespace momc_b200
