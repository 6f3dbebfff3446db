// Instantiation unit for the register-resident SB kernel, NMAX = 32, DMAX = 3 (parallel build).
#include "sampler_impl.cuh"

namespace momc_b200 {
int launch_small_n32_d3(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    return sbimpl::launch_variant<32, 4, 3>(p, nblocks, st);
}
}  // namespace momc_b200
