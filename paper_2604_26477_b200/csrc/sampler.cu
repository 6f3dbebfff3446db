// SB sampler dispatch (see sampler.cuh / sampler_impl.cuh).
#include <cuda_runtime.h>

#include "sampler_impl.cuh"

namespace momc_b200 {

bool sampler_uses_register_path(int n, double alpha) { return n >= 1 && n <= 64 && alpha > 0.0; }

int sampler_block_traj(int n, double alpha)
{
    if (!sampler_uses_register_path(n, alpha)) return kSampleBlock;
    return n <= 42 && !sbimpl::force_step_kernel() ? sbimpl::kBT / 4 : sbimpl::kThreads / 4;
}

int launch_sampler(const SamplerParams& p, long long nblocks, void* stream)
{
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int n = p.n;
    if (p.pad_dmax == 3) {
        if (n <= 16) return launch_small_n16_d3(p, nblocks, st);
        if (n <= 32) return launch_small_n32_d3(p, nblocks, st);
        if (n <= 42) return launch_small_n42_d3(p, nblocks, st);
        if (n <= 64) return launch_small_n64_d3(p, nblocks, st);
    } else {
        if (n <= 16) return launch_small_n16_d0(p, nblocks, st);
        if (n <= 32) return launch_small_n32_d0(p, nblocks, st);
        if (n <= 42) return launch_small_n42_d0(p, nblocks, st);
        if (n <= 64) return launch_small_n64_d0(p, nblocks, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace momc_b200
