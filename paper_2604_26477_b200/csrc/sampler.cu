// SB sampler dispatch (see sampler.cuh / sampler_impl.cuh).
#include <cuda_runtime.h>

#include "sampler_impl.cuh"

namespace momc_b200 {

int launch_sampler(const SamplerParams& p, long long nblocks, void* stream, int /*check_steps*/)
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
    return cudaErrorInvalidValue;  // n > 64: launch_sampler_generic
}

}  // namespace momc_b200
