// Roofline calibration: the noise generation alone, at the same per-word work
// as the sampler's fast path -- one Philox4x32-10 block per 4 words, the ziggurat fast test
// |hz| < kn[iz] and eta = hz * wn[iz] per word, tables in shared memory -- with nothing
// else (no slow-attempt bookkeeping, no spin update). Its normals/s bounds what the sampler's
// RNG share can reach on this GPU; bench / DESIGN restate the sampler against it.
#include <cuda_runtime.h>

#include <cstdint>

#include "ctx.cuh"
#include "rng.cuh"

namespace momc_b200 {

namespace {

__global__ void __launch_bounds__(256) k_rng_calib(uint64_t key, int blocks_per_thread, const ZigTables* __restrict__ zig,
                                                   double* sink)
{
    __shared__ ZigTables z;
    for (int q = threadIdx.x; q < static_cast<int>(sizeof(ZigTables) / 4); q += blockDim.x)
        reinterpret_cast<uint32_t*>(&z)[q] = reinterpret_cast<const uint32_t*>(zig)[q];
    __syncthreads();
    const uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
    const uint32_t tr = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    uint32_t slow = 0;
    for (int b = 0; b < blocks_per_thread; ++b) {
        const uint4 r = philox(k0, k1, static_cast<uint32_t>(b), 3u << 26, tr, 7u);
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t u = w[j];
            const uint32_t iz = u & 127u;
            const int32_t hz = static_cast<int32_t>(u);
            const uint32_t mag = hz < 0 ? 0u - u : u;
            slow += mag >= z.kn[iz];
            acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(hz), z.wn[iz]));
        }
    }
    if (acc == 1.2345 || slow == 0xFFFFFFFFu) sink[tr] = acc;  // keep the work alive
}

}  // namespace

// normals generated per second by the calibration kernel (148 x 8 CTAs of 256 threads)
double rng_calibrate(Ctx& c, int blocks_per_thread)
{
    const ZigTables* z = device_zig(c);
    DevBuf<double> sink;
    const int ctas = 148 * 8;
    sink.reserve(static_cast<size_t>(ctas) * 256);
    k_rng_calib<<<ctas, 256, 0, c.stream>>>(0x1234ull, blocks_per_thread, z, sink.p);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c.stream);
    k_rng_calib<<<ctas, 256, 0, c.stream>>>(0x5678ull, blocks_per_thread, z, sink.p);
    cudaEventRecord(b, c.stream);
    c.launches += 2;
    ck(cudaEventSynchronize(b), "calibration");
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    sink.release();
    const double normals = 4.0 * blocks_per_thread * ctas * 256.0;
    return normals / (static_cast<double>(ms) * 1e-3);
}

}  // namespace momc_b200
