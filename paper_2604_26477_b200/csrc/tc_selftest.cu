// Self-test of the hand-written tcgen05 int8 path (tc_i8.cuh): one CTA computes
// D (128 x 128, int32) = A (128 x K) . B (128 x K)^T with A, B signed int8, K-major,
// K a multiple of 128, through shared-memory descriptors, TMEM and tcgen05.mma.kind::i8.
// Checked against a host reference by tests/test_gpu_tc.py before the fused dense
// kernel relies on the same blocks.
#include <cuda_runtime.h>

#include <cstdint>

#include "ctx.cuh"
#include "tc_i8.cuh"

namespace momc_b200 {

namespace {

__global__ void __launch_bounds__(128, 1) k_tc_selftest(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                        int K, int32_t* __restrict__ D)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    uint8_t* sa = sm;
    uint8_t* sb = sm + 128 * tc::kChunkK;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tc::tmem_alloc<128>(&tslot);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tslot;
    constexpr uint32_t idesc = tc::idesc_i8(128, 128);
    uint32_t phase = 0;
    for (int kc = 0; kc < K / tc::kChunkK; ++kc) {
        for (int q = 0; q < tc::kChunkK / 16; ++q) {
            *reinterpret_cast<uint4*>(sa + tc::chunk_offset(tid, 16 * q)) =
                *reinterpret_cast<const uint4*>(A + static_cast<long long>(tid) * K + kc * tc::kChunkK + 16 * q);
            *reinterpret_cast<uint4*>(sb + tc::chunk_offset(tid, 16 * q)) =
                *reinterpret_cast<const uint4*>(B + static_cast<long long>(tid) * K + kc * tc::kChunkK + 16 * q);
        }
        tc::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t a0 = tc::smem_u32(sa), b0 = tc::smem_u32(sb);
#pragma unroll
            for (int k = 0; k < tc::kChunkK / 32; ++k)
                tc::mma_i8(tbase, tc::smem_desc(a0 + 256 * k), tc::smem_desc(b0 + 256 * k), idesc, kc > 0 || k > 0);
            tc::commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1;
        tc::fence_after();
    }
    // epilogue: warp w reads TMEM lanes [32 w, 32 w + 32) = rows of A
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) D[tid * 128 + c0 + j] = static_cast<int32_t>(v[j]);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<128>(tbase);
}

}  // namespace

void tc_i8_selftest(Ctx& c, const int8_t* hA, const int8_t* hB, int K, int32_t* hD)
{
    if (K <= 0 || K % tc::kChunkK) usage("selftest K must be a positive multiple of 128");
    DevBuf<int8_t> a, b;
    DevBuf<int32_t> d;
    a.reserve(static_cast<size_t>(128) * K);
    b.reserve(static_cast<size_t>(128) * K);
    d.reserve(128 * 128);
    ck(cudaMemcpyAsync(a.p, hA, static_cast<size_t>(128) * K, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(b.p, hB, static_cast<size_t>(128) * K, cudaMemcpyHostToDevice, c.stream), "H2D");
    const int smem = 2 * 128 * tc::kChunkK;
    ck(cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem");
    k_tc_selftest<<<1, 128, smem, c.stream>>>(a.p, b.p, K, d.p);
    c.launches++;
    ck(cudaGetLastError(), "tc selftest");
    ck(cudaMemcpyAsync(hD, d.p, sizeof(int32_t) * 128 * 128, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "tc selftest");
    a.release();
    b.release();
    d.release();
}

}  // namespace momc_b200
