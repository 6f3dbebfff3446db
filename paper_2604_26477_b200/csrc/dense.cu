// Dense dSB sampler for large n on the tensor cores (config C4, N=2000) and the tensor-core
// form of evaluate_cuts. Restates sb_step (solver.hpp:152-183) with phi = sgn(x),
// init_state (:108-124), fill_step_noise (:128-136), read_spins (:237-244) and
// evaluate_cuts (pareto.hpp:330-363).
//
// Exactness. With integer weights, H*J(c) = sum_k num_k w_k is an integer matrix. When
// |H*J| <= 127 it is exact in int8 (tcgen05 kind::i8, int32 accumulation); when |H*J| <= 256
// it is exact in bf16 (kind::f16, FP32 accumulation of integers below 2^24). sgn(x) = +-1 is
// exact in both. So D = sgn(X) (H J)^T is computed exactly; coupled = D / H then enters the
// FP64 update as c0/H * D, one rounding where the reference sums rounded FP64 products over j
// (scalarize.hpp:30, solver.hpp:161). Trajectories therefore agree with the reference within
// the FP tolerance of DESIGN.md §3 (spin words compared in tests/test_gpu_dense*.py), not
// bit-for-bit; the pool reports the path (Session.sampler_path).
//
// One persistent, warp-specialised kernel (k_dense_fused) runs init, all T steps and the
// readout of one work item = one 120-trajectory block of one (run, weight) pair at a time
// (MMA rows 120..127 are padding, so the 15 epilogue warps take 8 trajectories each).
// Per step it walks the spins in tiles of 128:
//   * the contraction: D_tile (128 traj x 128 spins, TMEM) = Phi (128 x n) . HJ_tile^T with
//     A = Phi from TMEM and B = the HJ tile from shared memory (TMA, 128-byte swizzle), K in
//     chunks of 128 bytes, 4 stages; two TMEM accumulators (tile s and s+1 overlap);
//   * a producer warp: one thread keeps the B TMA up to 4 chunks ahead and issues the
//     tcgen05.mma of every chunk;
//   * 4 io warps (one per TMEM lane quarter): expand the packed sign bits of Phi into the A
//     stage (tcgen05.st) and drain finished accumulators to shared memory (tcgen05.ld ->
//     64 KB swizzled [traj][spin] int32 tile, double-buffered);
//   * 15 epilogue warps: one warp per trajectory-tile, lanes over spins (32 per window). The
//     (trajectory, step) noise stream (rng.hpp:156-185) is resolved warp-wide: lane L tests
//     word head + L; slow words (wedge / tail attempts) are tested in parallel and a ballot +
//     popcount orders the produced normals into a 64-entry ring; each window takes 32. At
//     a tile end the stream position of the first unused normal is kept, and the next tile
//     regenerates from it. x / y (FP64, trajectory-major) stream from HBM; the new signs go
//     out as bits (Phi of the next step, and in the last step the packed pool words).
// D never touches HBM; the only per-step HBM traffic is x / y (32 B per spin-update) and
// the sign bits.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "tc_i8.cuh"
#include "rng.cuh"
#include "sampler.cuh"

namespace momc_b200 {

namespace {

// ---- H*J(c): row-major [weight][spin][npad] (K = the column index, contiguous), int8 or
// bf16 bits; columns >= n are exact zeros
__global__ void k_build_hj(int n, int npad, int k, const int* __restrict__ nums, const int* __restrict__ rowptr,
                           const int* __restrict__ col, const int* __restrict__ eidx, const int* __restrict__ wi,
                           void* hj, int bf16, int* maxabs)
{
    const int l = blockIdx.y;
    const int i = blockIdx.x;
    const long long rowo = (static_cast<long long>(l) * n + i) * npad;
    if (bf16) {
        uint16_t* row = static_cast<uint16_t*>(hj) + rowo;
        for (int j = threadIdx.x; j < npad; j += blockDim.x) row[j] = 0;
    } else {
        int8_t* row = static_cast<int8_t*>(hj) + rowo;
        for (int j = threadIdx.x; j < npad; j += blockDim.x) row[j] = 0;
    }
    __syncthreads();
    int mx = 0;
    for (int e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x) {
        int v = 0;
        for (int q = 0; q < k; ++q) v += nums[l * k + q] * wi[static_cast<long long>(eidx[e]) * k + q];
        mx = max(mx, abs(v));
        if (bf16) {
            // |v| <= 256 has at most 8 significant bits: the top half of the FP32 bits is exact
            static_cast<uint16_t*>(hj)[rowo + col[e]] = static_cast<uint16_t>(__float_as_uint(static_cast<float>(v)) >> 16);
        } else {
            static_cast<int8_t*>(hj)[rowo + col[e]] = static_cast<int8_t>(v);
        }
    }
    if (mx) atomicMax(maxabs, mx);
}

// ---- the fused kernel ----------------------------------------------------------------------
constexpr int kNT = 128;          // MMA M = TMEM lanes = trajectory rows per work item
constexpr int kNTV = 120;         // trajectories per work item (rows 120..127 are padding)
constexpr int kNS = 128;          // spins per tile: MMA N, TMEM columns per accumulator
constexpr int kStages = 3;        // K chunks in flight (A in TMEM, B in shared memory)
constexpr int kEpiWarps = 15;     // epilogue warps (8 trajectories each per tile)
constexpr int kEpiWarp0 = 5;      // warp 0: TMA + MMA; 1..4: io (expand / drain); 5..19: epilogue
// 20 warps = 5 per SM sub-partition, so each thread may hold 96 registers
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kRing = 256;        // noise words per epilogue warp
constexpr int kNBuf = 160;        // normals per epilogue warp: a tile's 128 + one round's overshoot
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColA = 256;   // A stages at TMEM columns [256, 256 + 32 kStages)
constexpr int kBStage = kNS * 128;  // bytes of one B stage (128 spins x 128 bytes of K)

// dynamic shared memory layout (offsets from the 1024-aligned base)
constexpr int kOffB = 0;
constexpr int kOffD = kOffB + kStages * kBStage;         // 2 x 64 KB int32 [traj][spin], swizzled
constexpr int kOffRing = kOffD + 2 * kNT * kNS * 4;
constexpr int kOffNBuf = kOffRing + kEpiWarps * kRing * 4;
constexpr int kOffZig = kOffNBuf + kEpiWarps * kNBuf * 8;
constexpr int kOffLut = kOffZig + static_cast<int>(sizeof(ZigTables));
constexpr int kOffPos = kOffLut + 256 * 16;
constexpr int kSmemBytes = kOffPos + kNT * 4 + 1024;  // + alignment slack

struct FusedArgs {
    int n, T, L, batch, chunks, ntiles, nchunks, nwp, wpc, H;
    long long b0, nblocks;  // items = flattened (run, weight, chunk) blocks [b0, b0 + nblocks)
    uint64_t seed;
    double dt, a0, alpha, sdt, init_scale;
    const double* c0;  // [L]
    const ZigTables* zig;
    double* x;         // [grid][kNT][n]
    double* y;
    uint32_t* phib;    // [grid][2][kNT][nwp] sign bits (bit = x >= 0)
    uint64_t* words;   // pool rows from row0
    long long row0;
    unsigned long long* block_end_ns;  // per item
    int* nan_block;                    // per item
};

struct ItemOf {
    int l, run, traj0, count;
};
__device__ __forceinline__ ItemOf item_of(const FusedArgs& a, long long it)
{
    const long long b = a.b0 + it;
    const int chunk = static_cast<int>(b % a.chunks);
    const long long rl = b / a.chunks;
    ItemOf r;
    r.l = static_cast<int>(rl % a.L);
    r.run = static_cast<int>(rl / a.L);
    r.traj0 = chunk * kNTV;
    r.count = min(kNTV, a.batch - r.traj0);
    return r;
}

__device__ __forceinline__ uint32_t zmag32(uint32_t u) { return static_cast<int32_t>(u) < 0 ? 0u - u : u; }

__device__ __noinline__ bool exp_decides(double lhs, double targ) { return lhs < exp(targ); }

// wedge test of the attempt at word u with uniform words (w1, w2) (rng.hpp:178-183): the FP32
// exp brackets the FP64 one within 1e-6 relative on [-6, 0]; the FP64 exp decides the band
__device__ __forceinline__ bool wedge_accept(uint32_t u, uint32_t w1, uint32_t w2, const ZigTables& z)
{
    const uint32_t iz = u & 127u;
    const double xv = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), z.wn[iz]);
    const double lhs = __dadd_rn(z.fn[iz], __dmul_rn(u01_from(w1, w2), __dsub_rn(z.fn[iz - 1], z.fn[iz])));
    const double targ = __dmul_rn(__dmul_rn(-0.5, xv), xv);
    const float ef = __expf(static_cast<float>(targ));
    if (lhs < static_cast<double>(ef) * (1.0 - 1e-5)) return true;
    if (lhs > static_cast<double>(ef) * (1.0 + 1e-5)) return false;
    return exp_decides(lhs, targ);
}

// the tail attempt starting at word p0 of the (key, lo, mid, hi) stream (rng.hpp:165-177):
// (x, y) trials of 4 words until 2y >= x^2; returns the normal and its length in words. Rare
// (one word in ~1,600), so it lives out of line and reads every word from the ring or Philox.
struct TailOut {
    double v;
    int len;
};
__device__ __noinline__ TailOut tail_attempt(const uint32_t* ring, int tail, int p0, uint32_t u, uint32_t k0, uint32_t k1,
                                             uint32_t lo, uint32_t mid, uint32_t hi)
{
    auto word = [&](int p) -> uint32_t {
        if (p < tail) return ring[p & 255];
        const uint4 v = philox(k0, k1, static_cast<uint32_t>(p >> 2), lo, mid, hi);
        const int c = p & 3;
        return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
    };
    const double rr = 3.442619855899;
    int qq = p0 + 1;
    for (;;) {
        const double xx = __ddiv_rn(-log(u01_open_from(word(qq), word(qq + 1))), rr);
        const double yy = -log(u01_open_from(word(qq + 2), word(qq + 3)));
        qq += 4;
        if (__dadd_rn(yy, yy) >= __dmul_rn(xx, xx))
            return {static_cast<int32_t>(u) > 0 ? __dadd_rn(rr, xx) : -__dadd_rn(rr, xx), qq - p0};
    }
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint4 ldcg4(const uint32_t* p)
{
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

// D tile element (trajectory r, spin column c) in the swizzled [128][128] int32 layout: the
// 16-byte unit index is XORed with r & 7, so the drain's row-wise 16-byte stores and the
// epilogue's column-contiguous warp reads are both conflict-free
__device__ __forceinline__ int dsw(int r, int c) { return r * kNS + (c ^ ((r & 7) << 2)); }

// Named hardware barrier (a waiting warp does not issue): the epilogue warps arrive at
// kBarDEmpty + b when done with D buffer b, the io warps sync on it before refilling it.
constexpr int kBarDEmpty = 1;
constexpr int kBarThreads = (4 + kEpiWarps) * 32;
__device__ __forceinline__ void named_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kBarThreads) : "memory"); }
__device__ __forceinline__ void named_arrive(int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(kBarThreads) : "memory"); }

struct FusedShared {
    uint64_t b_full[kStages], b_empty[kStages], a_full[kStages], a_empty[kStages];
    uint64_t d_full[2], d_empty[2], s_full[2];
    uint32_t tslot;
    int epi_cnt[2], tiles_done, init_cnt, init_done;
};

// BF16: kind::f16 with bf16 H*J (|H*J| <= 256); else kind::i8 (|H*J| <= 127).
// NOISY: alpha > 0 (the noise stream is consumed). UDT: dt == 1 and dt * a0 == 1.
template <bool BF16, bool NOISY, bool UDT>
__global__ void __launch_bounds__(kThreads, 1) k_dense_fused(const __grid_constant__ CUtensorMap tmB,
                                                             const __grid_constant__ FusedArgs a)
{
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    __shared__ FusedShared S;
    ZigTables& z = *reinterpret_cast<ZigTables*>(sm + kOffZig);
    int* pos = reinterpret_cast<int*>(sm + kOffPos);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int KC = BF16 ? 64 : 128;  // K elements (spins) per 128-byte chunk

    // ---- setup: tables, LUT, barriers, TMEM
    for (int q = tid; q < static_cast<int>(sizeof(ZigTables) / 4); q += blockDim.x)
        reinterpret_cast<uint32_t*>(&z)[q] = reinterpret_cast<const uint32_t*>(a.zig)[q];
    if (BF16) {  // byte -> 8 bf16 signs (+1 = 0x3F80, -1 = 0xBF80), element 0 in the low half
        uint32_t* lut = reinterpret_cast<uint32_t*>(sm + kOffLut);
        for (int b = tid; b < 256; b += blockDim.x)
            for (int w = 0; w < 4; ++w)
                lut[b * 4 + w] = ((b >> (2 * w)) & 1 ? 0x3F80u : 0xBF80u) | (((b >> (2 * w + 1)) & 1 ? 0x3F80u : 0xBF80u) << 16);
    } else {     // byte -> 8 int8 signs (+1 = 0x01, -1 = 0xFF), element 0 in the lowest byte
        uint32_t* lut = reinterpret_cast<uint32_t*>(sm + kOffLut);
        for (int b = tid; b < 256; b += blockDim.x)
            for (int w = 0; w < 2; ++w) {
                uint32_t v = 0;
                for (int q = 0; q < 4; ++q) v |= ((b >> (4 * w + q)) & 1 ? 0x01u : 0xFFu) << (8 * q);
                lut[b * 2 + w] = v;
            }
    }
    if (tid == 0) {
        for (int q = 0; q < kStages; ++q) {
            tc::mbar_init(&S.b_full[q], 1);
            tc::mbar_init(&S.b_empty[q], 1);
            tc::mbar_init(&S.a_full[q], 4);
            tc::mbar_init(&S.a_empty[q], 1);
        }
        for (int q = 0; q < 2; ++q) {
            tc::mbar_init(&S.d_full[q], 1);
            tc::mbar_init(&S.d_empty[q], 4);
            tc::mbar_init(&S.s_full[q], 4);
            S.epi_cnt[q] = 0;
        }
        S.tiles_done = 0;
        S.init_cnt = 0;
        S.init_done = 0;
        tc::fence_mbar_init();
        tc::prefetch_tmap(&tmB);
    }
    if (warp == 0) tc::tmem_alloc<kTmemCols>(&S.tslot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = S.tslot;
    const int nt = a.ntiles, nch = a.nchunks;
    const long long slot = blockIdx.x;

    if (warp == 0) {
        // ===== producer: one thread keeps the B TMA up to kStages chunks ahead and issues the
        //       MMAs of every chunk once its A (io warps) and B (TMA) stages are full
        if (lane == 0) {
            const uint32_t idesc = BF16 ? tc::idesc_bf16(kNT, kNS) : tc::idesc_i8(kNT, kNS);
            const long long my_items = a.nblocks > blockIdx.x ? (a.nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
            const long long g_total = my_items * a.T * nt * nch;
            long long g_tma = 0;
            int tma_c = 0, tma_m = 0, tma_t = 0;  // (step, tile, chunk) of chunk g_tma within its item
            long long tma_it = blockIdx.x;
            int tma_l = my_items > 0 ? item_of(a, tma_it).l : 0;
            auto issue = [&]() {
                const uint32_t st = static_cast<uint32_t>(g_tma % kStages);
                tc::mbar_expect_tx(&S.b_full[st], kBStage);
                tc::tma_load_2d(sm + kOffB + st * kBStage, &tmB, tma_c * KC, tma_l * a.n + tma_m * kNS, &S.b_full[st]);
                ++g_tma;
                if (++tma_c == nch) {
                    tma_c = 0;
                    if (++tma_m == nt) {
                        tma_m = 0;
                        if (++tma_t == a.T) {
                            tma_t = 0;
                            tma_it += gridDim.x;
                            if (tma_it < a.nblocks) tma_l = item_of(a, tma_it).l;
                        }
                    }
                }
            };
            auto b_free = [&](long long gq) {
                return tc::mbar_test(&S.b_empty[gq % kStages], (static_cast<uint32_t>(gq / kStages) & 1) ^ 1);
            };
            long long g = 0;
            // TMA of every chunk whose stage is free, up to kStages ahead of the MMA (non-blocking)
            auto pump = [&]() {
                while (g_tma < g_total && g_tma < g + kStages && b_free(g_tma)) issue();
            };
            uint32_t s = 0;
            for (long long it = blockIdx.x; it < a.nblocks; it += gridDim.x)
                for (int t = 0; t < a.T; ++t)
                    for (int m = 0; m < nt; ++m, ++s) {
                        const uint32_t buf = s & 1;
                        while (!tc::mbar_test(&S.d_empty[buf], ((s >> 1) & 1) ^ 1)) {
                            pump();
                            __nanosleep(64);
                        }
                        tc::fence_after();
                        const uint32_t dt = tbase + buf * kNS;
                        for (int c = 0; c < nch; ++c, ++g) {
                            const uint32_t st = static_cast<uint32_t>(g % kStages), ph = static_cast<uint32_t>(g / kStages) & 1;
                            pump();
                            while (g_tma <= g) {  // this chunk's own load (its stage frees with chunk g - kStages)
                                if (b_free(g_tma)) issue();
                                else __nanosleep(32);
                            }
                            while (!tc::mbar_test(&S.a_full[st], ph) || !tc::mbar_test(&S.b_full[st], ph)) {
                                pump();
                                __nanosleep(32);
                            }
                            tc::fence_after();
                            const uint32_t at = tbase + kColA + st * 32;
                            const uint32_t bs = tc::smem_u32(sm + kOffB + st * kBStage);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                if (BF16) tc::mma_f16_ts(dt, at + 8 * k, tc::smem_desc_sw128(bs + 32 * k), idesc, c > 0 || k > 0);
                                else tc::mma_i8_ts(dt, at + 8 * k, tc::smem_desc_sw128(bs + 32 * k), idesc, c > 0 || k > 0);
                            }
                            tc::commit(&S.a_empty[st]);
                            tc::commit(&S.b_empty[st]);
                        }
                        tc::commit(&S.d_full[buf]);
                    }
        }
        __syncwarp();
    } else if (warp < kEpiWarp0) {
        // ===== io warps (TMEM lane quarter = warp & 3): drain tile s-1, then expand the A chunks
        //       of tile s
        const int q = warp & 3;
        const int r = q * 32 + lane;  // trajectory row of this thread
        const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
        const uint32_t* lut = reinterpret_cast<const uint32_t*>(sm + kOffLut);
        uint32_t s = 0;
        long long g = 0;
        int ii = 0;
        auto drain = [&](uint32_t sd) {
            const uint32_t buf = sd & 1;
            tc::mbar_wait_sleep(&S.d_full[buf], (sd >> 1) & 1, 512);
            if (sd >= 2) named_sync(kBarDEmpty + buf);  // the epilogue is done with tile sd - 2
            tc::fence_after();
            int* D = reinterpret_cast<int*>(sm + kOffD + buf * (kNT * kNS * 4));
#pragma unroll 1
            for (int cg = 0; cg < kNS / 32; ++cg) {
                uint32_t v[32];
                tc::tmem_ld32(tbase + lane_addr + buf * kNS + cg * 32, v);
                if (BF16)
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = static_cast<uint32_t>(__float2int_rn(__uint_as_float(v[e])));
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    *reinterpret_cast<uint4*>(&D[dsw(r, cg * 32 + 4 * u)]) = make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive(&S.d_empty[buf]);
                tc::mbar_arrive(&S.s_full[buf]);
            }
        };
        bool prev = false;
        for (long long it = blockIdx.x; it < a.nblocks; it += gridDim.x, ++ii) {
            for (int t = 0; t < a.T; ++t) {
                const uint32_t* pb = a.phib + ((slot * 2 + (t & 1)) * kNT + r) * a.nwp;
                for (int m = 0; m < nt; ++m, ++s) {
                    if (prev) drain(s - 1);
                    prev = true;
                    for (int c = 0; c < nch; ++c, ++g) {
                        const uint32_t st = static_cast<uint32_t>(g % kStages), ph = static_cast<uint32_t>(g / kStages) & 1;
                        tc::mbar_wait_sleep(&S.a_empty[st], ph ^ 1, 256);
                        // the sign bits of Phi_t for this chunk: written by init (t = 0) or by the
                        // epilogue of step t-1, tile (c KC) / kNS
                        if (t == 0) {
                            while (vload(&S.init_done) < ii + 1) __nanosleep(1000);
                        } else {
                            const int need = static_cast<int>(s) - m - nt + (c * KC) / kNS + 1;
                            while (vload(&S.tiles_done) < need) __nanosleep(500);
                        }
                        __threadfence_block();
                        uint32_t v[32];
                        if (BF16) {  // 64 spins: 2 words -> 8 bytes -> 8 x 4 columns
                            const uint32_t w0 = __ldcg(pb + 2 * c), w1 = __ldcg(pb + 2 * c + 1);
#pragma unroll
                            for (int b = 0; b < 8; ++b) {
                                const uint32_t by = ((b < 4 ? w0 : w1) >> (8 * (b & 3))) & 0xFF;
                                const uint4 e = *reinterpret_cast<const uint4*>(&lut[by * 4]);
                                v[4 * b] = e.x;
                                v[4 * b + 1] = e.y;
                                v[4 * b + 2] = e.z;
                                v[4 * b + 3] = e.w;
                            }
                        } else {     // 128 spins: 4 words -> 16 bytes -> 16 x 2 columns
                            const uint4 w = ldcg4(pb + 4 * c);
                            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                            for (int b = 0; b < 16; ++b) {
                                const uint32_t by = (ww[b >> 2] >> (8 * (b & 3))) & 0xFF;
                                const uint2 e = *reinterpret_cast<const uint2*>(&lut[by * 2]);
                                v[2 * b] = e.x;
                                v[2 * b + 1] = e.y;
                            }
                        }
                        tc::tmem_st32(tbase + lane_addr + kColA + st * 32, v);
                        tc::tmem_wait_st();
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&S.a_full[st]);
                    }
                }
            }
        }
        if (prev) drain(s - 1);
        // the epilogue's arrivals for the last two tiles
        for (uint32_t sd = s >= 2 ? s - 2 : 0; sd < s; ++sd) named_sync(kBarDEmpty + (sd & 1));
    } else {
        // ===== epilogue warps
        const int e = warp - kEpiWarp0;
        uint32_t* ring = reinterpret_cast<uint32_t*>(sm + kOffRing) + e * kRing;
        double* nbuf = reinterpret_cast<double*>(sm + kOffNBuf) + e * kNBuf;
        const uint32_t lt = lanemask_lt();
        uint32_t s = 0;
        int ii = 0;
        for (long long it = blockIdx.x; it < a.nblocks; it += gridDim.x, ++ii) {
            ItemOf io = item_of(a, it);
            // opaque from here on: the 64-bit item decode must not be re-derived inside the loops
            asm volatile("" : "+r"(io.l), "+r"(io.run), "+r"(io.traj0), "+r"(io.count));
            const uint64_t key = run_key(a.seed, static_cast<uint32_t>(io.run));
            const uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
            const double c0h = __ddiv_rn(a.c0[io.l], static_cast<double>(a.H));
            bool nonfinite = false;
            // ---- init_state (solver.hpp:108-124): x, y from the init_x / init_y streams, spin
            //      i from words 2i, 2i+1 (block i/2); lanes 0-15 make the x blocks of a 32-spin
            //      window, lanes 16-31 the y blocks
            for (int jj = e; jj < kNTV; jj += kEpiWarps) {
                uint32_t* pb0 = a.phib + ((slot * 2 + 0) * kNT + jj) * a.nwp;
                if (jj >= io.count) continue;
                const long long rowb = (slot * kNT + jj) * static_cast<long long>(a.n);
                const uint32_t tr = static_cast<uint32_t>(io.traj0 + jj);
                for (int w0 = 0; w0 < a.nwp; w0 += 4) {
                    uint32_t bits[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int s0 = (w0 + u) * 32;
                        const uint32_t blk = static_cast<uint32_t>(s0 / 2 + (lane & 15));
                        const uint4 pv = philox(k0, k1, blk, tag_word(lane < 16 ? kTagInitX : kTagInitY, 0), tr,
                                                static_cast<uint32_t>(io.l));
                        const int src = lane >> 1;
                        const uint32_t xa = __shfl_sync(0xffffffffu, pv.x, src), xb = __shfl_sync(0xffffffffu, pv.y, src);
                        const uint32_t xc = __shfl_sync(0xffffffffu, pv.z, src), xd = __shfl_sync(0xffffffffu, pv.w, src);
                        const uint32_t ya = __shfl_sync(0xffffffffu, pv.x, src + 16), yb = __shfl_sync(0xffffffffu, pv.y, src + 16);
                        const uint32_t yc = __shfl_sync(0xffffffffu, pv.z, src + 16), yd = __shfl_sync(0xffffffffu, pv.w, src + 16);
                        const bool odd = lane & 1;
                        const int i = s0 + lane;
                        bool plus = false;
                        if (i < a.n) {
                            const double xv = __dmul_rn(a.init_scale, __dsub_rn(__dmul_rn(2.0, odd ? u01_from(xc, xd) : u01_from(xa, xb)), 1.0));
                            const double yv = __dmul_rn(a.init_scale, __dsub_rn(__dmul_rn(2.0, odd ? u01_from(yc, yd) : u01_from(ya, yb)), 1.0));
                            a.x[rowb + i] = xv;
                            a.y[rowb + i] = yv;
                            plus = !(xv < 0.0);
                        }
                        bits[u] = __ballot_sync(0xffffffffu, plus);
                    }
                    if (lane == 0) *reinterpret_cast<uint4*>(pb0 + w0) = make_uint4(bits[0], bits[1], bits[2], bits[3]);
                }
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&S.init_cnt, 1) == kEpiWarps - 1) {
                    S.init_cnt = 0;
                    __threadfence_block();
                    *reinterpret_cast<volatile int*>(&S.init_done) = ii + 1;
                }
            }
            // ---- the T steps. This warp's work units (t, tile m, trajectory jj) run in order. A
            //      unit first produces the tile's normals into nbuf (one loop over rounds), then
            //      updates its four 32-spin windows in straight-line code; the x / y of the next
            //      unit are loaded into each window's registers as soon as they are free.
            double xr[4], yr[4];
            double* const xs = a.x + slot * kNT * static_cast<long long>(a.n);  // this CTA's state rows
            double* const ys = a.y + slot * kNT * static_cast<long long>(a.n);
            if (e < io.count)
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int sp = 32 * g + lane;
                    xr[g] = sp < a.n ? xs[e * a.n + sp] : 0.0;
                    yr[g] = sp < a.n ? ys[e * a.n + sp] : 0.0;
                }
            for (int t = 0; t < a.T; ++t) {
                const double neg_drift = -__dsub_rn(a.a0, __ddiv_rn(static_cast<double>(t + 1), static_cast<double>(a.T)));
                const uint32_t lo = tag_word(kTagStepNoise, static_cast<uint32_t>(t));
                const bool last = t == a.T - 1;
                for (int jj = e; jj < kNTV; jj += kEpiWarps) pos[jj] = 0;  // own rows only
                for (int m = 0; m < nt; ++m, ++s) {
                    const uint32_t buf = s & 1;
                    tc::mbar_wait_sleep(&S.s_full[buf], (s >> 1) & 1, 128);  // the drain of tile s is complete
                    const int* D = reinterpret_cast<const int*>(sm + kOffD + buf * (kNT * kNS * 4));
                    const int sb = m * kNS;
                    const int ns = min(kNS, a.n - sb);  // spins of this tile
                    for (int jj = e; jj < io.count; jj += kEpiWarps) {
                        // the next unit of this warp
                        int nm = m, nj = jj + kEpiWarps;
                        bool has_next = true;
                        if (nj >= io.count) {
                            nj = e;
                            if (++nm == nt) {
                                nm = 0;
                                has_next = !last;
                            }
                        }
                        if (NOISY) {
                            // ---- the normals of this tile: (trajectory, step t) stream from the
                            //      position kept at the last tile (rng.hpp:156-185)
                            const uint32_t mid = static_cast<uint32_t>(io.traj0 + jj), hi = static_cast<uint32_t>(io.l);
                            int head = pos[jj], tail = head & ~3, ntl = 0, hlast = 0;
                            uint32_t plast = 0;
                            while (ntl < ns) {
                                if (tail - head < 40) {  // 32 Philox blocks: 128 words (a round reads <= 34 ahead)
                                    const uint4 v = philox(k0, k1, static_cast<uint32_t>(tail >> 2) + static_cast<uint32_t>(lane), lo, mid, hi);
                                    *reinterpret_cast<uint4*>(&ring[(tail + 4 * lane) & (kRing - 1)]) = v;
                                    tail += 128;
                                    __syncwarp();
                                }
                                // one round: lane L tests word head + L
                                const int H0 = head;
                                const uint32_t u = ring[(H0 + lane) & (kRing - 1)];
                                const bool slow = !(zmag32(u) < z.kn[u & 127u]);
                                const uint32_t smk = __ballot_sync(0xffffffffu, slow);
                                double v = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), z.wn[u & 127u]);
                                uint32_t prod = 0xffffffffu;
                                int end = 32;
                                if (smk) {
                                    // every slow word is tested as if it started an attempt (the ones inside
                                    // an earlier attempt are dropped below): wedges take 3 words, tails 1 + 4k
                                    bool good = !slow;
                                    int len = 1;
                                    if (slow) {
                                        if (u & 127u) {
                                            good = wedge_accept(u, ring[(H0 + lane + 1) & (kRing - 1)], ring[(H0 + lane + 2) & (kRing - 1)], z);
                                            len = 3;
                                        } else {  // tail: always a normal
                                            const TailOut to = tail_attempt(ring, tail, H0 + lane, u, k0, k1, lo, mid, hi);
                                            v = to.v;
                                            len = to.len;
                                            good = true;
                                        }
                                    }
                                    const uint32_t gm = __ballot_sync(0xffffffffu, good);
                                    uint32_t cons = 0, rem = smk;
                                    while (rem) {  // the attempts in order; their extra words are consumed
                                        const int qb = __ffs(rem) - 1;
                                        const int lq = __shfl_sync(0xffffffffu, len, qb);
                                        const uint32_t span = qb + lq >= 32 ? ~0u << qb : ((1u << lq) - 1u) << qb;
                                        cons |= span & ~(1u << qb);
                                        rem &= ~span;
                                        end = qb + lq > end ? qb + lq : end;
                                    }
                                    prod = gm & ~cons;
                                }
                                if ((prod >> lane) & 1u) nbuf[ntl + __popc(prod & lt)] = v;
                                ntl += __popc(prod);
                                head = H0 + end;
                                hlast = H0;
                                plast = prod;
                            }
                            const int left = ntl - ns;
                            if (left > 0) {  // next tile starts at the (k - left)-th producing word of the last round
                                const int idx = __popc(plast & lt);
                                const uint32_t hit = __ballot_sync(0xffffffffu, ((plast >> lane) & 1u) && idx == __popc(plast) - left);
                                head = hlast + __ffs(hit) - 1;
                            }
                            if (lane == 0) pos[jj] = head;
                            __syncwarp();
                        }
                        // ---- the updates (sb_step solver.hpp:159-181, phi = sgn(x)) of the four windows
                        double* xp = xs + jj * a.n + sb;
                        double* yp = ys + jj * a.n + sb;
                        const double* xnp = xs + nj * a.n + nm * kNS;
                        const double* ynp = ys + nj * a.n + nm * kNS;
                        const int nsn = min(kNS, a.n - nm * kNS);
                        uint32_t mybits = 0;  // lane g keeps the sign bits of window g
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            const int cnt = ns - 32 * g;
                            if (cnt > 0) {
                                bool plus = false;
                                if (lane < cnt) {
                                    const int dq = D[dsw(jj, 32 * g + lane)];
                                    double xi = xr[g], yi = yr[g];
                                    double d = __dsub_rn(__dmul_rn(neg_drift, xi), __dmul_rn(c0h, static_cast<double>(dq)));
                                    if (NOISY) d = __dadd_rn(d, __dmul_rn(a.alpha, nbuf[32 * g + lane]));
                                    yi = __dadd_rn(yi, UDT ? d : __dmul_rn(a.dt, d));
                                    xi = __dadd_rn(xi, UDT ? yi : __dmul_rn(a.sdt, yi));
                                    if (fabs(xi) > 1.0) {  // wall + clamp (both fire exactly when |x| > 1)
                                        yi = 0.0;
                                        xi = __hiloint2double((__double2hiint(xi) & static_cast<int>(0x80000000u)) | 0x3FF00000, 0);
                                    }
                                    // the first step with a non-finite x or y has a non-finite y
                                    nonfinite |= !(fabs(yi) <= 1.7976931348623157e308);
                                    xp[32 * g + lane] = xi;
                                    yp[32 * g + lane] = yi;
                                    plus = !(xi < 0.0);
                                }
                                const uint32_t b = __ballot_sync(0xffffffffu, plus);
                                if (lane == g) mybits = b;
                            }
                        }
                        // the next unit's x / y, all eight loads together: the next unit's noise phase
                        // covers their latency, and no wait of this unit shares a scoreboard with them
                        if (has_next)
#pragma unroll
                            for (int g = 0; g < 4; ++g)
                                if (32 * g + lane < nsn) {
                                    xr[g] = xnp[32 * g + lane];
                                    yr[g] = ynp[32 * g + lane];
                                }
                        if (!last) {
                            uint32_t* pbn = a.phib + ((slot * 2 + ((t + 1) & 1)) * kNT + jj) * a.nwp;
                            if (lane < 4) pbn[4 * m + lane] = mybits;
                        } else {  // read_spins + pack (solver.hpp:237-244, :288-297): 32-bit halves of the words
                            const long long row = (static_cast<long long>(io.run) * a.L + io.l) * a.batch + io.traj0 + jj - a.row0;
                            uint32_t* wr = reinterpret_cast<uint32_t*>(a.words + row * a.wpc);
                            if (lane < 4 && 4 * m + lane < 2 * a.wpc) wr[4 * m + lane] = mybits;
                        }
                        __syncwarp();  // nbuf is rewritten by the next unit
                    }
                    // tile done for this warp
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        if (atomicAdd(&S.epi_cnt[buf], 1) == kEpiWarps - 1) {
                            S.epi_cnt[buf] = 0;
                            __threadfence_block();
                            *reinterpret_cast<volatile int*>(&S.tiles_done) = static_cast<int>(s) + 1;
                            if (last && m == nt - 1 && a.block_end_ns) a.block_end_ns[it] = gtimer();
                        }
                    }
                    named_arrive(kBarDEmpty + buf);  // this warp is done with the D tile
                }
            }
            if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&a.nan_block[it], 1);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<kTmemCols>(tbase);
}

// TMA descriptor of a row-major matrix of 1- or 2-byte elements (rows x cols, row pitch
// cols * esize a multiple of 16): boxes of 128 bytes x 128 rows, 128-byte swizzle, zero fill
// outside
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap make_tmap(const void* base, long long rows, int cols, int esize)
{
    static PFN_encodeTiled encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q), "driver entry point");
        if (!fn || q != cudaDriverEntryPointSuccess) runtime("cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_encodeTiled>(fn);
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * esize};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esize), 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&m, esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
                              const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) runtime("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

struct DenseScratch {
    DevBuf<uint8_t> hj;           // H*J(c) per weight, int8 or bf16 bits
    DevBuf<double> x, y;          // in-flight state, [grid][128][n]
    DevBuf<uint32_t> phib;        // in-flight sign bits
    DevBuf<int> flags;
    long long hj_inst = -1, hj_weights = -1;  // H*J(c) built for this instance / lattice generation
    int hj_bf16 = 0, hj_npad = 0;
    DevBuf<uint8_t> wk;           // the K weight layers, dense int8, per instance (evaluate_cuts)
    long long wk_gen = -1;
    DevBuf<uint8_t> s8;           // evaluate_cuts: expanded spin configs (unused by the fused form)
};

DenseScratch& dscratch(Ctx& c)
{
    if (!c.dense_scratch) c.dense_scratch = std::shared_ptr<void>(new DenseScratch(), [](void* p) {
        auto* d = static_cast<DenseScratch*>(p);
        d->hj.release(); d->x.release(); d->y.release(); d->phib.release(); d->flags.release(); d->wk.release();
        d->s8.release();
        delete d;
    });
    return *static_cast<DenseScratch*>(c.dense_scratch.get());
}

// bound on |H*J(c)_ij| over the lattice: sum_k num_k max_e |w_k(e)|
long long hj_bound(Ctx& c)
{
    std::vector<int> nums(static_cast<size_t>(c.L) * c.k);
    ck(cudaMemcpy(nums.data(), c.d_nums.p, sizeof(int) * nums.size(), cudaMemcpyDeviceToHost), "D2H");
    std::vector<double> wmax(static_cast<size_t>(c.k), 0.0);
    for (int e = 0; e < c.m; ++e)
        for (int q = 0; q < c.k; ++q)
            wmax[static_cast<size_t>(q)] = std::max(wmax[static_cast<size_t>(q)], std::fabs(c.h_w[static_cast<size_t>(e) * c.k + q]));
    long long maxabs = 0;
    for (int l = 0; l < c.L; ++l) {
        double s = 0;
        for (int q = 0; q < c.k; ++q) s += nums[static_cast<size_t>(l) * c.k + q] * wmax[static_cast<size_t>(q)];
        maxabs = std::max(maxabs, static_cast<long long>(s));
    }
    return maxabs;
}

template <bool BF16, bool NOISY, bool UDT>
void launch_fused(const CUtensorMap& tm, const FusedArgs& fa, int grid, cudaStream_t st)
{
    auto kern = k_dense_fused<BF16, NOISY, UDT>;
    ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes), "smem attribute");
    cudaFuncAttributes fa_attr{};
    ck(cudaFuncGetAttributes(&fa_attr, kern), "function attributes");
    if (fa_attr.maxThreadsPerBlock < kThreads)
        runtime("dense sampler: " + std::to_string(fa_attr.numRegs) + " registers per thread allow only " +
                std::to_string(fa_attr.maxThreadsPerBlock) + " threads");
    kern<<<grid, kThreads, kSmemBytes, st>>>(tm, fa);
}


// ---- evaluate_cuts on the tensor cores (pareto.hpp:346-359): for layer k,
// h_k(u) = s_u^T W_k s_u and C_k(u) = 0.5 (W_k - 0.5 h_k(u)), exact for integer |w| <= 127.
// One work item = 128 configs (MMA M, TMEM lanes; A = the +-1 spins expanded from the packed
// words into TMEM), walked over the K layers and the spin tiles of 128 (B = the W_k tile by
// TMA); the epilogue thread of config u reads its row of D = S W_k^T (tcgen05.ld) and dots it
// with s_u over the tile's spins. No product ever touches HBM.
constexpr int kEvWarps = 9;  // 0: MMA, 1..4: io (expand A, TMA B), 5..8: epilogue
constexpr int kEvSmem = kStages * kBStage + 256 * 8 + 1024;

struct EvalArgs {
    int n, K, ntiles, nchunks, wpc;
    long long U;
    const uint64_t* words;
    const uint32_t* idx;  // optional row indices into words
    const double* W;      // [K] layer totals
    double* out;          // [U][K]
};

__global__ void __launch_bounds__(kEvWarps * 32, 1) k_eval_tc(const __grid_constant__ CUtensorMap tmW,
                                                             const __grid_constant__ EvalArgs a)
{
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    __shared__ uint64_t b_full[kStages], b_empty[kStages], a_full[kStages], a_empty[kStages], d_full[2], d_empty[2];
    __shared__ uint32_t tslot;
    uint32_t* lut = reinterpret_cast<uint32_t*>(sm + kStages * kBStage);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int b = tid; b < 256; b += blockDim.x)
        for (int w = 0; w < 2; ++w) {
            uint32_t v = 0;
            for (int q = 0; q < 4; ++q) v |= ((b >> (4 * w + q)) & 1 ? 0x01u : 0xFFu) << (8 * q);
            lut[b * 2 + w] = v;
        }
    if (tid == 0) {
        for (int q = 0; q < kStages; ++q) {
            tc::mbar_init(&b_full[q], 1);
            tc::mbar_init(&b_empty[q], 1);
            tc::mbar_init(&a_full[q], 4);
            tc::mbar_init(&a_empty[q], 1);
        }
        for (int q = 0; q < 2; ++q) {
            tc::mbar_init(&d_full[q], 1);
            tc::mbar_init(&d_empty[q], 4);
        }
        tc::fence_mbar_init();
        tc::prefetch_tmap(&tmW);
    }
    if (warp == 0) tc::tmem_alloc<kTmemCols>(&tslot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tslot;
    const long long items = (a.U + kNT - 1) / kNT;
    const int nt = a.ntiles, nch = a.nchunks;
    auto row_of = [&](long long u) -> long long {
        if (u >= a.U) u = a.U - 1;  // padding rows of the last item: any valid config
        return a.idx ? static_cast<long long>(a.idx[u]) : u;
    };
    if (warp == 0) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_i8(kNT, kNS);
            uint32_t g = 0, s = 0;
            for (long long it = blockIdx.x; it < items; it += gridDim.x)
                for (int k = 0; k < a.K; ++k)
                    for (int m = 0; m < nt; ++m, ++s) {
                        const uint32_t buf = s & 1;
                        tc::mbar_wait(&d_empty[buf], ((s >> 1) & 1) ^ 1);
                        tc::fence_after();
                        for (int c = 0; c < nch; ++c, ++g) {
                            const uint32_t st = g % kStages, ph = (g / kStages) & 1;
                            tc::mbar_wait(&a_full[st], ph);
                            tc::mbar_wait(&b_full[st], ph);
                            tc::fence_after();
                            const uint32_t bs = tc::smem_u32(sm + st * kBStage);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                tc::mma_i8_ts(tbase + buf * kNS, tbase + kColA + st * 32 + 8 * kk,
                                              tc::smem_desc_sw128(bs + 32 * kk), idesc, c > 0 || kk > 0);
                            tc::commit(&a_empty[st]);
                            tc::commit(&b_empty[st]);
                        }
                        tc::commit(&d_full[buf]);
                    }
        }
        __syncwarp();
    } else if (warp < 5) {
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
        uint32_t g = 0;
        for (long long it = blockIdx.x; it < items; it += gridDim.x) {
            const uint32_t* wr = reinterpret_cast<const uint32_t*>(a.words + row_of(it * kNT + r) * a.wpc);
            for (int k = 0; k < a.K; ++k)
                for (int m = 0; m < nt; ++m)
                    for (int c = 0; c < nch; ++c, ++g) {
                        const uint32_t st = g % kStages, ph = (g / kStages) & 1;
                        tc::mbar_wait(&a_empty[st], ph ^ 1);
                        if (q == 0 && lane == 0) {
                            tc::mbar_wait(&b_empty[st], ph ^ 1);
                            tc::mbar_expect_tx(&b_full[st], kBStage);
                            tc::tma_load_2d(sm + st * kBStage, &tmW, c * 128, k * a.n + m * kNS, &b_full[st]);
                        }
                        uint32_t ww[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) ww[h] = 4 * c + h < 2 * a.wpc ? wr[4 * c + h] : 0u;
                        uint32_t v[32];
#pragma unroll
                        for (int b = 0; b < 16; ++b) {
                            const uint2 e = *reinterpret_cast<const uint2*>(&lut[((ww[b >> 2] >> (8 * (b & 3))) & 0xFF) * 2]);
                            v[2 * b] = e.x;
                            v[2 * b + 1] = e.y;
                        }
                        tc::tmem_st32(tbase + lane_addr + kColA + st * 32, v);
                        tc::tmem_wait_st();
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&a_full[st]);
                    }
        }
    } else {
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
        uint32_t s = 0;
        for (long long it = blockIdx.x; it < items; it += gridDim.x) {
            const long long u = it * kNT + r;
            const uint32_t* wr = reinterpret_cast<const uint32_t*>(a.words + row_of(u) * a.wpc);
            for (int k = 0; k < a.K; ++k) {
                long long h = 0;
                for (int m = 0; m < nt; ++m, ++s) {
                    const uint32_t buf = s & 1;
                    tc::mbar_wait(&d_full[buf], (s >> 1) & 1);
                    tc::fence_after();
#pragma unroll 1
                    for (int cg = 0; cg < kNS / 32; ++cg) {
                        uint32_t v[32];
                        tc::tmem_ld32(tbase + lane_addr + buf * kNS + cg * 32, v);
                        const int s0 = m * kNS + cg * 32;
                        const uint32_t bw = s0 < a.n ? wr[s0 >> 5] : 0u;
                        const int lim = min(32, a.n - s0);
                        int part = 0;
#pragma unroll
                        for (int b = 0; b < 32; ++b) {
                            const int dv = static_cast<int>(v[b]);
                            if (b < lim) part += ((bw >> b) & 1u) ? dv : -dv;
                        }
                        h += part;
                    }
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&d_empty[buf]);
                }
                if (u < a.U) a.out[u * a.K + k] = 0.5 * (a.W[k] - 0.5 * static_cast<double>(h));
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<kTmemCols>(tbase);
}

__global__ void k_build_layers(int n, int npad, int k, const int* __restrict__ rowptr, const int* __restrict__ col,
                               const int* __restrict__ eidx, const int* __restrict__ wi, int8_t* Wk)
{
    const int layer = blockIdx.y, i = blockIdx.x;
    int8_t* row = Wk + (static_cast<long long>(layer) * n + i) * npad;
    for (int j = threadIdx.x; j < npad; j += blockDim.x) row[j] = 0;
    __syncthreads();
    for (int e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x)
        row[col[e]] = static_cast<int8_t>(wi[static_cast<long long>(eidx[e]) * k + layer]);
}

}  // namespace

// 0: no dense path; 1: int8 (|H*J| <= 127); 2: bf16 (|H*J| <= 256). dSB with integer weights
// and n >= the dense threshold only (bSB's phi = x has no exact narrow operand).
int dense_path_kind(Ctx& c, int variant)
{
    if (variant != 1 || !c.integer_weights || c.n < c.dense_min_n || c.L < 1 || c.H < 1) return 0;
    const long long b = hj_bound(c);
    return b <= 127 ? 1 : b <= 256 ? 2 : 0;
}
bool dense_path_ok(Ctx& c, int variant) { return dense_path_kind(c, variant) != 0; }

int dense_block_traj() { return kNTV; }

// Samples the flattened (run, weight, chunk) blocks [b0, b0+nblocks) of 120 trajectories
// (p.block_traj) with the fused tensor-core kernel.
void sample_dense(Ctx& c, const SamplerParams& p, long long b0, long long nblocks)
{
    if (p.block_traj != kNTV) runtime("dense path: block size must be " + std::to_string(kNTV) + " trajectories");
    DenseScratch& d = dscratch(c);
    const int kind = dense_path_kind(c, p.variant);
    if (!kind) runtime("dense path not applicable");
    const bool bf16 = kind == 2;
    const int n = c.n, L = c.L;
    const int npad = bf16 ? (n + 7) / 8 * 8 : (n + 15) / 16 * 16;
    const int esize = bf16 ? 2 : 1;
    if (d.hj_inst != c.inst_gen || d.hj_weights != c.weights_gen || d.hj_bf16 != static_cast<int>(bf16) || d.hj_npad != npad) {
        d.hj.reserve(static_cast<size_t>(L) * n * npad * esize);
        d.flags.reserve(4);
        ck(cudaMemsetAsync(d.flags.p, 0, sizeof(int) * 4, c.stream), "memset");
        k_build_hj<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>(L)), 256, 0, c.stream>>>(
            n, npad, c.k, c.d_nums.p, c.d_rowptr.p, c.d_col.p, c.d_eidx.p, c.d_wi.p, d.hj.p, bf16 ? 1 : 0, d.flags.p);
        c.launches++;
        int mx = 0;
        ck(cudaMemcpyAsync(&mx, d.flags.p, sizeof mx, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "hj");
        if (mx > (bf16 ? 256 : 127)) runtime("dense path: H*J(c) exceeds the operand range");
        d.hj_inst = c.inst_gen;
        d.hj_weights = c.weights_gen;
        d.hj_bf16 = bf16;
        d.hj_npad = npad;
    }
    int dev = 0, sms = 0;
    ck(cudaGetDevice(&dev), "device");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
    const int grid = static_cast<int>(std::min<long long>(nblocks, sms));
    if (grid < 1) return;
    const int ntiles = (n + kNS - 1) / kNS;
    const int nwp = ntiles * 4;
    d.x.reserve(static_cast<size_t>(grid) * kNT * n);
    d.y.reserve(static_cast<size_t>(grid) * kNT * n);
    d.phib.reserve(static_cast<size_t>(grid) * 2 * kNT * nwp);
    FusedArgs fa{};
    fa.n = n;
    fa.T = p.T;
    fa.L = L;
    fa.batch = p.batch;
    fa.chunks = p.chunks;
    fa.ntiles = ntiles;
    fa.nchunks = (n + (bf16 ? 64 : 128) - 1) / (bf16 ? 64 : 128);
    fa.nwp = nwp;
    fa.wpc = (n + 63) / 64;
    fa.H = c.H;
    fa.b0 = b0;
    fa.nblocks = nblocks;
    fa.seed = p.seed;
    fa.dt = p.dt;
    fa.a0 = p.a0;
    fa.alpha = p.alpha;
    fa.sdt = p.s_dt_a0;
    fa.init_scale = p.init_scale;
    fa.c0 = p.c0;
    fa.zig = p.zig;
    fa.x = d.x.p;
    fa.y = d.y.p;
    fa.phib = d.phib.p;
    fa.words = p.words;
    fa.row0 = p.row0;
    fa.block_end_ns = p.block_end_ns;
    fa.nan_block = p.nan_block;
    const CUtensorMap tm = make_tmap(d.hj.p, static_cast<long long>(L) * n, npad, esize);
    const bool noisy = p.alpha > 0.0, udt = p.dt == 1.0 && p.s_dt_a0 == 1.0;
    if (bf16) {
        if (noisy) udt ? launch_fused<true, true, true>(tm, fa, grid, c.stream) : launch_fused<true, true, false>(tm, fa, grid, c.stream);
        else udt ? launch_fused<true, false, true>(tm, fa, grid, c.stream) : launch_fused<true, false, false>(tm, fa, grid, c.stream);
    } else {
        if (noisy) udt ? launch_fused<false, true, true>(tm, fa, grid, c.stream) : launch_fused<false, true, false>(tm, fa, grid, c.stream);
        else udt ? launch_fused<false, false, true>(tm, fa, grid, c.stream) : launch_fused<false, false, false>(tm, fa, grid, c.stream);
    }
    c.launches++;
    ck(cudaGetLastError(), "dense sampler");
}

// evaluate_cuts through the tensor cores when every weight is an integer with |w| <= 127 and
// n is at least the dense threshold
bool eval_gemm_ok(const Ctx& c)
{
    if (!c.integer_weights || c.n < c.dense_min_n) return false;
    for (double v : c.h_w)
        if (v > 127 || v < -127) return false;
    return true;
}

void evaluate_cuts_gemm(Ctx& c, const uint64_t* d_words, const uint32_t* d_idx, long long U, double* d_out)
{
    if (U <= 0) return;
    DenseScratch& d = dscratch(c);
    const int n = c.n, K = c.k;
    const int npad = (n + 15) / 16 * 16;
    if (d.wk_gen != c.inst_gen) {  // dense int8 layers [K][n][npad], built once per instance
        d.wk.reserve(static_cast<size_t>(K) * n * npad);
        k_build_layers<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>(K)), 256, 0, c.stream>>>(
            n, npad, K, c.d_rowptr.p, c.d_col.p, c.d_eidx.p, c.d_wi.p, reinterpret_cast<int8_t*>(d.wk.p));
        c.launches++;
        d.wk_gen = c.inst_gen;
    }
    std::vector<double> W(static_cast<size_t>(K), 0.0);
    for (int e = 0; e < c.m; ++e)
        for (int q = 0; q < K; ++q) W[static_cast<size_t>(q)] += c.h_w[static_cast<size_t>(e) * K + q];
    d.flags.reserve(8);
    DevBuf<double> dW;
    dW.reserve(static_cast<size_t>(K));
    ck(cudaMemcpyAsync(dW.p, W.data(), sizeof(double) * K, cudaMemcpyHostToDevice, c.stream), "H2D");
    EvalArgs ea{};
    ea.n = n;
    ea.K = K;
    ea.ntiles = (n + kNS - 1) / kNS;
    ea.nchunks = (n + 127) / 128;
    ea.wpc = (n + 63) / 64;
    ea.U = U;
    ea.words = d_words;
    ea.idx = d_idx;
    ea.W = dW.p;
    ea.out = d_out;
    const CUtensorMap tm = make_tmap(d.wk.p, static_cast<long long>(K) * n, npad, 1);
    int dev = 0, sms = 0;
    ck(cudaGetDevice(&dev), "device");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
    const long long items = (U + kNT - 1) / kNT;
    const int grid = static_cast<int>(std::min<long long>(items, sms));
    ck(cudaFuncSetAttribute(k_eval_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kEvSmem), "smem attribute");
    k_eval_tc<<<grid, kEvWarps * 32, kEvSmem, c.stream>>>(tm, ea);
    c.launches++;
    ck(cudaGetLastError(), "evaluate_cuts (tensor cores)");
    dW.release();
}

}  // namespace momc_b200
