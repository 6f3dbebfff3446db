#pragma once
// SB sampler kernel implementation (see sampler.cuh), included by sampler_n*.cu. Design:
//   * one trajectory per thread, 128 trajectories of one (run, weight) per CTA;
//   * x (and y for n <= 42) live in registers, fully unrolled over NMAX spins;
//   * the coupling J(c_l) is a CSR row list in shared memory (broadcast reads); bSB/SimCIM
//     gather phi(x_j) = x_j from a per-thread column of shared memory, dSB gathers
//     sgn(x_j) from a 64-bit sign mask held in a register;
//   * per step, the Philox blocks of the (trajectory, step) noise stream are generated
//     up-front into shared memory (uniform work, no divergence), then the ziggurat
//     consumes them sequentially (rng.hpp:156-185) in groups of 8 spins, each group
//     immediately feeding its 8 spin updates;
//   * every FP64 operation uses an explicitly rounded intrinsic (__dmul_rn/__dadd_rn/
//     __dsub_rn) in the reference's order, so nvcc cannot contract into FMA.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "sampler.cuh"

namespace momc_b200 {

namespace sbimpl {

constexpr int kGroup = 8;  // spins whose normals are produced, then consumed, together

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct NoiseCursor {
    const uint32_t* ubuf;  // [NU][kSampleBlock] u32 of the current stream (this thread's column)
    int nu;                // pre-generated words
    int pos;               // next word
    uint32_t k0, k1, lo, mid, hi;

    __device__ __forceinline__ uint32_t fetch()
    {
        const int p = pos++;
        if (p < nu) return ubuf[p * kSampleBlock];
        // overflow past the pre-generated blocks (several slow draws in one step): recompute
        const uint4 b = philox(k0, k1, static_cast<uint32_t>(p >> 2), lo, mid, hi);
        const int q = p & 3;
        return q == 0 ? b.x : (q == 1 ? b.y : (q == 2 ? b.z : b.w));
    }
};

// rng.hpp:156-185 Stream::next_normal, words taken from the cursor in stream order.
__device__ __forceinline__ double next_normal(NoiseCursor& c, const uint32_t* __restrict__ kn,
                                              const double* __restrict__ wn, const double* __restrict__ fn)
{
    for (;;) {
        const uint32_t u = c.fetch();
        const int32_t hz = static_cast<int32_t>(u);
        const uint32_t iz = u & 127u;
        const uint32_t mag = hz < 0 ? static_cast<uint32_t>(-static_cast<int64_t>(hz)) : static_cast<uint32_t>(hz);
        if (mag < kn[iz]) return __dmul_rn(static_cast<double>(hz), wn[iz]);
        if (iz == 0) {
            const double r = 3.442619855899;
            for (;;) {
                const uint32_t a0 = c.fetch(), a1 = c.fetch();
                const double x = __ddiv_rn(-log(u01_open_from(a0, a1)), r);
                const uint32_t b0 = c.fetch(), b1 = c.fetch();
                const double y = -log(u01_open_from(b0, b1));
                if (__dadd_rn(y, y) >= __dmul_rn(x, x)) return hz > 0 ? __dadd_rn(r, x) : -__dadd_rn(r, x);
            }
        }
        const double x = __dmul_rn(static_cast<double>(hz), wn[iz]);
        const uint32_t a0 = c.fetch(), a1 = c.fetch();
        const double lhs = __dadd_rn(fn[iz], __dmul_rn(u01_from(a0, a1), __dsub_rn(fn[iz - 1], fn[iz])));
        if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return x;
    }
}

// Shared-memory carve-up for one CTA.
template <int NMAX>
struct SmemLayout {
    static constexpr int kNU = 4 * ((NMAX + 3) / 4 + 1);  // pre-generated u32 per step
    // byte offsets (all 16-B aligned)
    static constexpr int zig = 0;                                            // ZigTables (2560 B)
    static constexpr int ubuf = 2560;                                        // kNU * 128 * 4
    static constexpr int noise = ubuf + kNU * kSampleBlock * 4;              // kGroup * 128 * 8
    static constexpr int xs = noise + kGroup * kSampleBlock * 8;             // NMAX * 128 * 8 (bsb/simcim)
    __host__ __device__ static constexpr int ys_of(bool gather) { return xs + (gather ? NMAX * kSampleBlock * 8 : 0); }
    __host__ __device__ static constexpr int csr_of(bool gather, bool ys)
    {
        return ys_of(gather) + (ys ? NMAX * kSampleBlock * 8 : 0);
    }
};

template <int NMAX>
__host__ __device__ constexpr bool y_in_smem()
{
    return NMAX > 42;
}

// Register-resident integrator for n <= NMAX <= 64.
template <int NMAX, int VAR>
__global__ void __launch_bounds__(kSampleBlock, 2) sb_small_kernel(const SamplerParams p)
{
    constexpr bool kGather = VAR != 1;  // bsb / simcim gather x_j values; dsb uses a sign mask
    constexpr bool kYS = y_in_smem<NMAX>();
    using SL = SmemLayout<NMAX>;
    extern __shared__ __align__(16) unsigned char smem[];
    ZigTables* zig = reinterpret_cast<ZigTables*>(smem + SL::zig);
    uint32_t* ubuf = reinterpret_cast<uint32_t*>(smem + SL::ubuf);
    double* noise_s = reinterpret_cast<double*>(smem + SL::noise);
    double* xs = reinterpret_cast<double*>(smem + SL::xs);
    double* ys = reinterpret_cast<double*>(smem + SL::ys_of(kGather));
    unsigned char* csr = smem + SL::csr_of(kGather, kYS);
    int* rp = reinterpret_cast<int*>(csr);                                         // NMAX + 1
    double* cv = reinterpret_cast<double*>(csr + ((NMAX + 1) * 4 + 15) / 16 * 16);  // nnz
    int* cc = reinterpret_cast<int*>(cv + p.nnz);                                   // nnz

    const int n = p.n;
    const long long gblock = p.block_begin + blockIdx.x;
    const int chunk = static_cast<int>(gblock % p.chunks);
    const long long rl = gblock / p.chunks;
    const int l = static_cast<int>(rl % p.L);
    const int run = static_cast<int>(rl / p.L);
    const int tid = threadIdx.x;

    // ---- CTA setup: ziggurat tables, CSR of J(c_l)
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.zig);
        uint32_t* dst = reinterpret_cast<uint32_t*>(zig);
        for (int i = tid; i < static_cast<int>(sizeof(ZigTables) / 4); i += kSampleBlock) dst[i] = src[i];
        for (int i = tid; i <= n; i += kSampleBlock) rp[i] = p.row_ptr[i];
        const double* v = p.vals + static_cast<long long>(l) * p.nnz;
        for (int i = tid; i < p.nnz; i += kSampleBlock) {
            cv[i] = v[i];
            cc[i] = p.col[i];
        }
    }
    __syncthreads();

    const int traj = chunk * kSampleBlock + tid;
    if (traj >= p.batch) return;  // no CTA-wide barrier below this point

    const uint64_t key = run_key(p.seed, static_cast<uint32_t>(run));
    const uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
    const uint32_t wl = static_cast<uint32_t>(l), tr = static_cast<uint32_t>(traj);
    const double c0 = p.c0[l];

    // ---- init_state (solver.hpp:108-124): x then y, one next_symmetric per spin
    double x[NMAX];
    double y[kYS ? 1 : NMAX];
#pragma unroll
    for (int b = 0; b < (NMAX + 1) / 2; ++b) {
        if (2 * b < n) {
            const uint4 rx = philox(k0, k1, b, tag_word(kTagInitX, 0), tr, wl);
            x[2 * b] = __dmul_rn(p.init_scale, __dsub_rn(__dmul_rn(2.0, u01_from(rx.x, rx.y)), 1.0));
            if (2 * b + 1 < NMAX)
                x[2 * b + 1] = __dmul_rn(p.init_scale, __dsub_rn(__dmul_rn(2.0, u01_from(rx.z, rx.w)), 1.0));
            const uint4 ry = philox(k0, k1, b, tag_word(kTagInitY, 0), tr, wl);
            const double y0 = __dmul_rn(p.init_scale, __dsub_rn(__dmul_rn(2.0, u01_from(ry.x, ry.y)), 1.0));
            const double y1 = __dmul_rn(p.init_scale, __dsub_rn(__dmul_rn(2.0, u01_from(ry.z, ry.w)), 1.0));
            if constexpr (kYS) {
                ys[(2 * b) * kSampleBlock + tid] = y0;
                if (2 * b + 1 < NMAX) ys[(2 * b + 1) * kSampleBlock + tid] = y1;
            } else {
                y[2 * b] = y0;
                if (2 * b + 1 < NMAX) y[2 * b + 1] = y1;
            }
        } else {
            x[2 * b] = 0.0;
            if (2 * b + 1 < NMAX) x[2 * b + 1] = 0.0;
            if constexpr (!kYS) {
                y[2 * b] = 0.0;
                if (2 * b + 1 < NMAX) y[2 * b + 1] = 0.0;
            }
        }
    }
    // spins past n stay exactly 0 and are never read

    uint64_t negmask = 0;  // dsb: bit j set iff x_j < 0 (phi_j = -1)
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
        if (i < n) {
            if constexpr (kGather) xs[i * kSampleBlock + tid] = x[i];
            negmask |= static_cast<uint64_t>(x[i] < 0.0) << i;
        }
    }

    const uint32_t* kn = zig->kn;
    const double* wn = zig->wn;
    const double* fn = zig->fn;
    const bool noisy = p.alpha > 0.0;
    int first_bad = 0;

    for (int t = 0; t < p.T; ++t) {
        const double a_t = __ddiv_rn(static_cast<double>(t + 1), static_cast<double>(p.T));
        const double neg_drift = -__dsub_rn(p.a0, a_t);             // -(a0 - a_t)
        const double pump = __dmul_rn(-0.5, __dsub_rn(1.0, a_t));   // simcim_schedule
        const uint32_t lo = tag_word(kTagStepNoise, static_cast<uint32_t>(t));

        NoiseCursor cur;
        if (noisy) {
            // fill_step_noise (solver.hpp:128-136): stream (key, l, traj, tag_word(step_noise, t))
#pragma unroll
            for (int b = 0; b < SL::kNU / 4; ++b) {
                const uint4 r = philox(k0, k1, b, lo, tr, wl);
                ubuf[(4 * b + 0) * kSampleBlock + tid] = r.x;
                ubuf[(4 * b + 1) * kSampleBlock + tid] = r.y;
                ubuf[(4 * b + 2) * kSampleBlock + tid] = r.z;
                ubuf[(4 * b + 3) * kSampleBlock + tid] = r.w;
            }
            cur.ubuf = ubuf + tid;
            cur.nu = SL::kNU;
            cur.pos = 0;
            cur.k0 = k0;
            cur.k1 = k1;
            cur.lo = lo;
            cur.mid = tr;
            cur.hi = wl;
        }

        uint64_t newmask = 0;
#pragma unroll
        for (int g = 0; g < (NMAX + kGroup - 1) / kGroup; ++g) {
            if (g * kGroup < n) {
                if (noisy) {
                    const int cnt = min(kGroup, n - g * kGroup);
                    for (int q = 0; q < cnt; ++q) noise_s[q * kSampleBlock + tid] = next_normal(cur, kn, wn, fn);
                }
#pragma unroll
                for (int q = 0; q < kGroup; ++q) {
                    const int i = g * kGroup + q;
                    if (i < NMAX && i < n) {
                        // coupled_i = sum_j J_ij phi(x_j), j ascending, from +0.0 (shim GEMM order)
                        double coupled = 0.0;
                        const int e1 = rp[i + 1];
                        for (int e = rp[i]; e < e1; ++e) {
                            const int j = cc[e];
                            const double v = cv[e];
                            double term;
                            if constexpr (VAR == 1) {
                                term = ((negmask >> j) & 1ull) ? -v : v;  // J * (+-1) is exact
                            } else {
                                term = __dmul_rn(v, xs[j * kSampleBlock + tid]);
                            }
                            coupled = __dadd_rn(coupled, term);
                        }
                        double yi;
                        if constexpr (kYS) yi = ys[i * kSampleBlock + tid];
                        else yi = y[i];
                        double xi = x[i];
                        const double eta = noisy ? noise_s[q * kSampleBlock + tid] : 0.0;
                        if constexpr (VAR == 2) {
                            // simcim_step (solver.hpp:199-210)
                            double d = __dsub_rn(__dmul_rn(pump, xi), __dmul_rn(c0, coupled));
                            if (noisy) d = __dadd_rn(d, __dmul_rn(p.alpha, eta));
                            yi = __dadd_rn(__dmul_rn(0.9, yi), __dmul_rn(1.0 - 0.9, d));
                            xi = __dadd_rn(xi, __dmul_rn(p.dt, yi));
                        } else {
                            // sb_step (solver.hpp:167-178)
                            double d = __dsub_rn(__dmul_rn(neg_drift, xi), __dmul_rn(c0, coupled));
                            if (noisy) d = __dadd_rn(d, __dmul_rn(p.alpha, eta));
                            yi = __dadd_rn(yi, __dmul_rn(p.dt, d));
                            xi = __dadd_rn(xi, __dmul_rn(p.s_dt_a0, yi));
                            yi = fabs(xi) > 1.0 ? 0.0 : yi;
                        }
                        // cwiseMax(-1).cwiseMin(1) == std::max/std::min (NaN propagates)
                        xi = (xi < -1.0) ? -1.0 : xi;
                        xi = (1.0 < xi) ? 1.0 : xi;
                        x[i] = xi;
                        if constexpr (kYS) ys[i * kSampleBlock + tid] = yi;
                        else y[i] = yi;
                        newmask |= static_cast<uint64_t>(xi < 0.0) << i;
                        if (p.first_bad_step_task >= 0 && first_bad == 0 &&
                            (!isfinite(xi) || !isfinite(yi)))
                            first_bad = t + 1;
                    }
                }
            }
        }
        negmask = newmask;
        if constexpr (kGather) {
#pragma unroll
            for (int i = 0; i < NMAX; ++i)
                if (i < n) xs[i * kSampleBlock + tid] = x[i];
        }
    }

    // ---- read_spins + pack (solver.hpp:237-244, :288-297): bit i set iff !(x_i < 0)
    uint64_t word = 0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
        if (i < n) {
            word |= static_cast<uint64_t>(!(x[i] < 0.0)) << i;
            bad |= x[i] != x[i];
        }
    }
    const long long idx = (static_cast<long long>(run) * p.L + l) * p.batch + traj;
    p.words[idx] = word;
    if (bad) p.nan_block[blockIdx.x] = 1;
    if (p.first_bad_step_task >= 0 && first_bad) atomicMin(&p.bad_step[blockIdx.x], first_bad);
    if (p.block_end_ns && (tid & 31) == 0) atomicMax(&p.block_end_ns[blockIdx.x], globaltimer());
}

template <int NMAX, int VAR>
int launch_small(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    using SL = SmemLayout<NMAX>;
    constexpr bool kGather = VAR != 1;
    constexpr bool kYS = y_in_smem<NMAX>();
    const int smem = SL::csr_of(kGather, kYS) + ((NMAX + 1) * 4 + 15) / 16 * 16 + p.nnz * 12 + 16;
    auto kern = sb_small_kernel<NMAX, VAR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const long long kMaxGrid = 1ll << 30;
    for (long long b0 = 0; b0 < nblocks; b0 += kMaxGrid) {
        SamplerParams q = p;
        q.block_begin = p.block_begin + b0;
        const long long nb = nblocks - b0 < kMaxGrid ? nblocks - b0 : kMaxGrid;
        // per-block outputs are indexed by blockIdx.x: shift them for later slices
        q.nan_block = p.nan_block + b0;
        if (p.block_end_ns) q.block_end_ns = p.block_end_ns + b0;
        if (p.bad_step) q.bad_step = p.bad_step + b0;
        kern<<<static_cast<unsigned>(nb), kSampleBlock, smem, st>>>(q);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int NMAX>
int launch_variant(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    switch (p.variant) {
        case 0: return launch_small<NMAX, 0>(p, nblocks, st);
        case 1: return launch_small<NMAX, 1>(p, nblocks, st);
        default: return launch_small<NMAX, 2>(p, nblocks, st);
    }
}

}  // namespace sbimpl

// explicit instantiation units: sampler_n<NMAX>.cu
int launch_small_n16(const SamplerParams&, long long, cudaStream_t);
int launch_small_n32(const SamplerParams&, long long, cudaStream_t);
int launch_small_n42(const SamplerParams&, long long, cudaStream_t);
int launch_small_n64(const SamplerParams&, long long, cudaStream_t);

}  // namespace momc_b200
