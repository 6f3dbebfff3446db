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
// bit-for-bit; the context reports the path (momc_b200_sampler_path).
//
// Per step, two kernels over the (run, weight) pairs of a group:
//   * k_dense_gemm2: D (trajectories x spins, int32) = Phi . (H J)^T on the tensor cores.
//     Persistent CTA pairs (cta_group::2), warp-specialised: in each CTA one thread streams
//     128-byte K chunks of its 128 trajectories of Phi and its halves of the H*J(c) tiles
//     with TMA into a 4-stage ring, one thread of rank 0 issues tcgen05.mma for the pair
//     (M = 256, two N = 256 products per chunk into all 512 TMEM columns of both CTAs), and
//     eight epilogue warps per CTA move the finished item TMEM -> registers -> swizzled
//     shared memory -> TMA store.
//   * k_dense_warp: the FP64 update, one warp per trajectory, 32 spins per window, the
//     (trajectory, step) noise stream resolved warp-wide (below).
// State: Phi [pair][traj][ldp] (int8 or bf16), D [pair][traj][ldp] int32, x / y
// [pair][traj][n] FP64. A single fused kernel (D kept on chip) was built and measured first:
// 0.27 s for C4 against 0.16 s here; its 15 epilogue warps per SM (registers and the 128 KB
// D tiles bound them) could not keep enough x / y loads in flight.
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

struct PairOf {
    int run, l, traj0, count;
};

// the sign operand: int8 +-1, or bf16 +-1.0 (0x3F80 / 0xBF80)
template <typename PhiT>
__device__ __forceinline__ PhiT phi_of(bool neg);
template <>
__device__ __forceinline__ int8_t phi_of<int8_t>(bool neg) { return neg ? -1 : 1; }
template <>
__device__ __forceinline__ uint16_t phi_of<uint16_t>(bool neg) { return neg ? 0xBF80 : 0x3F80; }

// init_state (solver.hpp:108-124), trajectory-major: one warp per trajectory, lanes over
// spins; spin i takes words 2i, 2i+1 of the init_x / init_y streams (block i/2, half i%2).
// Per 32-spin window lanes 0-15 make the 16 init_x blocks and lanes 16-31 the init_y blocks
// (one Philox block per lane), shuffled to the lanes of their spins; every store of a warp is
// one contiguous run. Padding trajectories get Phi = +1 rows; K padding (H*J zero) too.
template <typename PhiT>
__global__ void __launch_bounds__(256) k_dense_init_t(int n, int ldp, int batch_pad, const PairOf* __restrict__ pairs,
                                                      uint64_t seed, double h, double* x, double* y, PhiT* phi)
{
    const PairOf pr = pairs[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 8 + warp;
    if (t >= batch_pad) return;
    const long long trow = static_cast<long long>(blockIdx.y) * batch_pad + t;
    PhiT* ph = phi + trow * ldp;
    if (t >= pr.count) {
        for (int i = lane; i < ldp; i += 32) ph[i] = phi_of<PhiT>(false);
        return;
    }
    const uint64_t key = run_key(seed, static_cast<uint32_t>(pr.run));
    const uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
    const uint32_t tr = static_cast<uint32_t>(pr.traj0 + t), wl = static_cast<uint32_t>(pr.l);
    const uint32_t tag = tag_word(lane < 16 ? kTagInitX : kTagInitY, 0);
    const int src = lane >> 1;
    const bool odd = lane & 1;
    for (int s0 = 0; s0 < ldp; s0 += 32) {
        const int i = s0 + lane;
        if (s0 >= n) {
            if (i < ldp) ph[i] = phi_of<PhiT>(false);
            continue;
        }
        const uint4 pv = philox(k0, k1, static_cast<uint32_t>(s0 / 2 + (lane & 15)), tag, tr, wl);
        const uint32_t xa = __shfl_sync(0xffffffffu, pv.x, src), xb = __shfl_sync(0xffffffffu, pv.y, src);
        const uint32_t xc = __shfl_sync(0xffffffffu, pv.z, src), xd = __shfl_sync(0xffffffffu, pv.w, src);
        const uint32_t ya = __shfl_sync(0xffffffffu, pv.x, src + 16), yb = __shfl_sync(0xffffffffu, pv.y, src + 16);
        const uint32_t yc = __shfl_sync(0xffffffffu, pv.z, src + 16), yd = __shfl_sync(0xffffffffu, pv.w, src + 16);
        if (i < n) {
            const double xv = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, odd ? u01_from(xc, xd) : u01_from(xa, xb)), 1.0));
            const double yv = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, odd ? u01_from(yc, yd) : u01_from(ya, yb)), 1.0));
            x[trow * n + i] = xv;
            y[trow * n + i] = yv;
            ph[i] = phi_of<PhiT>(xv < 0.0);
        } else if (i < ldp) {
            ph[i] = phi_of<PhiT>(false);
        }
    }
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t zmag32(uint32_t u) { return static_cast<int32_t>(u) < 0 ? 0u - u : u; }

__device__ __noinline__ bool exp_decides(double lhs, double targ) { return lhs < exp(targ); }

// wedge test of the attempt at word u with uniform words (w1, w2) (rng.hpp:178-183): the FP32
// exp brackets the FP64 one within 1e-6 relative on [-6, 0], so outside a +-1e-5 band around
// it the decision is taken in FP32 (lhs rounded to FP32 moves by < 1e-7 relative); the FP64
// exp decides inside the band
// the same decision from FP32 copies of wn / fn (the batch sampler's bracket, sampler_batch.cuh:
// x, -x^2/2 and lhs in FP32 are within ~4e-6 / 5e-7 relative of their FP64 values; a 4e-5 band
// leaves a 10x margin); the FP64 test only inside the band
__device__ __forceinline__ bool wedge_accept32(uint32_t u, uint32_t w1, uint32_t w2, const ZigTables& z,
                                               const float* wnf, const float* fnf)
{
    const uint32_t iz = u & 127u;
    const float xf = __int2float_rn(static_cast<int32_t>(u)) * wnf[iz];
    const float ef = __expf(-0.5f * xf * xf);
    const float uf = __uint2float_rz(w2 >> 8) * 0x1.0p-24f;  // the top 24 bits of u01, exact
    const float lf = __fmaf_rn(uf, fnf[iz - 1] - fnf[iz], fnf[iz]);
    if (lf < ef * (1.0f - 4e-5f)) return true;
    if (lf > ef * (1.0f + 4e-5f)) return false;
    const double xv = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), z.wn[iz]);
    const double lhs = __dadd_rn(z.fn[iz], __dmul_rn(u01_from(w1, w2), __dsub_rn(z.fn[iz - 1], z.fn[iz])));
    return exp_decides(lhs, __dmul_rn(__dmul_rn(-0.5, xv), xv));
}

__device__ __forceinline__ bool wedge_accept(uint32_t u, uint32_t w1, uint32_t w2, const ZigTables& z)
{
    const uint32_t iz = u & 127u;
    const double xv = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), z.wn[iz]);
    const double lhs = __dadd_rn(z.fn[iz], __dmul_rn(u01_from(w1, w2), __dsub_rn(z.fn[iz - 1], z.fn[iz])));
    const double targ = __dmul_rn(__dmul_rn(-0.5, xv), xv);
    const float ef = __expf(static_cast<float>(targ));
    const float lf = static_cast<float>(lhs);
    if (lf < ef * (1.0f - 2e-5f)) return true;
    if (lf > ef * (1.0f + 2e-5f)) return false;
    return exp_decides(lhs, targ);
}

// ---- warp-per-trajectory dSB update. x, y and D are stored
// trajectory-major ([pair][traj][spin]); a warp integrates one trajectory, 32 spins per
// window, lane L taking spin s0 + L, so every x / y / D / phi access of a warp is one
// contiguous run. The (trajectory, step) noise stream (rng.hpp:156-185) is resolved per
// window of 32 normals, warp-wide:
//   * the 32 lanes generate Philox blocks together (block tail/4 + L on lane L) into a
//     256-word ring per warp, 128 words at a time;
//   * round 1: lane L tests the word at head + L (|hz| < kn[iz]); slow words are wedge
//     attempts (3 words), tested in parallel by their lanes; a ballot gives the producing
//     positions (fast words not consumed by an attempt, accepted attempts) and each lane's
//     normal index is the popcount below it; round 2 (words after round 1's last attempt)
//     supplies the normals round 1 fell short of;
//   * windows with a tail attempt, a slow word inside another attempt's words, or a round 2
//     that falls short (about 1 in 10) are walked sequentially by the whole warp.
// The values go through a 32-entry shared buffer to the lanes of their spins.
constexpr int kWRing = 256;  // words per warp

// shared-memory accesses by 32-bit shared-window address (the per-warp rings and value
// buffers: through generic pointers the compiler rebuilt their window base every window)
__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v)
{
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ double ldsf64(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void stsf64(uint32_t a, double v)
{
    asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory");
}
constexpr int kWWarps = 8;   // trajectories (warps) per CTA

struct DensePairArg {
    uint32_t k0, k1;  // run_key(seed, run)
    int l, traj0, count;
    int pad_;
    double c0h;  // c0_l / H, rounded once
};
constexpr int kDensePairsPerLaunch = 256;
// per-launch arguments, passed by value: per-pair values are indexed by blockIdx.y and load
// as per-CTA constants
struct DenseStepArgs {
    int n, batch_pad, t_step, pair0;   // pair0: index of pair[0] in the group's state arrays
    double neg_drift, dt, alpha, sdt;  // -(a0 - a_t) (solver.hpp:70-76), dt, alpha, dt * a0
    const ZigTables* zig;
    const int* D;
    double* x;
    double* y;
    void* phi;
    int* bad;
    int ldp;  // row pitch (elements) of D and Phi; x / y rows are n long
    DensePairArg pair[kDensePairsPerLaunch];
};




// UDT: dt == 1 and dt * a0 == 1, so dt * d and dt a0 * y are exact and skipped. CHECK: record
// the first step with a non-finite y (check_finite, solver.hpp:138-143). Only NaN survives a
// step (an infinite y makes |x| > 1, and the wall and clamp reset both), and NaN is sticky, so
// unchecked steps plus a final-state scan find every failing trajectory; the steps are re-run
// with CHECK only then, for the step index.
template <bool NOISY, bool UDT, typename PhiT, bool CHECK>
__global__ void __launch_bounds__(kWWarps * 32, 6) k_dense_warp(const __grid_constant__ DenseStepArgs a)
{
    __shared__ __align__(16) ZigTables z;
    __shared__ float zwf[128], zff[128];
    // per warp: the word ring, then the 32-entry value buffer at a fixed offset
    struct __align__(16) WarpRing {
        uint32_t words[kWRing];
        double vals[32];
    };
    __shared__ WarpRing rings[kWWarps];
    if constexpr (NOISY) {
        static_assert(sizeof(ZigTables) % 16 == 0, "16-byte copies");
        for (int q = threadIdx.x; q < static_cast<int>(sizeof(ZigTables) / 16); q += blockDim.x)
            reinterpret_cast<uint4*>(&z)[q] = __ldg(reinterpret_cast<const uint4*>(a.zig) + q);
        for (int q = threadIdx.x; q < 128; q += blockDim.x) {
            zwf[q] = static_cast<float>(a.zig->wn[q]);
            zff[q] = static_cast<float>(a.zig->fn[q]);
        }
        __syncthreads();
    }
    const DensePairArg& pr = a.pair[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * kWWarps + warp;
    if (t >= pr.count) return;  // whole warps; no CTA barrier below
    const int n = a.n;
    uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(rings[warp].words));
    // opaque: the compiler would otherwise rebuild it from the generic window at every use (8 %
    // of the kernel's instructions)
    asm volatile("" : "+r"(ring));
    const uint32_t val = ring + 4u * kWRing;
    auto rw = [&](int p) { return lds32(ring + 4u * static_cast<uint32_t>(p & (kWRing - 1))); };
    const uint32_t k0 = pr.k0, k1 = pr.k1, lo = tag_word(kTagStepNoise, static_cast<uint32_t>(a.t_step));
    const uint32_t mid = static_cast<uint32_t>(pr.traj0 + t), hi = static_cast<uint32_t>(pr.l);
    const double c0h = pr.c0h;
    const uint32_t lt = lanemask_lt();
    int head = 0, tail = 0;  // next unread word / words generated (warp-uniform)
    auto gen = [&]() {       // 128 words: block tail/4 + lane on each lane
        const uint4 v = philox(k0, k1, static_cast<uint32_t>(tail >> 2) + static_cast<uint32_t>(lane), lo, mid, hi);
        sts128(ring + 4u * static_cast<uint32_t>((tail + 4 * lane) & (kWRing - 1)), v);
        tail += 128;
        __syncwarp();
    };
    auto word = [&](int p) -> uint32_t {  // any position: the ring, or generated directly (slow path)
        if (p < tail) return rw(p);
        const uint4 v = philox(k0, k1, static_cast<uint32_t>(p >> 2), lo, mid, hi);
        const int c = p & 3;
        return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
    };
    auto is_fast = [&](uint32_t u) { return zmag32(u) < z.kn[u & 127u]; };
    auto fast_val = [&](uint32_t u) { return __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), z.wn[u & 127u]); };

    // element index of (trajectory t, spin 0) in x / y / D / phi (< 2^32 within a group)
    const uint32_t trow = static_cast<uint32_t>(a.pair0 + static_cast<int>(blockIdx.y)) * static_cast<uint32_t>(a.batch_pad) +
                          static_cast<uint32_t>(t);
    const uint32_t row = trow * static_cast<uint32_t>(n);             // x / y
    const uint32_t prow = trow * static_cast<uint32_t>(a.ldp);        // D / Phi
    bool nonfinite = false;
    // resolve the next window: k normals (lane L < k gets normal L in eta)
    auto resolve = [&](int& k, double& eta) {
        k = 32;
        eta = 0.0;
        if constexpr (NOISY) {
            if (tail - head < 96) gen();
            const int H = head;
            const uint32_t u = rw(H + lane);
            const bool slow = !is_fast(u);
            const uint32_t sm = __ballot_sync(0xffffffffu, slow);
            if (sm == 0) {  // 32 fast words: lane L's normal is its own word
                eta = fast_val(u);
                head = H + 32;
                return;
            }
            // every slow word is tested as if an attempt started there (the ones inside another
            // attempt's words are discarded below): wedges take 3 words, tails 1 + 4k and always
            // give a normal (rng.hpp:164-184)
            double v = 0.0;
            bool good = !slow;  // this word gives a normal if it starts an attempt / is free
            int len = 1;
            if (slow) {
                if (u & 127u) {
                    good = wedge_accept32(u, rw(H + lane + 1), rw(H + lane + 2), z,
                                          zwf, zff);
                    len = 3;
                } else {
                    const double r = 3.442619855899;
                    int qq = H + lane + 1;
                    for (;;) {
                        const double xx = __ddiv_rn(-log(u01_open_from(word(qq), word(qq + 1))), r);
                        const double yy = -log(u01_open_from(word(qq + 2), word(qq + 3)));
                        qq += 4;
                        if (__dadd_rn(yy, yy) >= __dmul_rn(xx, xx)) {
                            v = static_cast<int32_t>(u) > 0 ? __dadd_rn(r, xx) : -__dadd_rn(r, xx);
                            break;
                        }
                    }
                    len = qq - (H + lane);
                    good = true;
                }
            }
            if (good && !(slow && (u & 127u) == 0)) v = fast_val(u);
            const uint32_t gm = __ballot_sync(0xffffffffu, good);
            // the attempts, in order: the first slow word starts one, its words are consumed
            uint32_t cons = 0, rem = sm;
            int end = 32;  // first word after the window's last attempt (relative to H)
            while (rem) {
                const int q = __ffs(rem) - 1;
                const int lq = __shfl_sync(0xffffffffu, len, q);
                const uint32_t span = q + lq >= 32 ? ~0u << q : ((1u << lq) - 1u) << q;
                cons |= span & ~(1u << q);
                rem &= ~span;
                end = q + lq > end ? q + lq : end;
            }
            const uint32_t prod = gm & ~cons;  // positions that give this window's normals
            k = __popc(prod);
            head = H + end;
            if ((prod >> lane) & 1u) stsf64(val + 8u * __popc(prod & lt), v);
            __syncwarp();
            eta = ldsf64(val + 8u * lane);
            __syncwarp();  // read before the next window writes
        }
    };
    // software pipeline: the loads of window w are in flight while window w+1's noise is
    // resolved (the noise does not depend on the state)
    int s0 = 0, k;  // first spin / normal count of the current window
    double eta;
    resolve(k, eta);
    while (s0 < n) {
        const bool upd = s0 + lane < n && lane < k;
        const uint32_t e = row + static_cast<uint32_t>(s0 + lane), ep = prow + static_cast<uint32_t>(s0 + lane);
        double xi = 0.0, yi = 0.0;
        int dq = 0;
        if (upd) {
            xi = a.x[e];
            yi = a.y[e];
            dq = a.D[ep];
        }
        int kn = 0;
        double etan = 0.0;
        if (s0 + k < n) resolve(kn, etan);
        asm volatile("" : "+r"(dq)::"memory");  // keep the conversion (a wait on the load) here
        // ---- the update of spin s0 + lane (sb_step solver.hpp:159-181, phi = sgn(x))
        if (upd) {
            double d = __dsub_rn(__dmul_rn(a.neg_drift, xi), __dmul_rn(c0h, static_cast<double>(dq)));
            if constexpr (NOISY) d = __dadd_rn(d, __dmul_rn(a.alpha, eta));
            yi = __dadd_rn(yi, UDT ? d : __dmul_rn(a.dt, d));
            xi = __dadd_rn(xi, UDT ? yi : __dmul_rn(a.sdt, yi));
            {  // wall + clamp (both fire exactly when |x| > 1): one predicate, one LOP3 for +-1
                uint32_t xl = static_cast<uint32_t>(__double2loint(xi)), xh = static_cast<uint32_t>(__double2hiint(xi));
                uint32_t yl = static_cast<uint32_t>(__double2loint(yi)), yh = static_cast<uint32_t>(__double2hiint(yi));
                asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %4, 0d3FF0000000000000;\n\t"
                    "@p lop3.b32 %1, %1, 0x80000000, %5, 0xEA;\n\t@p mov.b32 %0, 0;\n\t"
                    "@p mov.b32 %2, 0;\n\t@p mov.b32 %3, 0;\n\t}"
                    : "+r"(xl), "+r"(xh), "+r"(yl), "+r"(yh)
                    : "d"(fabs(xi)), "r"(0x3FF00000u));
                xi = __hiloint2double(static_cast<int>(xh), static_cast<int>(xl));
                yi = __hiloint2double(static_cast<int>(yh), static_cast<int>(yl));
            }
            // the first step with a non-finite x or y has a non-finite y (x = x + dt a0 y, walls)
            if constexpr (CHECK) nonfinite |= !(fabs(yi) <= 1.7976931348623157e308);
            a.x[e] = xi;
            a.y[e] = yi;
            static_cast<PhiT*>(a.phi)[ep] = phi_of<PhiT>(xi < 0.0);
        }
        s0 += k;
        k = kn;
        eta = etan;
    }
    if constexpr (CHECK)
        if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicMin(a.bad, a.t_step + 1);
}

// ---- D = Phi . (H J)^T on the tensor cores (persistent, warp-specialised) -------------------
constexpr int kGM = 128;              // trajectories per CTA (TMEM lanes)
constexpr int kGH = 2;                // trajectory tiles per item: 256 rows, one per CTA of a pair
constexpr int kGN = 256;              // spins per MMA (N)
constexpr int kGOut = 32 * 32 * 4;    // one epilogue store box: 32 trajectories x 32 spins int32
constexpr int kGEpi = 8;              // epilogue warps: TMEM lane quarter = warp & 3, column half = (warp - 2) / 4
constexpr int kGThreads = (2 + kGEpi) * 32;  // 0: TMA, 1: MMA (+ TMEM), 2..9: epilogue

struct GemmArgs {
    int n, ldp, batch_pad, ntn, nch, tiles_per_pair;  // tiles_per_pair: items of kGH x 128 trajectories
    int pair_begin;           // first pair (of the group's state arrays) of this launch
    long long items;          // pairs x tiles_per_pair x ntn, spin tiles fastest
    const PairOf* pairs;
};

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1), "r"(tc::smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read()
{
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}

// ---- the same product on CTA pairs (cta_group::2): an item is 256 trajectories x 256 kG2NT
// spins; rank r of the pair stages trajectory rows [128 r, 128 r + 128) and, of each 256-spin
// product u, spin rows (of H J) [256 u + 128 r, + 128) of every K chunk; rank 0 issues the
// M = 256, N = 256 MMAs, which read both CTAs' shared memory, and each CTA's TMEM holds its
// 128 rows x 256 kG2NT spins. The operands come from L2 at (256 + 256 kG2NT) bytes per K
// step for 65,536 kG2NT outputs: the kernel is bound by that traffic (tensor pipe 50 % busy,
// L2 at 70 % of its throughput with kG2NT = 1, the same cycles as the single-CTA kernel
// above), so kG2NT = 2 (12 B per output instead of 16) fills the 512 TMEM columns with one
// accumulator; with kG2NT = 1 two accumulators alternate and an item's MMAs overlap the
// previous item's epilogue.
constexpr int kG2M = 128;                          // trajectories per CTA (MMA M = 256 per pair)
constexpr int kG2NT = 2;                           // N = 256 products per item (spins 256 kG2NT)
constexpr int kG2Acc = kG2NT == 1 ? 2 : 1;         // TMEM accumulators (512 columns)
constexpr int kG2Stages = kG2NT == 1 ? 5 : 4;
constexpr int kG2StageA = kG2M * 128;              // bytes: 128 rows x 128 bytes of K
constexpr int kG2StageB = kG2NT * (kGN / 2) * 128;  // this CTA's half of each product's 256 spin rows
constexpr int kG2Stage = kG2StageA + kG2StageB;
constexpr int kG2Smem = kG2Stages * kG2Stage + kGEpi * kGOut + 1024;
static_assert(kG2Smem <= 232448, "shared memory per CTA");

template <bool BF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGThreads, 1)
    k_dense_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmD, const __grid_constant__ GemmArgs a)
{
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[kG2Stages], empty[kG2Stages], d_full[2], d_empty[2];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_rank();
    const long long pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    constexpr int KC = BF16 ? 64 : 128;  // K elements per 128-byte chunk
    if (threadIdx.x == 0) {
        for (int q = 0; q < kG2Stages; ++q) {
            tc::mbar_init(&full[q], 1);   // rank 0's: its expect_tx arrival + both CTAs' bytes
            tc::mbar_init(&empty[q], 1);  // each CTA's: the pair's MMA commit
        }
        for (int q = 0; q < kG2Acc; ++q) {
            tc::mbar_init(&d_full[q], 1);           // each CTA's: the pair's MMA commit
            tc::mbar_init(&d_empty[q], 2 * kGEpi);  // rank 0's: both CTAs' epilogue warps
        }
        tc::fence_mbar_init();
        tc::prefetch_tmap(&tmA);
        tc::prefetch_tmap(&tmB);
        tc::prefetch_tmap(&tmD);
    }
    if (warp == 1) tc::tmem_alloc_2sm<512>(&tslot);
    tc::fence_before();
    tc::cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
    tc::fence_after();
    const uint32_t tbase = tslot;
    if (warp == 0) {
        if (lane == 0) {  // TMA producer (both CTAs): this CTA's half of A and of B
            uint32_t g = 0;
            for (long long it = pair_id; it < a.items; it += npairs) {
                const int j = static_cast<int>(it % a.ntn);
                const long long pt = it / a.ntn;
                const int q = a.pair_begin + static_cast<int>(pt / a.tiles_per_pair), i = static_cast<int>(pt % a.tiles_per_pair);
                const int arow = q * a.batch_pad + i * kGH * kGM + static_cast<int>(rank) * kG2M;
                const int brow = a.pairs[q].l * a.n + j * kGN * kG2NT + static_cast<int>(rank) * (kGN / 2);
                for (int c = 0; c < a.nch; ++c, ++g) {
                    const uint32_t st = g % kG2Stages, ph = (g / kG2Stages) & 1;
                    tc::mbar_wait(&empty[st], ph ^ 1);
                    uint8_t* sa = sm + st * kG2Stage;
                    const uint32_t fb = tc::mapa(tc::smem_u32(&full[st]), 0);
                    if (rank == 0) tc::mbar_expect_tx(&full[st], 2 * kG2Stage);
                    tc::tma_load_2d_2sm(sa, &tmA, c * KC, arow, fb);
#pragma unroll
                    for (int u = 0; u < kG2NT; ++u)
                        tc::tma_load_2d_2sm(sa + kG2StageA + u * (kGN / 2) * 128, &tmB, c * KC, brow + u * kGN, fb);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {  // MMA issuer of the pair
            const uint32_t idesc = BF16 ? tc::idesc_bf16(2 * kG2M, kGN) : tc::idesc_i8(2 * kG2M, kGN);
            uint32_t g = 0, s = 0;
            for (long long it = pair_id; it < a.items; it += npairs, ++s) {
                const uint32_t acc = s % kG2Acc, use = s / kG2Acc;
                tc::mbar_wait(&d_empty[acc], (use & 1) ^ 1);  // both epilogues drained it
                tc::fence_after();
                for (int c = 0; c < a.nch; ++c, ++g) {
                    const uint32_t st = g % kG2Stages, ph = (g / kG2Stages) & 1;
                    tc::mbar_wait(&full[st], ph);
                    tc::fence_after();
                    const uint32_t as = tc::smem_u32(sm + st * kG2Stage), bs = as + kG2StageA;
#pragma unroll
                    for (int u = 0; u < kG2NT; ++u) {
                        const uint32_t dt = tbase + (acc * kG2NT + u) * kGN, bu = bs + u * (kGN / 2) * 128;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (BF16) tc::mma_f16_2sm(dt, tc::smem_desc_sw128(as + 32 * k), tc::smem_desc_sw128(bu + 32 * k), idesc, c > 0 || k > 0);
                            else tc::mma_i8_2sm(dt, tc::smem_desc_sw128(as + 32 * k), tc::smem_desc_sw128(bu + 32 * k), idesc, c > 0 || k > 0);
                        }
                    }
                    tc::commit_2sm(&empty[st], 0x3);
                }
                tc::commit_2sm(&d_full[acc], 0x3);
            }
        }
        __syncwarp();
    } else {
        // epilogue warp (both CTAs): TMEM lane quarter q = 32 of this CTA's 128 trajectories,
        // column half ch; per 32-spin column group TMEM -> registers -> swizzled box -> TMA store
        const int q = warp & 3, ch = (warp - 2) / 4;
        const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
        uint8_t* ob = sm + kG2Stages * kG2Stage + (warp - 2) * kGOut;
        uint32_t s = 0, nst = 0;
        for (long long it = pair_id; it < a.items; it += npairs, ++s) {
            const uint32_t acc = s % kG2Acc, use = s / kG2Acc;
            const int j = static_cast<int>(it % a.ntn);
            const long long pt = it / a.ntn;
            const int qq = a.pair_begin + static_cast<int>(pt / a.tiles_per_pair), i = static_cast<int>(pt % a.tiles_per_pair);
            tc::mbar_wait(&d_full[acc], use & 1);
            tc::fence_after();
            const int row0 = qq * a.batch_pad + i * kGH * kGM + static_cast<int>(rank) * kG2M + q * 32;
#pragma unroll 1
            for (int cc = 0; cc < 4 * kG2NT; ++cc) {
                const int cg = ch * 4 * kG2NT + cc;  // 32-spin column group of the item
                const int col0 = j * kGN * kG2NT + cg * 32;
                if (col0 >= a.n) continue;
                uint32_t v[32];
                tc::tmem_ld32(tbase + lane_addr + acc * kG2NT * kGN + cg * 32, v);
                if (BF16)
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = static_cast<uint32_t>(__float2int_rn(__uint_as_float(v[e])));
                if (lane == 0 && nst >= 1) bulk_wait_read<0>();  // the previous store has read the box
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    *reinterpret_cast<uint4*>(ob + lane * 128 + ((u ^ (lane & 7)) << 4)) =
                        make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) tma_store_2d(&tmD, ob, col0, row0);
                ++nst;
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&d_empty[acc]), 0));
        }
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
    }
    tc::fence_before();
    tc::cluster_sync();  // the peer's MMAs, arrivals and TMEM use are over
    tc::fence_after();
    if (warp == 1) tc::tmem_free_2sm<512>(tbase);
}

__global__ void k_dense_readout(int n, int batch_pad, int batch, int L, const PairOf* __restrict__ pairs,
                                const double* __restrict__ x, uint64_t* words, long long row0, int* nanflag)
{
    const PairOf pr = pairs[blockIdx.y];
    const long long pb = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= pr.count) return;
    const int wpc = (n + 63) / 64;
    const long long idx = (static_cast<long long>(pr.run) * L + pr.l) * batch + pr.traj0 + t;
    const double* xr = x + (pb * batch_pad + t) * n;
    bool bad = false;
    for (int wd = 0; wd < wpc; ++wd) {
        uint64_t word = 0;
        for (int b = 0; b < 64 && wd * 64 + b < n; ++b) {
            const double v = xr[wd * 64 + b];
            word |= static_cast<uint64_t>(!(v < 0.0)) << b;
            bad |= v != v;
        }
        words[(idx - row0) * wpc + wd] = word;
    }
    if (bad) atomicOr(nanflag, 1);
}

// ---- evaluate_cuts on the tensor cores (pareto.hpp:346-359): for layer k,
// h_k(u) = s_u^T W_k s_u and C_k(u) = 0.5 (W_k - 0.5 h_k(u)), exact for integer |w| <= 127.
// One work item = 128 configs (MMA M, TMEM lanes; A = the +-1 spins expanded from the packed
// words into TMEM), walked over the K layers and the spin tiles of 128 (B = the W_k tile by
// TMA); the epilogue thread of config u reads its row of D = S W_k^T (tcgen05.ld) and dots it
// with s_u over the tile's spins. No product ever touches HBM.
constexpr int kEvM = 128;            // configs per work item (MMA M, TMEM lanes)
constexpr int kEvN = 128;            // spins per tile (MMA N)
constexpr int kEvStages = 4;
constexpr int kEvStageB = kEvN * 128;
constexpr uint32_t kEvColA = 256;    // A stages (the +-1 spins, expanded into TMEM) from column 256
constexpr int kEvWarps = 9;  // 0: MMA, 1..4: io (expand A, TMA B), 5..8: epilogue
constexpr int kEvSmem = kEvStages * kEvStageB + 256 * 8 + 1024;

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
    __shared__ uint64_t b_full[kEvStages], b_empty[kEvStages], a_full[kEvStages], a_empty[kEvStages], d_full[2], d_empty[2];
    __shared__ uint32_t tslot;
    uint32_t* lut = reinterpret_cast<uint32_t*>(sm + kEvStages * kEvStageB);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int b = tid; b < 256; b += blockDim.x)
        for (int w = 0; w < 2; ++w) {
            uint32_t v = 0;
            for (int q = 0; q < 4; ++q) v |= ((b >> (4 * w + q)) & 1 ? 0x01u : 0xFFu) << (8 * q);
            lut[b * 2 + w] = v;
        }
    if (tid == 0) {
        for (int q = 0; q < kEvStages; ++q) {
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
    if (warp == 0) tc::tmem_alloc<512>(&tslot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tslot;
    const long long items = (a.U + kEvM - 1) / kEvM;
    const int nt = a.ntiles, nch = a.nchunks;
    auto row_of = [&](long long u) -> long long {
        if (u >= a.U) u = a.U - 1;  // padding rows of the last item: any valid config
        return a.idx ? static_cast<long long>(a.idx[u]) : u;
    };
    if (warp == 0) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_i8(kEvM, kEvN);
            uint32_t g = 0, s = 0;
            for (long long it = blockIdx.x; it < items; it += gridDim.x)
                for (int k = 0; k < a.K; ++k)
                    for (int m = 0; m < nt; ++m, ++s) {
                        const uint32_t buf = s & 1;
                        tc::mbar_wait(&d_empty[buf], ((s >> 1) & 1) ^ 1);
                        tc::fence_after();
                        for (int c = 0; c < nch; ++c, ++g) {
                            const uint32_t st = g % kEvStages, ph = (g / kEvStages) & 1;
                            tc::mbar_wait(&a_full[st], ph);
                            tc::mbar_wait(&b_full[st], ph);
                            tc::fence_after();
                            const uint32_t bs = tc::smem_u32(sm + st * kEvStageB);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                tc::mma_i8_ts(tbase + buf * kEvN, tbase + kEvColA + st * 32 + 8 * kk,
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
            const uint32_t* wr = reinterpret_cast<const uint32_t*>(a.words + row_of(it * kEvM + r) * a.wpc);
            for (int k = 0; k < a.K; ++k)
                for (int m = 0; m < nt; ++m)
                    for (int c = 0; c < nch; ++c, ++g) {
                        const uint32_t st = g % kEvStages, ph = (g / kEvStages) & 1;
                        tc::mbar_wait(&a_empty[st], ph ^ 1);
                        if (q == 0 && lane == 0) {
                            tc::mbar_wait(&b_empty[st], ph ^ 1);
                            tc::mbar_expect_tx(&b_full[st], kEvStageB);
                            tc::tma_load_2d(sm + st * kEvStageB, &tmW, c * 128, k * a.n + m * kEvN, &b_full[st]);
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
                        tc::tmem_st32(tbase + lane_addr + kEvColA + st * 32, v);
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
            const long long u = it * kEvM + r;
            const uint32_t* wr = reinterpret_cast<const uint32_t*>(a.words + row_of(u) * a.wpc);
            for (int k = 0; k < a.K; ++k) {
                long long h = 0;
                for (int m = 0; m < nt; ++m, ++s) {
                    const uint32_t buf = s & 1;
                    tc::mbar_wait(&d_full[buf], (s >> 1) & 1);
                    tc::fence_after();
#pragma unroll 1
                    for (int cg = 0; cg < kEvN / 32; ++cg) {
                        uint32_t v[32];
                        tc::tmem_ld32(tbase + lane_addr + buf * kEvN + cg * 32, v);
                        const int s0 = m * kEvN + cg * 32;
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
    if (warp == 0) tc::tmem_free<512>(tbase);
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

// TMA descriptor of a row-major matrix (rows x cols elements of esize bytes, row pitch
// `pitch` elements, a multiple of 16 bytes): boxes of box_cols x box_rows, 128-byte swizzle
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap make_tmap(const void* base, long long rows, int cols, long long pitch, int esize, int box_cols, int box_rows)
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
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * esize};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                                : CU_TENSOR_MAP_DATA_TYPE_INT32;
    const CUresult r = encode(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) runtime("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

struct DenseScratch {
    DevBuf<uint8_t> hj;     // H*J(c) per weight, [weight][spin][npad], int8 or bf16 bits
    DevBuf<uint8_t> phi;    // [pair][traj][ldp] int8 or bf16
    DevBuf<int> D, flags;   // D [pair][traj][ldp]
    DevBuf<double> x, y;    // [pair][traj][n]
    DevBuf<PairOf> pairs;
    long long hj_inst = -1, hj_weights = -1;  // H*J(c) built for this instance / lattice generation
    int hj_bf16 = 0, hj_npad = 0;
    long long bound_inst = -1, bound_weights = -1, bound = 0;  // cached hj_bound
    DevBuf<uint8_t> wk;     // the K weight layers, dense int8, per instance (evaluate_cuts)
    long long wk_gen = -1;
};

DenseScratch& dscratch(Ctx& c)
{
    if (!c.dense_scratch) c.dense_scratch = std::shared_ptr<void>(new DenseScratch(), [](void* p) {
        auto* d = static_cast<DenseScratch*>(p);
        d->hj.release(); d->phi.release(); d->D.release(); d->flags.release(); d->x.release(); d->y.release();
        d->pairs.release(); d->wk.release();
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

template <typename PhiT, bool CHECK>
void launch_warp(const DenseStepArgs& sa, dim3 grid, cudaStream_t st, bool noisy, bool udt)
{
    if (noisy) udt ? k_dense_warp<true, true, PhiT, CHECK><<<grid, kWWarps * 32, 0, st>>>(sa)
                   : k_dense_warp<true, false, PhiT, CHECK><<<grid, kWWarps * 32, 0, st>>>(sa);
    else udt ? k_dense_warp<false, true, PhiT, CHECK><<<grid, kWWarps * 32, 0, st>>>(sa)
             : k_dense_warp<false, false, PhiT, CHECK><<<grid, kWWarps * 32, 0, st>>>(sa);
}

}  // namespace

// 0: no dense path; 1: int8 (|H*J| <= 127); 2: bf16 (|H*J| <= 256). dSB with integer weights
// and n >= the dense threshold only (bSB's phi = x has no exact narrow operand).
int dense_path_kind(Ctx& c, int variant)
{
    if (variant != 1 || !c.integer_weights || c.n < c.dense_min_n || c.L < 1 || c.H < 1) return 0;
    DenseScratch& d = dscratch(c);
    if (d.bound_inst != c.inst_gen || d.bound_weights != c.weights_gen) {
        d.bound = hj_bound(c);
        d.bound_inst = c.inst_gen;
        d.bound_weights = c.weights_gen;
    }
    return d.bound <= 127 ? 1 : d.bound <= 256 ? 2 : 0;
}
bool dense_path_ok(Ctx& c, int variant) { return dense_path_kind(c, variant) != 0; }
int dense_block_traj() { return kGM; }

// Samples the flattened (run, weight, chunk) blocks [b0, b0+nblocks) of 128 trajectories
// (p.block_traj): per step the tcgen05 GEMM, then the warp-per-trajectory update.
void sample_dense(Ctx& c, const SamplerParams& p, long long b0, long long nblocks)
{
    DenseScratch& d = dscratch(c);
    const int kind = dense_path_kind(c, p.variant);
    if (!kind) runtime("dense path not applicable");
    const bool bf16 = kind == 2;
    const int n = c.n, L = c.L;
    const int esize = bf16 ? 2 : 1;
    const int npad = (n + 15) / 16 * 16;  // row pitch of H*J, Phi and D (16-byte rows for TMA in every type)
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
    // group the block range into (run, weight) pairs of contiguous trajectories
    std::vector<PairOf> pairs;
    const int bt = p.block_traj;
    for (long long b = b0; b < b0 + nblocks; ++b) {
        const int chunk = static_cast<int>(b % p.chunks);
        const long long rl = b / p.chunks;
        const int l = static_cast<int>(rl % L), run = static_cast<int>(rl / L);
        const int first = chunk * bt, cnt = std::min(bt, p.batch - first);
        if (!pairs.empty() && pairs.back().run == run && pairs.back().l == l &&
            pairs.back().traj0 + pairs.back().count == first)
            pairs.back().count += cnt;
        else
            pairs.push_back({run, l, first, cnt});
    }
    if (pairs.empty()) return;
    std::vector<double> c0_host(static_cast<size_t>(L));
    ck(cudaMemcpyAsync(c0_host.data(), p.c0, sizeof(double) * L, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "c0");
    int maxc = 0;
    for (auto& q : pairs) maxc = std::max(maxc, q.count);
    const int batch_pad = (maxc + kGH * kGM - 1) / (kGH * kGM) * (kGH * kGM);  // GEMM items never span two pairs
    int dev = 0, sms = 0;
    ck(cudaGetDevice(&dev), "device");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
    auto gemm = bf16 ? k_dense_gemm2<true> : k_dense_gemm2<false>;
    ck(cudaFuncSetAttribute(gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kG2Smem), "smem attribute");
    // process pairs in groups bounded by memory (~24 GB of state)
    const size_t per_pair = static_cast<size_t>(batch_pad) * (static_cast<size_t>(n) * 16 + static_cast<size_t>(npad) * (4 + esize));
    const size_t group = std::max<size_t>(1, (24ull << 30) / per_pair);
    for (size_t g0 = 0; g0 < pairs.size(); g0 += group) {
        const int G = static_cast<int>(std::min(group, pairs.size() - g0));
        d.pairs.reserve(static_cast<size_t>(G));
        ck(cudaMemcpyAsync(d.pairs.p, pairs.data() + g0, sizeof(PairOf) * G, cudaMemcpyHostToDevice, c.stream), "H2D");
        const size_t rows = static_cast<size_t>(G) * batch_pad;
        d.x.reserve(rows * n);
        d.y.reserve(rows * n);
        d.D.reserve(rows * npad);
        d.phi.reserve(rows * npad * esize);
        d.flags.reserve(4);
        // pass 0 unchecked; pass 1 (only when the final state holds a NaN) re-runs the group with
        // per-step checks for the failing step (test hook MOMC_TEST_DENSE_CHECKED: checked at once)
        static const bool force_checked = std::getenv("MOMC_TEST_DENSE_CHECKED") != nullptr;
        for (int pass = force_checked ? 1 : 0; pass < 2; ++pass) {
            const bool checked = pass == 1;
            ck(cudaMemsetAsync(d.flags.p, 0x7f, sizeof(int), c.stream), "memset");
            ck(cudaMemsetAsync(d.flags.p + 1, 0, sizeof(int), c.stream), "memset");
            const dim3 igrid(static_cast<unsigned>((batch_pad + 7) / 8), static_cast<unsigned>(G));
            if (bf16)
                k_dense_init_t<uint16_t><<<igrid, 256, 0, c.stream>>>(n, npad, batch_pad, d.pairs.p, p.seed, p.init_scale, d.x.p,
                                                                      d.y.p, reinterpret_cast<uint16_t*>(d.phi.p));
            else
                k_dense_init_t<int8_t><<<igrid, 256, 0, c.stream>>>(n, npad, batch_pad, d.pairs.p, p.seed, p.init_scale, d.x.p,
                                                                    d.y.p, reinterpret_cast<int8_t*>(d.phi.p));
            c.launches++;
            const int KC = bf16 ? 64 : 128;
            const CUtensorMap tmA = make_tmap(d.phi.p, static_cast<long long>(rows), npad, npad, esize, KC, kG2M);
            const CUtensorMap tmB = make_tmap(d.hj.p, static_cast<long long>(L) * n, npad, npad, esize, KC, kGN / 2);
            const CUtensorMap tmD = make_tmap(d.D.p, static_cast<long long>(rows), n, npad, 4, 32, 32);
            // One stream: GEMM(t) then update(t) over all pairs of the group. (Two pair halves on
            // two streams did not overlap: the update kernel fills every SM, so a GEMM CTA of the
            // other half never finds the shared memory it needs.)
            GemmArgs g;
            g.n = n;
            g.ldp = npad;
            g.batch_pad = batch_pad;
            g.ntn = (n + kGN * kG2NT - 1) / (kGN * kG2NT);
            g.nch = (npad + KC - 1) / KC;
            g.tiles_per_pair = batch_pad / (kGH * kGM);
            g.pair_begin = 0;
            g.items = static_cast<long long>(G) * g.tiles_per_pair * g.ntn;
            g.pairs = d.pairs.p;
            // 8 KB of launch arguments, per call (contexts may sample from several host threads)
            const auto sa_p = std::make_unique<DenseStepArgs>();
            DenseStepArgs& sa = *sa_p;
            sa.n = n;
            sa.ldp = npad;
            sa.batch_pad = batch_pad;
            sa.dt = p.dt;
            sa.alpha = p.alpha;
            sa.sdt = p.s_dt_a0;
            sa.zig = p.zig;
            sa.D = d.D.p;
            sa.x = d.x.p;
            sa.y = d.y.p;
            sa.phi = d.phi.p;
            sa.bad = d.flags.p;
            const bool udt = p.dt == 1.0 && p.s_dt_a0 == 1.0, noisy = p.alpha > 0.0;
            const cudaStream_t st = c.stream;
            const int ggrid = 2 * static_cast<int>(std::min<long long>(g.items, sms / 2));  // CTA pairs
            for (int t = 0; t < p.T; ++t) {
                const int kg = c.ktimer.begin(st);
                gemm<<<ggrid, kGThreads, kG2Smem, st>>>(tmA, tmB, tmD, g);
                c.ktimer.end(kg, kKDenseGemm, st);
                c.launches++;
                for (int s0 = 0; s0 < G; s0 += kDensePairsPerLaunch) {
                    const int np = std::min(kDensePairsPerLaunch, G - s0);
                    sa.t_step = t;
                    sa.pair0 = s0;
                    sa.neg_drift = -(p.a0 - static_cast<double>(t + 1) / static_cast<double>(p.T));
                    for (int q = 0; q < np; ++q) {
                        const PairOf& pq = pairs[g0 + s0 + q];
                        const uint64_t key = run_key(p.seed, static_cast<uint32_t>(pq.run));
                        sa.pair[q] = {static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32), pq.l, pq.traj0, pq.count, 0,
                                      c0_host[static_cast<size_t>(pq.l)] / static_cast<double>(c.H)};
                    }
                    const dim3 wgrid(static_cast<unsigned>((maxc + kWWarps - 1) / kWWarps), static_cast<unsigned>(np));
                    const int ku = c.ktimer.begin(st);
                    if (bf16) checked ? launch_warp<uint16_t, true>(sa, wgrid, st, noisy, udt)
                                      : launch_warp<uint16_t, false>(sa, wgrid, st, noisy, udt);
                    else checked ? launch_warp<int8_t, true>(sa, wgrid, st, noisy, udt)
                                 : launch_warp<int8_t, false>(sa, wgrid, st, noisy, udt);
                    c.ktimer.end(ku, kKDenseUpdate, st);
                    c.launches++;
                }
            }
            const dim3 rgrid(static_cast<unsigned>((batch_pad + 127) / 128), static_cast<unsigned>(G));
            k_dense_readout<<<rgrid, 128, 0, c.stream>>>(n, batch_pad, p.batch, L, d.pairs.p, d.x.p, p.words, p.row0, d.flags.p + 1);
            c.launches++;
            ck(cudaGetLastError(), "dense sampler");
            int fl[2] = {0, 0};
            ck(cudaMemcpyAsync(fl, d.flags.p, sizeof fl, cudaMemcpyDeviceToHost, c.stream), "D2H");
            ck(cudaStreamSynchronize(c.stream), "dense sampler");
            c.ktimer.collect();
            if (fl[0] != 0x7f7f7f7f)
                runtime("numerical failure at step " + std::to_string(fl[0]) + " (run " + std::to_string(pairs[g0].run) +
                        ", weight " + std::to_string(pairs[g0].l) + ")");
            if (fl[1] == 0) break;  // no trajectory ended non-finite
            if (checked) runtime("numerical failure (non-finite final state)");
        }
    }
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
    d.flags.reserve(8);
    EvalArgs ea{};
    ea.n = n;
    ea.K = K;
    ea.ntiles = (n + kEvN - 1) / kEvN;
    ea.nchunks = (n + 127) / 128;
    ea.wpc = (n + 63) / 64;
    ea.U = U;
    ea.words = d_words;
    ea.idx = d_idx;
    ea.W = weight_totals(c);
    ea.out = d_out;
    const CUtensorMap tm = make_tmap(d.wk.p, static_cast<long long>(K) * n, npad, npad, 1, 128, kEvN);
    int dev = 0, sms = 0;
    ck(cudaGetDevice(&dev), "device");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
    const long long items = (U + kEvM - 1) / kEvM;
    const int grid = static_cast<int>(std::min<long long>(items, sms));
    ck(cudaFuncSetAttribute(k_eval_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kEvSmem), "smem attribute");
    const int ke = c.ktimer.begin(c.stream);
    k_eval_tc<<<grid, kEvWarps * 32, kEvSmem, c.stream>>>(tm, ea);
    c.ktimer.end(ke, kKEvalGemm, c.stream);
    c.launches++;
    ck(cudaGetLastError(), "evaluate_cuts (tensor cores)");
}

}  // namespace momc_b200
