// Dense dSB sampler for large n on the tensor cores (config C4, N=2000) and the GEMM form
// of evaluate_cuts. Restates sb_step (solver.hpp:159-181) with phi = sgn(x) and
// evaluate_cuts (pareto.hpp:346-359).
//
// Exactness. With integer weights, H*J(c) = sum_k num_k w_k is an integer matrix; when
// |H*J| <= 127 it is exact in int8, and sgn(x) is exact in int8, so the contraction
// D = sgn(X)^T (H*J) is computed exactly by the int8 tensor cores with int32 accumulation.
// coupled = D / H is then one correctly rounded FP64 division, where the reference sums
// rounded FP64 products over j (scalarize.hpp:30, solver.hpp:161): the two agree to ~n ulp,
// so trajectories agree within the FP tolerance stated in DESIGN.md (spin words are compared
// against the reference in tests/test_gpu_dense.py), not bit-for-bit.
//
// Layout (one batch per (run, weight) pair), default path:
//   Phi  int8  [pair][traj][spin]   (GEMM B operand, K-major)
//   HJ   int8  [weight][spin][spin] (GEMM A operand; symmetric)
//   D    int32 [pair][traj][spin]   (GEMM output D^T = (H J) Phi^T)
//   x, y f64   [pair][traj][spin]
// The update kernel (k_dense_warp) integrates one trajectory per warp, 32 spins per window:
// every access of a warp is one contiguous run, and the trajectory's sequential noise stream
// (rng.hpp:156-185) is resolved warp-wide per window. The GEMM is cuBLASLt's int8 batched
// matmul (a plain library GEMM). The fused tcgen05 step (MOMC_DENSE_TC=1) keeps x, y
// spin-major ([pair][spin][traj]) and one thread per trajectory.
#include <cublasLt.h>
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

void ckb(cublasStatus_t s, const char* what)
{
    if (s != CUBLAS_STATUS_SUCCESS) runtime(std::string("cuBLASLt error in ") + what + ": " + std::to_string(static_cast<int>(s)));
}

__global__ void k_build_hj(int n, int k, int nnz, int L, const int* __restrict__ nums, const int* __restrict__ rowptr,
                           const int* __restrict__ col, const int* __restrict__ eidx, const int* __restrict__ wi,
                           signed char* hj, int* overflow)
{
    const int l = blockIdx.y;
    const int i = blockIdx.x;
    signed char* row = hj + (static_cast<long long>(l) * n + i) * n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) row[j] = 0;
    __syncthreads();
    for (int e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x) {
        int v = 0;
        for (int q = 0; q < k; ++q) v += nums[l * k + q] * wi[static_cast<long long>(eidx[e]) * k + q];
        if (v > 127 || v < -127) atomicOr(overflow, 1);
        row[col[e]] = static_cast<signed char>(v);
    }
}

struct PairOf {
    int run, l, traj0, count;
};

// init_state (solver.hpp:108-124) for one (run, weight) pair block of trajectories
// x / y element of (pair pb, spin i, trajectory t): spin-major [pair][spin][traj] for the
// per-thread kernels, trajectory-major [pair][traj][spin] for the warp-per-trajectory update
__host__ __device__ __forceinline__ long long xy_at(long long pb, int n, int batch_pad, int i, int t, bool tmajor)
{
    return tmajor ? (pb * batch_pad + t) * n + i : (pb * n + i) * batch_pad + t;
}

__global__ void k_dense_init(int n, int batch_pad, const PairOf* __restrict__ pairs, uint64_t seed, double h,
                             double* x, double* y, signed char* phi, bool tmajor)
{
    const PairOf pr = pairs[blockIdx.y];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const long long pb = blockIdx.y;
    if (t < pr.count) {
        const uint64_t key = run_key(seed, static_cast<uint32_t>(pr.run));
        DevStream sx, sy;
        sx.init(key, pr.l, pr.traj0 + t, tag_word(kTagInitX, 0));
        sy.init(key, pr.l, pr.traj0 + t, tag_word(kTagInitY, 0));
        signed char* ph = phi + (pb * batch_pad + t) * n;
        for (int i = 0; i < n; ++i) {
            const double u = static_cast<double>(sx.next_u64() >> 11) * 0x1.0p-53;
            const double xv = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, u), 1.0));
            x[xy_at(pb, n, batch_pad, i, t, tmajor)] = xv;
            ph[i] = xv < 0.0 ? -1 : 1;
        }
        for (int i = 0; i < n; ++i) {
            const double u = static_cast<double>(sy.next_u64() >> 11) * 0x1.0p-53;
            y[xy_at(pb, n, batch_pad, i, t, tmajor)] = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, u), 1.0));
        }
    } else if (t < batch_pad) {  // padding trajectories: phi = +1 rows (never read back)
        signed char* ph = phi + (pb * batch_pad + t) * n;
        for (int i = 0; i < n; ++i) ph[i] = 1;
    }
}

// Per-thread word ring in shared memory for the (trajectory, step) noise stream
// (rng.hpp:113-121): word w of thread t at ring[(w & 15) * 128 + t] (a warp always hits 32
// banks). Blocks are generated warp-synchronously: before every 4 spins each thread tops its
// ring up to >= 8 words, which in steady state is one Philox block for every thread at the
// same time; only slow attempts that outrun the ring generate on their own (<= 7 + 4 < 16).
struct WordRing {
    uint32_t* r;  // this thread's column
    uint32_t k0, k1, lo, mid, hi, blk;
    int head, tail;
    __device__ __forceinline__ void block()
    {
        const uint4 v = philox(k0, k1, blk++, lo, mid, hi);
        r[((tail + 0) & 15) * 128] = v.x;
        r[((tail + 1) & 15) * 128] = v.y;
        r[((tail + 2) & 15) * 128] = v.z;
        r[((tail + 3) & 15) * 128] = v.w;
        tail += 4;
    }
    __device__ __forceinline__ void ensure(int k)
    {
        while (tail - head < k) block();
    }
    __device__ __forceinline__ uint32_t at(int i) const { return r[((head + i) & 15) * 128]; }
};

// next_normal (rng.hpp:156-185) from the ring: the fast path inline, the rest (wedge and
// tail attempts, ~2.75 % of words) out of line. The slow path takes the ring state by value
// and returns it, so the caller's WordRing stays in registers.
struct RingSlow {
    double v;
    int head, tail;
    uint32_t blk;
};

__device__ __noinline__ RingSlow ring_normal_slow(uint32_t* r, uint32_t k0, uint32_t k1, uint32_t lo, uint32_t mid,
                                                  uint32_t hi, uint32_t blk, int head, int tail,
                                                  const ZigTables* __restrict__ z)
{
    WordRing w{r, k0, k1, lo, mid, hi, blk, head, tail};
    for (;;) {
        w.ensure(1);
        const uint32_t u = w.at(0);
        const int32_t hz = static_cast<int32_t>(u);
        const uint32_t iz = u & 127u;
        const uint32_t mag = hz < 0 ? 0u - u : u;
        if (mag < z->kn[iz]) {
            ++w.head;
            return {__dmul_rn(static_cast<double>(hz), z->wn[iz]), w.head, w.tail, w.blk};
        }
        if (iz == 0) {  // tail: (x, y) trials of 4 words each
            ++w.head;
            const double rr = 3.442619855899;
            for (;;) {
                w.ensure(4);
                const double xx = __ddiv_rn(-log(u01_open_from(w.at(0), w.at(1))), rr);
                const double yy = -log(u01_open_from(w.at(2), w.at(3)));
                w.head += 4;
                if (__dadd_rn(yy, yy) >= __dmul_rn(xx, xx))
                    return {hz > 0 ? __dadd_rn(rr, xx) : -__dadd_rn(rr, xx), w.head, w.tail, w.blk};
            }
        }
        w.ensure(3);
        const double xv = __dmul_rn(static_cast<double>(hz), z->wn[iz]);
        const double u01 = u01_from(w.at(1), w.at(2));
        w.head += 3;
        const double lhs = __dadd_rn(z->fn[iz], __dmul_rn(u01, __dsub_rn(z->fn[iz - 1], z->fn[iz])));
        const double targ = __dmul_rn(__dmul_rn(-0.5, xv), xv);
        // FP32 exp brackets the FP64 one within 1e-6 relative on [-6, 0]; the FP64 exp is
        // only evaluated inside the +-1e-5 band (same decision as rng.hpp:180-183)
        const float ef = __expf(static_cast<float>(targ));
        bool accept;
        if (lhs < static_cast<double>(ef) * (1.0 - 1e-5)) accept = true;
        else if (lhs > static_cast<double>(ef) * (1.0 + 1e-5)) accept = false;
        else accept = lhs < exp(targ);
        if (accept) return {xv, w.head, w.tail, w.blk};
    }
}

__device__ __forceinline__ double ring_normal(WordRing& w, const ZigTables* __restrict__ z)
{
    if (w.tail - w.head >= 1) {
        const uint32_t u = w.at(0);
        const int32_t hz = static_cast<int32_t>(u);
        const uint32_t iz = u & 127u;
        const uint32_t mag = hz < 0 ? 0u - u : u;
        if (mag < z->kn[iz]) {
            ++w.head;
            return __dmul_rn(static_cast<double>(hz), z->wn[iz]);
        }
    }
    const RingSlow r = ring_normal_slow(w.r, w.k0, w.k1, w.lo, w.mid, w.hi, w.blk, w.head, w.tail, z);
    w.head = r.head;
    w.tail = r.tail;
    w.blk = r.blk;
    return r.v;
}

// init_state (solver.hpp:108-124) in the trajectory-major layout: one warp per trajectory,
// lanes over spins; spin i takes words 2i, 2i+1 of the init_x / init_y streams (block i/2,
// half i%2), so every store of a warp is one contiguous run
__global__ void __launch_bounds__(256) k_dense_init_t(int n, int batch_pad, const PairOf* __restrict__ pairs,
                                                      uint64_t seed, double h, double* x, double* y, signed char* phi)
{
    const PairOf pr = pairs[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 8 + warp;
    if (t >= batch_pad) return;
    const long long rowe = (static_cast<long long>(blockIdx.y) * batch_pad + t) * n;
    if (t >= pr.count) {  // padding trajectories: phi = +1 rows (never read back)
        for (int i = lane; i < n; i += 32) phi[rowe + i] = 1;
        return;
    }
    const uint64_t key = run_key(seed, static_cast<uint32_t>(pr.run));
    const uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
    const uint32_t tr = static_cast<uint32_t>(pr.traj0 + t), wl = static_cast<uint32_t>(pr.l);
    for (int i = lane; i < n; i += 32) {
        const uint4 rx = philox(k0, k1, static_cast<uint32_t>(i >> 1), tag_word(kTagInitX, 0), tr, wl);
        const uint4 ry = philox(k0, k1, static_cast<uint32_t>(i >> 1), tag_word(kTagInitY, 0), tr, wl);
        const bool odd = i & 1;
        const double xv = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, odd ? u01_from(rx.z, rx.w) : u01_from(rx.x, rx.y)), 1.0));
        const double yv = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, odd ? u01_from(ry.z, ry.w) : u01_from(ry.x, ry.y)), 1.0));
        x[rowe + i] = xv;
        y[rowe + i] = yv;
        phi[rowe + i] = xv < 0.0 ? -1 : 1;
    }
}

// ---- warp-per-trajectory dSB update (the default dense path). x, y and D are stored
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
    signed char* phi;
    int* bad;
    DensePairArg pair[kDensePairsPerLaunch];
};

__device__ __forceinline__ uint32_t zmag32(uint32_t u) { return static_cast<int32_t>(u) < 0 ? 0u - u : u; }

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
    return lhs < exp(targ);
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// UDT: dt == 1 and dt * a0 == 1, so dt * d and dt a0 * y are exact and skipped
template <bool NOISY, bool UDT>
__global__ void __launch_bounds__(kWWarps * 32, 6) k_dense_warp(const __grid_constant__ DenseStepArgs a)
{
    __shared__ ZigTables z;
    __shared__ __align__(16) uint32_t rings[kWWarps][kWRing];
    __shared__ double vals[kWWarps][32];
    if constexpr (NOISY) {
        for (int q = threadIdx.x; q < static_cast<int>(sizeof(ZigTables) / 4); q += blockDim.x)
            reinterpret_cast<uint32_t*>(&z)[q] = reinterpret_cast<const uint32_t*>(a.zig)[q];
        __syncthreads();
    }
    const DensePairArg& pr = a.pair[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * kWWarps + warp;
    if (t >= pr.count) return;  // whole warps; no CTA barrier below
    const int n = a.n;
    uint32_t* ring = rings[warp];
    double* val = vals[warp];
    const uint32_t k0 = pr.k0, k1 = pr.k1, lo = tag_word(kTagStepNoise, static_cast<uint32_t>(a.t_step));
    const uint32_t mid = static_cast<uint32_t>(pr.traj0 + t), hi = static_cast<uint32_t>(pr.l);
    const uint32_t lt = lanemask_lt();
    int head = 0, tail = 0;  // next unread word / words generated (warp-uniform)
    auto gen = [&]() {       // 128 words: block tail/4 + lane on each lane
        const uint4 v = philox(k0, k1, static_cast<uint32_t>(tail >> 2) + static_cast<uint32_t>(lane), lo, mid, hi);
        *reinterpret_cast<uint4*>(&ring[(tail + 4 * lane) & (kWRing - 1)]) = v;
        tail += 128;
        __syncwarp();
    };
    auto word = [&](int p) -> uint32_t {  // any position: the ring, or generated directly (slow path)
        if (p < tail) return ring[p & (kWRing - 1)];
        const uint4 v = philox(k0, k1, static_cast<uint32_t>(p >> 2), lo, mid, hi);
        const int c = p & 3;
        return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
    };
    auto is_fast = [&](uint32_t u) { return zmag32(u) < z.kn[u & 127u]; };
    auto fast_val = [&](uint32_t u) { return __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), z.wn[u & 127u]); };

    // element index of (trajectory t, spin 0) in x / y / D / phi (< 2^32 within a group)
    const uint32_t row = (static_cast<uint32_t>(a.pair0 + static_cast<int>(blockIdx.y)) * static_cast<uint32_t>(a.batch_pad) +
                          static_cast<uint32_t>(t)) * static_cast<uint32_t>(n);
    bool nonfinite = false;
    // resolve the next window: k normals (lane L < k gets normal L in eta)
    auto resolve = [&](int& k, double& eta) {
        k = 32;
        eta = 0.0;
        if constexpr (NOISY) {
            if (tail - head < 96) gen();
            const int H = head;
            const uint32_t u = ring[(H + lane) & (kWRing - 1)];
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
                    good = wedge_accept(u, ring[(H + lane + 1) & (kWRing - 1)], ring[(H + lane + 2) & (kWRing - 1)], z);
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
            if ((prod >> lane) & 1u) val[__popc(prod & lt)] = v;
            __syncwarp();
            eta = val[lane];
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
        const uint32_t e = row + static_cast<uint32_t>(s0 + lane);
        double xi = 0.0, yi = 0.0;
        int dq = 0;
        if (upd) {
            xi = a.x[e];
            yi = a.y[e];
            dq = a.D[e];
        }
        int kn = 0;
        double etan = 0.0;
        if (s0 + k < n) resolve(kn, etan);
        asm volatile("" : "+r"(dq)::"memory");  // keep the conversion (a wait on the load) here
        // ---- the update of spin s0 + lane (sb_step solver.hpp:159-181, phi = sgn(x))
        if (upd) {
            double d = __dsub_rn(__dmul_rn(a.neg_drift, xi), __dmul_rn(pr.c0h, static_cast<double>(dq)));
            if constexpr (NOISY) d = __dadd_rn(d, __dmul_rn(a.alpha, eta));
            yi = __dadd_rn(yi, UDT ? d : __dmul_rn(a.dt, d));
            xi = __dadd_rn(xi, UDT ? yi : __dmul_rn(a.sdt, yi));
            if (fabs(xi) > 1.0) {  // wall + clamp (both fire exactly when |x| > 1)
                yi = 0.0;
                xi = __hiloint2double((__double2hiint(xi) & static_cast<int>(0x80000000u)) | 0x3FF00000, 0);
            }
            // the first step with a non-finite x or y has a non-finite y (x = x + dt a0 y, walls)
            nonfinite |= !(fabs(yi) <= 1.7976931348623157e308);
            a.x[e] = xi;
            a.y[e] = yi;
            a.phi[e] = xi < 0.0 ? -1 : 1;
        }
        s0 += k;
        k = kn;
        eta = etan;
    }
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicMin(a.bad, a.t_step + 1);
}

// ---- fused tensor-core step (the default dense path): one CTA owns 128 trajectories of
// one (run, weight) pair and walks the output spins in tiles of 128. Per tile, the
// contraction D (128 traj x 128 spins) = Phi_t (128 x n, int8) . (H J)^T (n x 128, int8) runs
// on the tensor cores: thread 0 streams 128-wide K chunks of both operands with TMA
// (128-byte swizzle, two smem stages, mbarrier completion) and issues tcgen05.mma kind::i8
// into a TMEM accumulator; the epilogue thread of trajectory t then reads its row of D
// (tcgen05.ld) and applies the dSB update to the tile's spins in order (the noise stream is
// sequential in the spin index), writing x, y and Phi_{t+1}. D never touches HBM.
constexpr int kTcN = 128;
constexpr int kTcStage = 2 * 128 * tc::kChunkK;  // A + B chunk
constexpr int kTcSmem = 1024 + 2 * kTcStage + 128 * (kTcN + 4) + 16 * 128 * 4 + static_cast<int>(sizeof(ZigTables));

__global__ void __launch_bounds__(128) k_dense_tc_step(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB, int n, int batch_pad,
                                                       int H, const PairOf* __restrict__ pairs, uint64_t seed,
                                                       int t_step, int T, double dt, double a0, double alpha,
                                                       double sdt, const double* __restrict__ c0s,
                                                       const ZigTables* __restrict__ zig, signed char* phi_next,
                                                       double* x, double* y, int* bad)
{
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    __shared__ uint64_t full[2], done[2], tile_done;
    __shared__ uint32_t tslot;
    auto tile = reinterpret_cast<signed char(*)[kTcN + 4]>(sm + 2 * kTcStage);
    uint32_t* ring = reinterpret_cast<uint32_t*>(sm + 2 * kTcStage + 128 * (kTcN + 4));
    ZigTables* z = reinterpret_cast<ZigTables*>(sm + 2 * kTcStage + 128 * (kTcN + 4) + 16 * 128 * 4);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int q = tid; q < static_cast<int>(sizeof(ZigTables) / 4); q += blockDim.x)
        reinterpret_cast<uint32_t*>(z)[q] = reinterpret_cast<const uint32_t*>(zig)[q];
    if (warp == 0) tc::tmem_alloc<128>(&tslot);
    if (tid == 0) {
        tc::prefetch_tmap(&tmA);
        tc::prefetch_tmap(&tmB);
        for (int q = 0; q < 2; ++q) {
            tc::mbar_init(&full[q], 1);
            tc::mbar_init(&done[q], 1);
        }
        tc::mbar_init(&tile_done, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tslot;

    const PairOf pr = pairs[blockIdx.y];
    const long long pb = blockIdx.y;
    const int t0 = blockIdx.x * 128;
    const int t = t0 + tid;
    const bool active = t < pr.count;
    const double c0h = __ddiv_rn(c0s[pr.l], static_cast<double>(H));
    const double a_t = __ddiv_rn(static_cast<double>(t_step + 1), static_cast<double>(T));
    const double neg_drift = -__dsub_rn(a0, a_t);
    const bool noisy = alpha > 0.0;
    WordRing w;
    {
        const uint64_t key = run_key(seed, static_cast<uint32_t>(pr.run));
        w.r = ring + tid;
        w.k0 = static_cast<uint32_t>(key);
        w.k1 = static_cast<uint32_t>(key >> 32);
        w.lo = tag_word(kTagStepNoise, static_cast<uint32_t>(t_step));
        w.mid = static_cast<uint32_t>(pr.traj0 + t);
        w.hi = static_cast<uint32_t>(pr.l);
        w.blk = 0;
        w.head = w.tail = 0;
    }
    double* xs = x + pb * n * static_cast<long long>(batch_pad);
    double* ys = y + pb * n * static_cast<long long>(batch_pad);
    constexpr uint32_t idesc = tc::idesc_i8(128, kTcN);
    const int nk = (n + tc::kChunkK - 1) / tc::kChunkK;
    const int arow = static_cast<int>(pb * batch_pad + t0), brow = pr.l * n;
    // chunk g (global over tiles) uses stage g & 1; its full / done barriers complete their
    // (g >> 1)-th phase
    auto issue_tma = [&](int g, int kc, int nb) {
        const int st = g & 1;
        if (g >= 2) tc::mbar_wait(&done[st], ((g - 2) >> 1) & 1);  // the MMAs that read this stage
        uint8_t* sa = sm + st * kTcStage;
        tc::mbar_expect_tx(&full[st], kTcStage);
        tc::tma_load_2d(sa, &tmA, kc * tc::kChunkK, arow, &full[st]);
        tc::tma_load_2d(sa + 128 * tc::kChunkK, &tmB, kc * tc::kChunkK, brow + nb, &full[st]);
    };
    bool nonfinite = false;
    int g = 0;
    for (int nb = 0; nb < n; nb += kTcN, g += nk) {
        if (tid == 0) {
            issue_tma(g, 0, nb);
            for (int kc = 0; kc < nk; ++kc) {
                if (kc + 1 < nk) issue_tma(g + kc + 1, kc + 1, nb);
                const int gc = g + kc, st = gc & 1;
                tc::mbar_wait(&full[st], (gc >> 1) & 1);
                tc::fence_after();
                const uint32_t a_s = tc::smem_u32(sm + st * kTcStage), b_s = a_s + 128 * tc::kChunkK;
#pragma unroll
                for (int k = 0; k < tc::kChunkK / 32; ++k)
                    tc::mma_i8(tbase, tc::smem_desc_sw128(a_s + 32 * k), tc::smem_desc_sw128(b_s + 32 * k), idesc,
                               kc > 0 || k > 0);
                tc::commit(&done[st]);
            }
            tc::commit(&tile_done);  // completes once per tile: waiters are never a phase behind
        }
        tc::mbar_wait(&tile_done, (nb / kTcN) & 1);
        tc::fence_after();
        // ---- epilogue: trajectory t updates the tile's spins in order, 8 at a time: the 16
        //      x / y loads of a group are issued together (memory parallelism at 8 warps/SM)
        const int lim = min(kTcN, n - nb);
        for (int c0 = 0; c0 < lim; c0 += 8) {
            uint32_t v[8];
            tc::tmem_ld8(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            if (active) {
                double xg[8], yg[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const long long o = static_cast<long long>(nb + c0 + j) * batch_pad + t;
                    xg[j] = c0 + j < lim ? xs[o] : 0.0;
                    yg[j] = c0 + j < lim ? ys[o] : 0.0;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int c = c0 + j;
                    if (c >= lim) break;
                    if (noisy && (c & 3) == 0) {
                        while (w.tail - w.head < 8) w.block();  // warp-synchronous top-up
                    }
                    double xi = xg[j], yi = yg[j];
                    const double eta = noisy ? ring_normal(w, z) : 0.0;
                    double d = __dsub_rn(__dmul_rn(neg_drift, xi),
                                         __dmul_rn(c0h, static_cast<double>(static_cast<int32_t>(v[j]))));
                    if (noisy) d = __dadd_rn(d, __dmul_rn(alpha, eta));
                    yi = __dadd_rn(yi, __dmul_rn(dt, d));
                    xi = __dadd_rn(xi, __dmul_rn(sdt, yi));
                    if (fabs(xi) > 1.0) {  // wall + clamp (both fire exactly when |x| > 1)
                        yi = 0.0;
                        xi = __hiloint2double((__double2hiint(xi) & static_cast<int>(0x80000000u)) | 0x3FF00000, 0);
                    }
                    nonfinite |= !isfinite(xi) || !isfinite(yi);
                    const long long o = static_cast<long long>(nb + c) * batch_pad + t;
                    xs[o] = xi;
                    ys[o] = yi;
                    tile[tid][c] = xi < 0.0 ? -1 : 1;
                }
            } else {
                for (int j = 0; j < 8 && c0 + j < lim; ++j) tile[tid][c0 + j] = 1;  // padding rows stay +1
            }
        }
        tc::fence_before();
        __syncthreads();  // the tile's TMEM reads are done before the next tile's MMAs
        // coalesced store of Phi_{t+1} for the tile: rows of `lim` bytes, 4 bytes per thread and step
        for (int q = tid; q < 128 * (kTcN / 4); q += blockDim.x) {
            const int r = q / (kTcN / 4), c4 = (q % (kTcN / 4)) * 4;
            if (t0 + r < batch_pad && c4 < lim) {
                const uint32_t val = *reinterpret_cast<const uint32_t*>(&tile[r][c4]);
                *reinterpret_cast<uint32_t*>(phi_next + (pb * batch_pad + t0 + r) * n + nb + c4) = val;
            }
        }
        __syncthreads();
        tc::fence_after();
    }
    if (nonfinite) atomicMin(bad, t_step + 1);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<128>(tbase);
}

// TMA descriptor of a row-major int8 matrix (rows x cols, cols % 16 == 0): 128 x 128 boxes,
// 128-byte swizzle, zero fill outside
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap make_tmap_i8(const void* base, long long rows, int cols)
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
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols)};
    const cuuint32_t box[2] = {128, 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) runtime("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

__global__ void k_dense_readout(int n, int batch_pad, int batch, int L, const PairOf* __restrict__ pairs,
                                const double* __restrict__ x, uint64_t* words, long long row0, int* nanflag, bool tmajor)
{
    const PairOf pr = pairs[blockIdx.y];
    const long long pb = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= pr.count) return;
    const int wpc = (n + 63) / 64;
    const long long idx = (static_cast<long long>(pr.run) * L + pr.l) * batch + pr.traj0 + t;
    bool bad = false;
    for (int wd = 0; wd < wpc; ++wd) {
        uint64_t word = 0;
        for (int b = 0; b < 64 && wd * 64 + b < n; ++b) {
            const double v = x[xy_at(pb, n, batch_pad, wd * 64 + b, t, tmajor)];
            word |= static_cast<uint64_t>(!(v < 0.0)) << b;
            bad |= v != v;
        }
        words[(idx - row0) * wpc + wd] = word;
    }
    if (bad) atomicOr(nanflag, 1);
}

// cuBLASLt int8 GEMM with the plan (descriptors + heuristic algorithm) cached per shape:
// the heuristic query costs far more than a 2000x2000x3000 int8 GEMM.
struct LtPlan {
    int m, n, k, batches;
    long long sa, sb, sd;
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t la = nullptr, lb = nullptr, ld = nullptr;
    cublasLtMatmulAlgo_t algo{};
};

struct LtGemm {
    cublasLtHandle_t h = nullptr;
    DevBuf<unsigned char> ws;
    std::vector<LtPlan> plans;
    ~LtGemm()
    {
        for (auto& p : plans) {
            cublasLtMatrixLayoutDestroy(p.la);
            cublasLtMatrixLayoutDestroy(p.lb);
            cublasLtMatrixLayoutDestroy(p.ld);
            cublasLtMatmulDescDestroy(p.op);
        }
        if (h) cublasLtDestroy(h);
        ws.release();
    }
};

constexpr size_t kLtWorkspace = 64ull << 20;

const LtPlan& lt_plan(LtGemm& g, int m, int n, int k, long long sa, long long sb, long long sd, int batches)
{
    for (const auto& p : g.plans)
        if (p.m == m && p.n == n && p.k == k && p.sa == sa && p.sb == sb && p.sd == sd && p.batches == batches) return p;
    if (!g.h) ckb(cublasLtCreate(&g.h), "create");
    g.ws.reserve(kLtWorkspace);
    LtPlan p{m, n, k, batches, sa, sb, sd};
    ckb(cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32I, CUDA_R_32I), "desc");
    const cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
    ckb(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof tA), "transa");
    ckb(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof tB), "transb");
    ckb(cublasLtMatrixLayoutCreate(&p.la, CUDA_R_8I, k, m, k), "la");
    ckb(cublasLtMatrixLayoutCreate(&p.lb, CUDA_R_8I, k, n, k), "lb");
    ckb(cublasLtMatrixLayoutCreate(&p.ld, CUDA_R_32I, m, n, m), "ld");
    for (auto lay_stride : {std::make_pair(p.la, sa), std::make_pair(p.lb, sb), std::make_pair(p.ld, sd)}) {
        ckb(cublasLtMatrixLayoutSetAttribute(lay_stride.first, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batches, sizeof batches),
            "batch");
        long long st = lay_stride.second;
        ckb(cublasLtMatrixLayoutSetAttribute(lay_stride.first, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &st, sizeof st),
            "stride");
    }
    cublasLtMatmulPreference_t pref;
    ckb(cublasLtMatmulPreferenceCreate(&pref), "pref");
    const size_t wsz = kLtWorkspace;
    ckb(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof wsz), "ws");
    cublasLtMatmulHeuristicResult_t res{};
    int found = 0;
    ckb(cublasLtMatmulAlgoGetHeuristic(g.h, p.op, p.la, p.lb, p.ld, p.ld, pref, 1, &res, &found), "heuristic");
    cublasLtMatmulPreferenceDestroy(pref);
    if (!found) runtime("cuBLASLt: no int8 algorithm for this shape");
    p.algo = res.algo;
    g.plans.push_back(p);
    return g.plans.back();
}

// D[b] (m x n, col-major int32) = A[b]^T (A stored k x m col-major int8) x B[b] (k x n int8)
void gemm_i8_batched(Ctx& c, LtGemm& g, int m, int n, int k, const signed char* A, long long strideA,
                     const signed char* B, long long strideB, int* D, long long strideD, int batches)
{
    const LtPlan& p = lt_plan(g, m, n, k, strideA, strideB, strideD, batches);
    const int32_t alpha = 1, beta = 0;
    ckb(cublasLtMatmul(g.h, p.op, &alpha, A, p.la, B, p.lb, &beta, D, p.ld, D, p.ld, &p.algo, g.ws.p, kLtWorkspace,
                       c.stream),
        "matmul");
    c.launches++;
}

struct DenseScratch {
    LtGemm gemm;
    DevBuf<signed char> hj, phi, phi2, s8;
    DevBuf<int> D, flags;
    DevBuf<double> x, y;
    DevBuf<PairOf> pairs;
    long long hj_inst = -1, hj_weights = -1;  // H*J(c) built for this instance / lattice generation
    DevBuf<signed char> wk;  // the K weight layers as dense int8 (evaluate_cuts), per instance
    long long wk_gen = -1;
};

DenseScratch& dscratch(Ctx& c)
{
    if (!c.dense_scratch) c.dense_scratch = std::shared_ptr<void>(new DenseScratch(), [](void* p) {
        auto* d = static_cast<DenseScratch*>(p);
        d->hj.release(); d->phi.release(); d->phi2.release(); d->s8.release(); d->D.release(); d->flags.release(); d->wk.release();
        d->x.release(); d->y.release(); d->pairs.release();
        delete d;
    });
    return *static_cast<DenseScratch*>(c.dense_scratch.get());
}

}  // namespace

// true when the dense int8 tensor path applies (dSB, integer weights, |H*J| <= 127)
bool dense_path_ok(Ctx& c, int variant)
{
    if (variant != 1 || !c.integer_weights || c.n < c.dense_min_n || c.L < 1) return false;
    long long maxabs = 0;
    std::vector<int> nums(static_cast<size_t>(c.L) * c.k);
    ck(cudaMemcpy(nums.data(), c.d_nums.p, sizeof(int) * nums.size(), cudaMemcpyDeviceToHost), "D2H");
    std::vector<double> wmax(static_cast<size_t>(c.k), 0.0);
    for (int e = 0; e < c.m; ++e)
        for (int q = 0; q < c.k; ++q)
            wmax[static_cast<size_t>(q)] = std::max(wmax[static_cast<size_t>(q)], std::fabs(c.h_w[static_cast<size_t>(e) * c.k + q]));
    for (int l = 0; l < c.L; ++l) {
        double s = 0;
        for (int q = 0; q < c.k; ++q) s += nums[static_cast<size_t>(l) * c.k + q] * wmax[static_cast<size_t>(q)];
        maxabs = std::max(maxabs, static_cast<long long>(s));
    }
    return maxabs <= 127 && c.n % 16 == 0;
}

// Samples the flattened (run, weight, chunk) blocks [b0, b0+nblocks) of block_traj
// trajectories with the dense path; returns seconds of device time via events.
void sample_dense(Ctx& c, const SamplerParams& p, long long b0, long long nblocks)
{
    DenseScratch& d = dscratch(c);
    const int n = c.n, L = c.L;
    // H*J(c_l) in int8 (rebuilt when the weights change)
    if (d.hj_inst != c.inst_gen || d.hj_weights != c.weights_gen) {
        d.hj.reserve(static_cast<size_t>(L) * n * n);
        d.flags.reserve(4);
        ck(cudaMemsetAsync(d.flags.p, 0, sizeof(int) * 4, c.stream), "memset");
        k_build_hj<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>(L)), 256, 0, c.stream>>>(
            n, c.k, c.nnz, L, c.d_nums.p, c.d_rowptr.p, c.d_col.p, c.d_eidx.p, c.d_wi.p, d.hj.p, d.flags.p);
        c.launches++;
        int ovf = 0;
        ck(cudaMemcpyAsync(&ovf, d.flags.p, sizeof ovf, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "hj");
        if (ovf) runtime("dense path: H*J(c) exceeds int8");
        d.hj_inst = c.inst_gen;
        d.hj_weights = c.weights_gen;
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
    const int batch_pad = (maxc + 15) / 16 * 16;
    // cuBLASLt's int8 GEMM followed by the update kernel (default), or the fused tcgen05 step
    // (MOMC_DENSE_TC=1): identical words (D is exact). The fused step is correct but its
    // epilogue runs at 8 warps/SM (2 CTAs: TMA stages + TMEM), 2x slower for now.
    const char* tc_env = std::getenv("MOMC_DENSE_TC");
    const bool use_tc = tc_env != nullptr && tc_env[0] == '1';
    // process pairs in groups bounded by memory (~24 GB of state)
    const size_t per_pair = static_cast<size_t>(n) * batch_pad * (8 + 8 + 4 + 1);
    const size_t group = std::max<size_t>(1, (24ull << 30) / per_pair);
    for (size_t g0 = 0; g0 < pairs.size(); g0 += group) {
        const int G = static_cast<int>(std::min(group, pairs.size() - g0));
        d.pairs.reserve(static_cast<size_t>(G));
        ck(cudaMemcpyAsync(d.pairs.p, pairs.data() + g0, sizeof(PairOf) * G, cudaMemcpyHostToDevice, c.stream), "H2D");
        const size_t cells = static_cast<size_t>(G) * n * batch_pad;
        d.x.reserve(cells);
        d.y.reserve(cells);
        if (!use_tc) d.D.reserve(cells);
        d.phi.reserve(cells);
        d.flags.reserve(4);
        ck(cudaMemsetAsync(d.flags.p, 0x7f, sizeof(int), c.stream), "memset");
        ck(cudaMemsetAsync(d.flags.p + 1, 0, sizeof(int), c.stream), "memset");
        const dim3 grid(static_cast<unsigned>((batch_pad + 127) / 128), static_cast<unsigned>(G));
        if (use_tc)
            k_dense_init<<<grid, 128, 0, c.stream>>>(n, batch_pad, d.pairs.p, p.seed, p.init_scale, d.x.p, d.y.p, d.phi.p,
                                                     false);
        else
            k_dense_init_t<<<dim3(static_cast<unsigned>((batch_pad + 7) / 8), static_cast<unsigned>(G)), 256, 0, c.stream>>>(
                n, batch_pad, d.pairs.p, p.seed, p.init_scale, d.x.p, d.y.p, d.phi.p);
        c.launches++;
        // all pairs of a group must share the weight stride pattern: B operand per pair = HJ of its weight
        // -> run one strided-batch GEMM per maximal run of consecutive weights within the group
        if (use_tc) {
            d.phi2.reserve(cells);
            ck(cudaFuncSetAttribute(k_dense_tc_step, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem), "smem");
            const dim3 tgrid(static_cast<unsigned>((batch_pad + 127) / 128), static_cast<unsigned>(G));
            const long long rows = static_cast<long long>(G) * batch_pad;
            const CUtensorMap tm_phi[2] = {make_tmap_i8(d.phi.p, rows, n), make_tmap_i8(d.phi2.p, rows, n)};
            const CUtensorMap tm_hj = make_tmap_i8(d.hj.p, static_cast<long long>(L) * n, n);
            signed char* bufs[2] = {d.phi.p, d.phi2.p};
            for (int t = 0; t < p.T; ++t) {
                k_dense_tc_step<<<tgrid, 128, kTcSmem, c.stream>>>(tm_phi[t & 1], tm_hj, n, batch_pad, c.H, d.pairs.p,
                                                                   p.seed, t, p.T, p.dt, p.a0, p.alpha, p.s_dt_a0, p.c0,
                                                                   p.zig, bufs[(t + 1) & 1], d.x.p, d.y.p, d.flags.p);
                c.launches++;
            }
        } else {
            // D^T per pair = (H J) . Phi^T: m = spins, n = trajectories, so D lands trajectory-major
            // 8 KB of launch arguments, per call (contexts may sample from several host threads)
            const auto step_args_p = std::make_unique<DenseStepArgs>();
            DenseStepArgs& step_args = *step_args_p;
            step_args.n = n;
            step_args.batch_pad = batch_pad;
            step_args.dt = p.dt;
            step_args.alpha = p.alpha;
            step_args.sdt = p.s_dt_a0;
            step_args.zig = p.zig;
            step_args.D = d.D.p;
            step_args.x = d.x.p;
            step_args.y = d.y.p;
            step_args.phi = d.phi.p;
            step_args.bad = d.flags.p;
            for (int t = 0; t < p.T; ++t) {
                int q0 = 0;
                while (q0 < G) {
                    int q1 = q0 + 1;
                    const PairOf& a = pairs[g0 + q0];
                    while (q1 < G && pairs[g0 + q1].l == pairs[g0 + q1 - 1].l + 1 && pairs[g0 + q1].run == a.run) ++q1;
                    const long long pstride = static_cast<long long>(n) * batch_pad;
                    gemm_i8_batched(c, d.gemm, n, batch_pad, n, d.hj.p + static_cast<long long>(a.l) * n * n,
                                    static_cast<long long>(n) * n, d.phi.p + q0 * pstride, pstride, d.D.p + q0 * pstride,
                                    pstride, q1 - q0);
                    q0 = q1;
                }
                for (int s0 = 0; s0 < G; s0 += kDensePairsPerLaunch) {
                    const int np = std::min(kDensePairsPerLaunch, G - s0);
                    step_args.t_step = t;
                    step_args.pair0 = s0;
                    step_args.neg_drift = -(p.a0 - static_cast<double>(t + 1) / static_cast<double>(p.T));
                    for (int q = 0; q < np; ++q) {
                        const PairOf& pq = pairs[g0 + s0 + q];
                        const uint64_t key = run_key(p.seed, static_cast<uint32_t>(pq.run));
                        step_args.pair[q] = {static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32), pq.l, pq.traj0,
                                             pq.count, 0, c0_host[static_cast<size_t>(pq.l)] / static_cast<double>(c.H)};
                    }
                    const dim3 wgrid(static_cast<unsigned>((maxc + kWWarps - 1) / kWWarps), static_cast<unsigned>(np));
                    const bool udt = p.dt == 1.0 && p.s_dt_a0 == 1.0;
                    if (p.alpha > 0.0) {
                        if (udt) k_dense_warp<true, true><<<wgrid, kWWarps * 32, 0, c.stream>>>(step_args);
                        else k_dense_warp<true, false><<<wgrid, kWWarps * 32, 0, c.stream>>>(step_args);
                    } else {
                        if (udt) k_dense_warp<false, true><<<wgrid, kWWarps * 32, 0, c.stream>>>(step_args);
                        else k_dense_warp<false, false><<<wgrid, kWWarps * 32, 0, c.stream>>>(step_args);
                    }
                    c.launches++;
                }
            }
        }
        k_dense_readout<<<grid, 128, 0, c.stream>>>(n, batch_pad, p.batch, L, d.pairs.p, d.x.p, p.words, p.row0,
                                                    d.flags.p + 1, !use_tc);
        c.launches++;
        ck(cudaGetLastError(), "dense sampler");
        int fl[2] = {0, 0};
        ck(cudaMemcpyAsync(fl, d.flags.p, sizeof fl, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "dense sampler");
        if (fl[0] != 0x7f7f7f7f)
            runtime("numerical failure at step " + std::to_string(fl[0]) + " (run " + std::to_string(pairs[g0].run) +
                    ", weight " + std::to_string(pairs[g0].l) + ")");
    }
}

// evaluate_cuts for integer weights |w| <= 127 through int8 GEMMs: for layer k,
// h(u) = s_u^T W_k s_u and C_k(u) = (W_k - h/2)/2, exact (integers).
__global__ void k_unpack_s8(const uint64_t* __restrict__ words, const uint32_t* __restrict__ idx, long long U0,
                            int cnt, int n, int wpc, signed char* s)
{
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < static_cast<long long>(cnt) * n;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int u = static_cast<int>(q / n), i = static_cast<int>(q % n);
        const long long row = idx ? idx[U0 + u] : U0 + u;
        s[q] = (words[row * wpc + (i >> 6)] >> (i & 63)) & 1ull ? 1 : -1;
    }
}

__global__ void k_build_layer(int n, int k, int layer, const int* __restrict__ rowptr, const int* __restrict__ col,
                              const int* __restrict__ eidx, const int* __restrict__ wi, signed char* Wk)
{
    const int i = blockIdx.x;
    signed char* row = Wk + static_cast<long long>(i) * n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) row[j] = 0;
    __syncthreads();
    for (int e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x)
        row[col[e]] = static_cast<signed char>(wi[static_cast<long long>(eidx[e]) * k + layer]);
}

// out[u*K + layer] = 0.5 * (W - 0.5 * sum_i s_u[i] * D[i][u])
// h_u = s_u . (W_k s_u): D[i][u] = (W_k s_u)_i from the GEMM; s_u from the packed words
// (bit i set = +1). A CTA of 256 threads takes 32 configs x 8 slices of the spin range (the
// slices' partial sums meet in shared memory): coalesced D loads, 8x the memory parallelism
// of one thread per config.
__global__ void __launch_bounds__(256) k_cut_from_gemm(const int* __restrict__ D, const uint64_t* __restrict__ words,
                                                       const uint32_t* __restrict__ idx, int cnt, int ld, int n,
                                                       int wpc, int K, int layer, double W, long long U0, double* out)
{
    __shared__ long long part[8][32];
    const int ul = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int u = blockIdx.x * 32 + ul;
    long long h = 0;
    if (u < cnt) {
        const long long row = idx ? idx[U0 + u] : U0 + u;
        const uint64_t* wr = words + row * wpc;
        const int len = (n + 7) / 8;
        const int i0 = sl * len, i1 = min(n, i0 + len);
        uint64_t wv = i0 < i1 ? wr[i0 >> 6] : 0ull;
#pragma unroll 4
        for (int i = i0; i < i1; ++i) {
            if ((i & 63) == 0) wv = wr[i >> 6];
            const int dv = D[static_cast<long long>(i) * ld + u];
            h += ((wv >> (i & 63)) & 1ull) ? dv : -dv;
        }
    }
    part[sl][ul] = h;
    __syncthreads();
    if (sl == 0 && u < cnt) {
        long long t = 0;
        for (int q = 0; q < 8; ++q) t += part[q][ul];
        out[(U0 + u) * K + layer] = 0.5 * (W - 0.5 * static_cast<double>(t));
    }
}

bool eval_gemm_ok(const Ctx& c)
{
    if (!c.integer_weights || c.n < c.dense_min_n || c.n % 16 != 0) return false;
    for (double v : c.h_w)
        if (v > 127 || v < -127) return false;
    return true;
}

void evaluate_cuts_gemm(Ctx& c, const uint64_t* d_words, const uint32_t* d_idx, long long U, double* d_out)
{
    DenseScratch& d = dscratch(c);
    const int n = c.n, K = c.k, wpc = (n + 63) / 64;
    const int chunk = 16384;
    d.s8.reserve(static_cast<size_t>(chunk) * n);
    d.D.reserve(static_cast<size_t>(chunk) * n);
    if (d.wk_gen != c.inst_gen) {  // dense int8 layers, built once per instance
        d.wk.reserve(static_cast<size_t>(K) * n * n);
        for (int layer = 0; layer < K; ++layer) {
            k_build_layer<<<n, 256, 0, c.stream>>>(n, K, layer, c.d_rowptr.p, c.d_col.p, c.d_eidx.p, c.d_wi.p,
                                                   d.wk.p + static_cast<size_t>(layer) * n * n);
            c.launches++;
        }
        d.wk_gen = c.inst_gen;
    }
    std::vector<double> W(static_cast<size_t>(K), 0.0);
    for (int e = 0; e < c.m; ++e)
        for (int q = 0; q < K; ++q) W[static_cast<size_t>(q)] += c.h_w[static_cast<size_t>(e) * K + q];
    for (int layer = 0; layer < K; ++layer) {
        const signed char* Wk = d.wk.p + static_cast<size_t>(layer) * n * n;
        for (long long u0 = 0; u0 < U; u0 += chunk) {
            const int cnt = static_cast<int>(std::min<long long>(chunk, U - u0));
            const int cntp = (cnt + 15) / 16 * 16;
            k_unpack_s8<<<1024, 256, 0, c.stream>>>(d_words, d_idx, u0, cnt, n, wpc, d.s8.p);
            if (cntp > cnt)
                ck(cudaMemsetAsync(d.s8.p + static_cast<size_t>(cnt) * n, 1, static_cast<size_t>(cntp - cnt) * n, c.stream),
                   "memset");
            c.launches++;
            gemm_i8_batched(c, d.gemm, cntp, n, n, d.s8.p, 0, Wk, 0, d.D.p, 0, 1);
            k_cut_from_gemm<<<(cnt + 31) / 32, 256, 0, c.stream>>>(d.D.p, d_words, d_idx, cnt, cntp, n, wpc, K,
                                                                    layer, W[static_cast<size_t>(layer)], u0, d_out);
            c.launches++;
        }
    }
    ck(cudaGetLastError(), "evaluate_cuts_gemm");
}

}  // namespace momc_b200
