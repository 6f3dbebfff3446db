#pragma once
// SB sampler kernel implementation (see sampler.cuh), included by sampler_n*.cu.
//
// Design. A CTA of 256 threads integrates TPC = 256/LANES trajectories
// of one (run, weight). The LANES consecutive lanes of a warp that own a trajectory each
// keep NQ = ceil(NMAX/LANES) of its spins (x, y) in registers, fully unrolled. Splitting a
// trajectory over lanes cuts the per-thread state and the unrolled step loop (which must
// stay inside the 32 KB L1.5 instruction cache; a one-thread-per-trajectory version
// thrashed it) and raises the number of resident warps. Spins past n ("phantoms", when
// LANES*NQ > n) are integrated too: they have no couplings, draw their normals after the
// n real ones, and are masked out of the readout, so no per-spin bound checks are needed.
//
// Per step t the (trajectory, t) noise stream (solver.hpp:128-136) is handled in three
// branch-light phases instead of the reference's sequential next_normal():
//   A1  the lanes generate the Philox blocks of the stream (block b on lane b % LANES)
//       into shared memory and mark, per word, whether a ziggurat attempt starting there
//       takes the fast path (|hz| < kn[iz]) -> 128-bit mask F (OR-reduced over the lanes);
//   A2  every lane walks only the slow attempts (~0.5 per trajectory-step): wedge
//       accept/reject and tail draws exactly as rng.hpp:156-185, producing a short list
//       of "offset changes" / "special values" for the normal indices they affect;
//   B   the unrolled spin update reconstructs normal i as hz*wn[iz] of word i + off(i)
//       (or the special value): every fast normal is independent of the others.
// phi(x_j) (x_j for bSB/SimCIM, sgn(x_j) for dSB) is gathered from the trajectory's
// shared-memory column, rewritten once per step. Rows of J(c_l) are runtime CSR rows
// (DMAX = 0) or rows padded to DMAX entries with exact zeros (DMAX > 0). All FP64
// arithmetic is explicitly rounded (__dmul_rn/__dadd_rn/__dsub_rn) in the reference's
// order: final spins are bit-identical to the shim build of the reference.
// Noise-free runs (alpha = 0) take the sequential path (sampler_generic.cu).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "sampler.cuh"

namespace momc_b200 {

namespace sbimpl {

constexpr int kThreads = 256;

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// |hz| as in rng.hpp:161-163 (INT_MIN -> 2^31)
__device__ __forceinline__ uint32_t zmag(uint32_t u)
{
    return static_cast<int32_t>(u) < 0 ? 0u - u : u;
}

template <int NMAX, int LANES, int VAR>
struct Geo {
    static constexpr int kTPC = kThreads / LANES;           // trajectories per CTA
    static constexpr int kNQ = (NMAX + LANES - 1) / LANES;  // spins per lane
    static constexpr int kNP = kNQ * LANES;                 // integrated spins (>= n)
    static constexpr int kNB = ((kNP + 3) / 4 + 2 + LANES - 1) / LANES * LANES;  // Philox blocks per step
    static constexpr int kNU = 4 * kNB;                     // words covered by the fast mask
    static constexpr int kNA = kNU + 40;                    // allocated words (A2 extends on demand; P(overflow) ~ 1e-15)
    // word rows, trajectory-major, stride == 4 mod 32 words: a block's 4 words are one
    // STS.128, and the 4 lanes x 8 trajectories of a warp reading spin s0 + s hit 32 banks
    static constexpr int kUS = (kNA + 27) / 32 * 32 + 4;
    static constexpr int kECAP = 16;                        // event entries per trajectory-step (P(>16) ~ 1e-14)
    static constexpr int zig = 0;                                           // ZigTables (2560 B)
    static constexpr int ubuf = 2560;                                       // kTPC x kUS u32
    static constexpr int ent = ubuf + kTPC * kUS * 4;                       // kECAP x kTPC u32
    // phi(x_j) rows, trajectory-major: dSB keeps the sign as a u32 mask (J_ij phi_j is J_ij
    // with its sign flipped), bSB / SimCIM keep x as f64. Row strides put the 4 lanes x 8
    // trajectories of a warp on distinct banks for both the writes (spin s0 + s of lane h) and
    // the neighbour gathers (j ~ i +- 1 on a heavy-hex chain): u32 rows == 4 mod 32, f64 rows
    // == 2 mod 16 elements.
    static constexpr int kPhiW = VAR == 1 ? 4 : 8;
    static constexpr int kPStr = VAR == 1 ? (kNP + 27) / 32 * 32 + 4 : (kNP + 13) / 16 * 16 + 2;
    static constexpr int phi = ent + kECAP * kTPC * 4;                      // kTPC x kPStr phi entries
    static constexpr int csr = (phi + kTPC * kPStr * kPhiW + 15) / 16 * 16;
    static_assert(kNU <= 128, "mask covers at most 128 words");
    static_assert(kNA <= 255, "word positions are stored in 8 bits");
    static_assert(kNQ <= 16, "word offsets are packed in 16 fields");
};

// first p in [from, kNU) whose mask bit is clear, else kNU
template <int kNU>
__device__ __forceinline__ int next_slow(uint64_t F0, uint64_t F1, int from)
{
    constexpr uint64_t v0 = kNU >= 64 ? ~0ull : ((1ull << (kNU & 63)) - 1);
    constexpr uint64_t v1 = kNU >= 128 ? ~0ull : (kNU > 64 ? ((1ull << ((kNU - 64) & 63)) - 1) : 0ull);
    if (from < 64) {
        const uint64_t s0 = ~F0 & v0 & (~0ull << from);
        if (s0) return __ffsll(static_cast<long long>(s0)) - 1;
    }
    if (kNU > 64) {
        const int f1 = from > 64 ? from - 64 : 0;
        if (f1 < 64) {
            const uint64_t s1 = ~F1 & v1 & (~0ull << f1);
            if (s1) return 64 + __ffsll(static_cast<long long>(s1)) - 1;
        }
    }
    return kNU;
}

template <int LANES>
constexpr int min_blocks()
{
    return LANES == 4 ? 3 : 2;
}

template <int LANES>
__device__ __forceinline__ uint64_t lane_or(unsigned mask, uint64_t v)
{
#pragma unroll
    for (int o = 1; o < LANES; o <<= 1) v |= __shfl_xor_sync(mask, v, o);
    return v;
}

// Register-resident integrator for n <= NMAX <= 64, LANES lanes per trajectory.
// UDT: dt == 1 and dt * a0 == 1 (the paper's setting): the products dt * d and dt a0 * y are
// exact, so they are skipped (bit-identical, two FP64 operations off each spin's chain)
template <int NMAX, int LANES, int VAR, int DMAX, bool UDT>
__global__ void __launch_bounds__(kThreads, min_blocks<LANES>()) sb_small_kernel(const SamplerParams p)
{
    using G = Geo<NMAX, LANES, VAR>;
    constexpr int TPC = G::kTPC;
    constexpr int NQ = G::kNQ;
    constexpr int NP = G::kNP;
    constexpr int US = G::kUS;
    extern __shared__ __align__(16) unsigned char smem[];
    ZigTables* zig = reinterpret_cast<ZigTables*>(smem + G::zig);
    uint32_t* ubuf = reinterpret_cast<uint32_t*>(smem + G::ubuf);
    uint32_t* ent = reinterpret_cast<uint32_t*>(smem + G::ent);
    unsigned char* phis = smem + G::phi;
    unsigned char* csr = smem + G::csr;
    // DMAX == 0: rp[NP+1] | cv[nnz] | cc[nnz];  DMAX == 3: one 48-byte record per spin,
    // {J_i,j0, J_i,j1 | J_i,j2, off_j0, off_j1 | off_j2, -, -, -} (off = byte offset of phi_j
    // in a trajectory's row), three LDS.128 per spin
    //                DMAX == 3 and dSB (TAB): a 16-byte record {off_j0, off_j1, off_j2, -} per
    // spin, then per spin the 8 values c0 * coupled_i of its 2^3 neighbour sign patterns
    // (table entry f0 + 2 f1 + 4 f2, f_k = 1 iff x_jk < 0), each summed j-ascending from +0.0
    // and multiplied by c0 exactly as the reference does per trajectory (bit-identical)
    int* rp = reinterpret_cast<int*>(csr);
    double* cv = reinterpret_cast<double*>(csr + ((NP + 1) * 4 + 15) / 16 * 16);
    int* cc = reinterpret_cast<int*>(cv + p.nnz);
    static_assert(DMAX == 0 || DMAX == 3, "padded rows are 3 wide");
    constexpr bool TAB = VAR == 1 && DMAX == 3;

    const int n = p.n;
    const long long gblock = p.block_begin + blockIdx.x;
    const int chunk = static_cast<int>(gblock % p.chunks);
    const long long rl = gblock / p.chunks;
    const int l = static_cast<int>(rl % p.L);
    const int run = static_cast<int>(rl / p.L);
    const int tid = threadIdx.x;
    const int t_loc = tid / LANES;  // trajectory within the CTA
    const int h = tid % LANES;      // which quarter/half of the spins this lane owns

    {  // CTA setup: ziggurat tables, coupling rows of J(c_l) (phantom rows: empty / zero)
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.zig);
        uint32_t* dst = reinterpret_cast<uint32_t*>(zig);
        for (int i = tid; i < static_cast<int>(sizeof(ZigTables) / 4); i += kThreads) dst[i] = src[i];
        if constexpr (DMAX == 0) {
            for (int i = tid; i <= NP; i += kThreads) rp[i] = p.row_ptr[i < n ? i : n];
            const double* v = p.vals + static_cast<long long>(l) * p.nnz;
            for (int i = tid; i < p.nnz; i += kThreads) {
                cv[i] = v[i];
                cc[i] = p.col[i];
            }
        } else if constexpr (TAB) {
            const double* v = p.pad_vals + static_cast<long long>(l) * n * DMAX;
            const double c0l = p.c0[l];
            for (int i = tid; i < NP; i += kThreads) {  // phantom rows: zero couplings to themselves
                int* ro = reinterpret_cast<int*>(csr + i * 16);
                for (int d = 0; d < 3; ++d) ro[d] = (i < n ? p.pad_col[i * 3 + d] : i) * G::kPhiW;
                ro[3] = 0;
            }
            double* tab = reinterpret_cast<double*>(csr + NP * 16);
            for (int e = tid; e < NP * 8; e += kThreads) {
                const int i = e >> 3, pat = e & 7;
                double coupled = 0.0;
                for (int d = 0; d < 3; ++d) {
                    const double jv = i < n ? v[i * 3 + d] : 0.0;
                    coupled = __dadd_rn(coupled, (pat >> d) & 1 ? -jv : jv);  // J_ij sgn(x_j): a sign flip
                }
                tab[e] = __dmul_rn(c0l, coupled);
            }
        } else {
            const double* v = p.pad_vals + static_cast<long long>(l) * n * DMAX;
            for (int i = tid; i < NP; i += kThreads) {  // phantom rows: zero couplings to themselves
                double* rv = reinterpret_cast<double*>(csr + i * 48);
                int* ro = reinterpret_cast<int*>(csr + i * 48 + 24);
                for (int d = 0; d < 3; ++d) {
                    rv[d] = i < n ? v[i * 3 + d] : 0.0;
                    ro[d] = (i < n ? p.pad_col[i * 3 + d] : i) * G::kPhiW;
                }
                ro[3] = 0;
            }
        }
    }
    __syncthreads();

    const int traj = chunk * TPC + t_loc;
    const unsigned wmask = __ballot_sync(0xffffffffu, traj < p.batch);  // trajectories never split
    if (traj >= p.batch) return;  // no CTA-wide barrier below this point

    const uint64_t key = run_key(p.seed, static_cast<uint32_t>(run));
    const uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
    const uint32_t wl = static_cast<uint32_t>(l), tr = static_cast<uint32_t>(traj);
    const double c0 = p.c0[l];
    const double alpha = p.alpha, dt = p.dt, sdt = p.s_dt_a0;
    const int s0 = h * NQ;  // first spin of this lane

    // ---- init_state (solver.hpp:108-124): spin i uses words 2i, 2i+1 of the init_x /
    //      init_y streams (block i/2, half i%2)
    //      Block c = s0/2 + c' serves slots 2c'-1 .. 2c'+1 depending on the parity of s0, so
    //      each block is generated once (NQ/2 + 1 per stream instead of NQ).
    double x[NQ];
    double y[NQ];
    {
        const bool par = s0 & 1;  // odd first spin: slot s takes block (s + 1) / 2
        const uint32_t bx = static_cast<uint32_t>(s0 >> 1);
        const uint32_t tx = tag_word(kTagInitX, 0), ty = tag_word(kTagInitY, 0);
        auto init_val = [&](uint32_t lo, uint32_t hi) {
            return __dmul_rn(p.init_scale, __dsub_rn(__dmul_rn(2.0, u01_from(lo, hi)), 1.0));
        };
        uint4 px = philox(k0, k1, bx, tx, tr, wl), py = philox(k0, k1, bx, ty, tr, wl);
        x[0] = init_val(par ? px.z : px.x, par ? px.w : px.y);
        y[0] = init_val(par ? py.z : py.x, par ? py.w : py.y);
#pragma unroll
        for (int c = 1; c <= NQ / 2; ++c) {
            const uint4 cx = philox(k0, k1, bx + c, tx, tr, wl), cy = philox(k0, k1, bx + c, ty, tr, wl);
            if (2 * c - 1 < NQ) {  // slot 2c-1: the previous block's high half, or this block's low half
                x[2 * c - 1] = init_val(par ? cx.x : px.z, par ? cx.y : px.w);
                y[2 * c - 1] = init_val(par ? cy.x : py.z, par ? cy.y : py.w);
            }
            if (2 * c < NQ) {  // slot 2c: this block's low half, or its high half
                x[2 * c] = init_val(par ? cx.z : cx.x, par ? cx.w : cx.y);
                y[2 * c] = init_val(par ? cy.z : cy.x, par ? cy.w : cy.y);
            }
            px = cx;
            py = cy;
        }
    }

    unsigned char* phb = phis + t_loc * G::kPStr * G::kPhiW;  // this trajectory's phi row
    // dSB: phi = (x < 0 ? -1 : +1) (solver.hpp:161-165) kept as the sign mask of the product
    auto put_phi = [&](int j, double xv) {
        if constexpr (TAB) reinterpret_cast<uint32_t*>(phb)[j] = xv < 0.0 ? 8u : 0u;  // table byte step
        else if constexpr (VAR == 1) reinterpret_cast<uint32_t*>(phb)[j] = xv < 0.0 ? 0x80000000u : 0u;
        else reinterpret_cast<double*>(phb)[j] = xv;
    };
    // J_ij * phi_j for the phi entry at byte offset o: exact (a sign flip for dSB)
    auto term = [&](double jv, int o) -> double {
        if constexpr (VAR == 1)
            return __longlong_as_double(__double_as_longlong(jv) ^
                                        (static_cast<long long>(*reinterpret_cast<const uint32_t*>(phb + o)) << 32));
        else return __dmul_rn(jv, *reinterpret_cast<const double*>(phb + o));
    };
#pragma unroll
    for (int s = 0; s < NQ; ++s) put_phi(s0 + s, x[s]);

    const uint32_t* kn = zig->kn;
    const double* wn = zig->wn;
    const double* fn = zig->fn;
    uint32_t* ub = ubuf + t_loc * US;  // this trajectory's word row
    uint32_t* en = ent + t_loc;   // this trajectory's event column, stride TPC
    const uint4* recs = reinterpret_cast<const uint4*>(csr) + s0 * (TAB ? 1 : 3);  // this lane's coupling records
    const unsigned char* tabl = csr + NP * 16 + s0 * 64;  // TAB: this lane's c0 * coupled tables
    bool overflow = false;
    int ovf_code = 0;  // which buffer overflowed (diagnostics)
    __syncwarp(wmask);

    for (int t = 0; t < p.T; ++t) {
        // -(a0 - a_t) and simcim's -0.5 (1 - a_t), a_t = (t + 1) / T (solver.hpp:70-76),
        // tabulated on the host with the same IEEE operations
        const double neg_drift = p.sched[2 * t];
        const double pump = p.sched[2 * t + 1];
        const uint32_t lo = tag_word(kTagStepNoise, static_cast<uint32_t>(t));

        // ---- A1: Philox blocks (lane h: blocks h, h+LANES, ...) + fast-attempt mask
        uint64_t F0 = 0, F1 = 0;
#pragma unroll 4
        for (int b = h; b < G::kNB; b += LANES) {
            const uint4 r = philox(k0, k1, static_cast<uint32_t>(b), lo, tr, wl);
            *reinterpret_cast<uint4*>(ub + 4 * b) = r;
            const uint64_t f = static_cast<uint64_t>(zmag(r.x) < kn[r.x & 127u]) |
                               static_cast<uint64_t>(zmag(r.y) < kn[r.y & 127u]) << 1 |
                               static_cast<uint64_t>(zmag(r.z) < kn[r.z & 127u]) << 2 |
                               static_cast<uint64_t>(zmag(r.w) < kn[r.w & 127u]) << 3;
            const int pp = 4 * b;
            if (pp < 64) F0 |= f << pp;
            else F1 |= f << (pp - 64);
        }
        F0 = lane_or<LANES>(wmask, F0);
        F1 = lane_or<LANES>(wmask, F1);
        __syncwarp(wmask);  // the other lanes' words are visible

        // ---- A2w: the slow attempts' positions (rng.hpp:164-184), identically on every lane.
        //      A wedge attempt takes 3 words whatever its outcome and a tail 1 + 4k, so the
        //      positions follow from the fast mask alone; candidates are listed until even
        //      all-rejected wedges would have produced n normals before them. Tails (rare)
        //      are resolved here; entry = q | tail length << 8 | tail flag << 16.
        int m = 0;
        {
            int gen = G::kNU;  // words present in ub
            int pos = 0;       // next attempt position
            int slow = 0;      // words taken by the listed slow attempts
            // fast walk: wedges whose words lie inside the mask (the common case); anything
            // else (a tail, words beyond the mask, a full list) continues in the general walk
            bool general = false;
            if constexpr (G::kNU <= 64) {
                // the remaining slow words as one mask, consumed from the bottom
                uint64_t rem = ~F0 & (G::kNU >= 64 ? ~0ull : ((1ull << (G::kNU & 63)) - 1));
                for (;;) {
                    const int lastq = n - 1 + slow;
                    const uint32_t rlo = static_cast<uint32_t>(rem), rhi = static_cast<uint32_t>(rem >> 32);
                    const int q = rlo ? __ffs(rlo) - 1 : (rhi ? 31 + __ffs(rhi) : G::kNU);  // kNU when none is left
                    if (q > lastq) break;
                    if (q + 2 >= G::kNU || m >= G::kECAP || (ub[q] & 127u) == 0) {
                        general = true;
                        break;
                    }
                    en[m * TPC] = static_cast<uint32_t>(q);
                    ++m;
                    slow += 3;
                    pos = q + 3;
                    rem = pos >= 64 ? 0ull : rem & (~0ull << pos);  // pos <= kNU here (q + 2 < kNU)
                }
            } else {
                for (;;) {
                    const int lastq = n - 1 + slow;
                    const int q = next_slow<G::kNU>(F0, F1, pos);  // kNU when none is left
                    if (q > lastq) break;
                    if (q + 2 >= G::kNU || m >= G::kECAP || (ub[q] & 127u) == 0) {
                        general = true;
                        break;
                    }
                    en[m * TPC] = static_cast<uint32_t>(q);
                    ++m;
                    slow += 3;
                    pos = q + 3;
                }
            }
            for (; general;) {
                const int lastq = n - 1 + slow;  // fast normals before q = q - slow must stay < n
                int q = next_slow<G::kNU>(F0, F1, pos);
                if (q >= G::kNU) {  // beyond the mask: extend the word buffer, test on demand
                    q = pos > G::kNU ? pos : G::kNU;
                    for (; q <= lastq; ++q) {
                        if (q >= G::kNA) break;
                        while (gen <= q) {  // every lane writes the same words
                            const uint4 r = philox(k0, k1, static_cast<uint32_t>(gen >> 2), lo, tr, wl);
                            *reinterpret_cast<uint4*>(ub + gen) = r;
                            gen += 4;
                        }
                        const uint32_t w = ub[q];
                        if (!(zmag(w) < kn[w & 127u])) break;
                    }
                }
                if (q > lastq) break;
                if (m >= G::kECAP || q + 9 >= G::kNA) {
                    overflow = true;
                    ovf_code |= 4;
                    break;
                }
                while (gen <= q + 8) {  // words a wedge attempt may read
                    const uint4 r = philox(k0, k1, static_cast<uint32_t>(gen >> 2), lo, tr, wl);
                    *reinterpret_cast<uint4*>(ub + gen) = r;
                    gen += 4;
                }
                const uint32_t u = ub[q];
                if ((u & 127u) == 0) {  // tail: 4 words per (x, y) trial
                    const double r = 3.442619855899;
                    int qq = q + 1;
                    double sval = 0.0;
                    for (;;) {
                        if (qq + 4 > G::kNA) {
                            overflow = true;
                            ovf_code |= 8;
                            break;
                        }
                        while (gen < qq + 4) {
                            const uint4 rr = philox(k0, k1, static_cast<uint32_t>(gen >> 2), lo, tr, wl);
                            *reinterpret_cast<uint4*>(ub + gen) = rr;
                            gen += 4;
                        }
                        const double xx = __ddiv_rn(-log(u01_open_from(ub[qq], ub[qq + 1])), r);
                        const double yy = -log(u01_open_from(ub[qq + 2], ub[qq + 3]));
                        qq += 4;
                        if (__dadd_rn(yy, yy) >= __dmul_rn(xx, xx)) {
                            sval = static_cast<int32_t>(u) > 0 ? __dadd_rn(r, xx) : -__dadd_rn(r, xx);
                            break;
                        }
                    }
                    if (overflow) break;
                    en[m * TPC] = static_cast<uint32_t>(q) | (static_cast<uint32_t>(qq - q) << 8) | (1u << 16);
                    // the tail's value goes into its last two words (read by the normal's spin in B:
                    // lo at the normal's word, hi just before it; no other attempt reads them)
                    ub[qq - 1] = static_cast<uint32_t>(__double2loint(sval));
                    ub[qq - 2] = static_cast<uint32_t>(__double2hiint(sval));
                    slow += qq - q;
                    pos = qq;
                } else {
                    en[m * TPC] = static_cast<uint32_t>(q);
                    slow += 3;
                    pos = q + 3;
                }
                ++m;
            }
        }
        __syncwarp(wmask);  // candidate list and extension words visible

        // ---- A2t: the wedge tests, candidate j on lane j % LANES; accept iff
        //      fn[iz] + u01 (fn[iz-1] - fn[iz]) < exp(-x^2 / 2) (tails always give a normal)
        uint32_t acc = 0;
        for (int j = h; j < m; j += LANES) {
            const uint32_t e = en[j * TPC];
            if (e >> 16) {
                acc |= 1u << j;
                continue;
            }
            const int q = static_cast<int>(e & 0xFFu);
            const uint32_t u = ub[q];
            const uint32_t iz = u & 127u;
            const double xv = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), wn[iz]);
            const double lhs = __dadd_rn(
                fn[iz], __dmul_rn(u01_from(ub[q + 1], ub[q + 2]), __dsub_rn(fn[iz - 1], fn[iz])));
            const double targ = __dmul_rn(__dmul_rn(-0.5, xv), xv);
            // FP32 exp brackets the FP64 one within 1e-6 relative on [-6, 0]; decide from it
            // unless lhs falls in the +-1e-5 band, then use the FP64 exp
            const float ef = __expf(static_cast<float>(targ));
            bool accept;
            if (lhs < static_cast<double>(ef) * (1.0 - 1e-5)) accept = true;
            else if (lhs > static_cast<double>(ef) * (1.0 + 1e-5)) accept = false;
            else accept = lhs < exp(targ);
            acc |= static_cast<uint32_t>(accept) << j;
        }
        acc = static_cast<uint32_t>(lane_or<LANES>(wmask, acc));

        // ---- A2e: walk the candidates with their outcomes; every lane keeps the word offset
        //      of each of its spins as a byte offset (4 x word offset) in 8-bit fields of four
        //      words (spins 0..3, 4..7, 8..11, 12..15: one byte-permute extracts a field in B),
        //      and a mask of its tail normals (their value already sits in the tail's last two
        //      words). Offsets only grow along the stream, so each attempt adds its increase to
        //      the fields from its normal on (bytes never carry: offsets stay <= 63).
        uint32_t W0 = 0, W1 = 0, W2 = 0, W3 = 0;
        uint32_t specm = 0;
        {
            // fields from bit b on (b <= 0: all of them, >= 32: none): the funnel shift clamps
            // its count to 32
            auto from = [](int b) -> uint32_t { return __funnelshift_lc(0u, ~0u, static_cast<uint32_t>(max(b, 0))); };
            int pos = 0, i = 0, cur = 0;  // cur: the word offset of the next fast normal
#pragma unroll 2
            for (int j = 0; j < m; ++j) {
                const uint32_t e = en[j * TPC];
                const int q = static_cast<int>(e & 0xFFu);
                i += q - pos;  // fast normals before the attempt
                if (i >= n) break;  // phantom spins (>= n) read any word: no couplings
                const bool tail = e >> 16;
                const int new_pos = tail ? q + static_cast<int>((e >> 8) & 0xFFu) : q + 3;
                const int new_i = tail ? i + 1 : i + static_cast<int>((acc >> j) & 1u);
                const int idx = tail ? i : new_i;  // from this normal on, words sit at +off
                const int off = new_pos - new_i;
                const int jl = idx - s0;
                if (jl < NQ) {
                    if (off > 63) {
                        overflow = true;
                        ovf_code |= 16;
                    }
                    const uint32_t rep = static_cast<uint32_t>(off - cur) * 0x04040404u;
                    const int bb = 8 * jl;
                    W0 += rep & from(bb);
                    if constexpr (NQ > 4) W1 += rep & from(bb - 32);
                    if constexpr (NQ > 8) W2 += rep & from(bb - 64);
                    if constexpr (NQ > 12) W3 += rep & from(bb - 96);
                    if (tail && jl >= 0) specm |= 1u << jl;
                }
                cur = off;
                pos = new_pos;
                i = new_i;
                if (i >= n) break;
            }
        }

        // ---- B: spin updates (sb_step solver.hpp:159-181 / simcim_step :196-210)
        const uint32_t* ubs = ub + s0;
#pragma unroll
        for (int s = 0; s < NQ; ++s) {
            const uint32_t Wq = s < 4 ? W0 : s < 8 ? W1 : s < 12 ? W2 : W3;
            const uint32_t boff = __byte_perm(Wq, 0u, 0x4440u + static_cast<uint32_t>(s & 3));
            const uint32_t* wp = reinterpret_cast<const uint32_t*>(reinterpret_cast<const unsigned char*>(ubs + s) + boff);
            const uint32_t u = wp[0];
            double eta = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), wn[u & 127u]);
            if (specm & (1u << s)) eta = __hiloint2double(static_cast<int>(wp[-1]), static_cast<int>(u));
            // coupled_i = sum_j J_ij phi(x_j), j ascending, from +0.0 (shim GEMM order)
            double coupled = 0.0;
            double c0c = 0.0;  // TAB: c0 * coupled_i from the sign-pattern table
            if constexpr (TAB) {
                const uint4 rc = recs[s];
                const uint32_t f0 = *reinterpret_cast<const uint32_t*>(phb + rc.x);
                const uint32_t f1 = *reinterpret_cast<const uint32_t*>(phb + rc.y);
                const uint32_t f2 = *reinterpret_cast<const uint32_t*>(phb + rc.z);
                c0c = *reinterpret_cast<const double*>(tabl + s * 64 + (f0 + 2 * f1 + 4 * f2));
            } else if constexpr (DMAX > 0) {
                const uint4 r0 = recs[3 * s], r1 = recs[3 * s + 1], r2 = recs[3 * s + 2];
                coupled = __dadd_rn(coupled, term(__hiloint2double(r0.y, r0.x), static_cast<int>(r1.z)));
                coupled = __dadd_rn(coupled, term(__hiloint2double(r0.w, r0.z), static_cast<int>(r1.w)));
                coupled = __dadd_rn(coupled, term(__hiloint2double(r1.y, r1.x), static_cast<int>(r2.x)));
            } else {
                const int i = s0 + s;
                const int e1 = rp[i + 1];
                for (int q = rp[i]; q < e1; ++q) coupled = __dadd_rn(coupled, term(cv[q], cc[q] * G::kPhiW));
            }
            double xi = x[s], yi = y[s];
            if constexpr (VAR == 2) {
                const double d = __dadd_rn(__dsub_rn(__dmul_rn(pump, xi), __dmul_rn(c0, coupled)), __dmul_rn(alpha, eta));
                yi = __dadd_rn(__dmul_rn(0.9, yi), __dmul_rn(1.0 - 0.9, d));
                xi = __dadd_rn(xi, UDT ? yi : __dmul_rn(dt, yi));
            } else {
                if constexpr (!TAB) c0c = __dmul_rn(c0, coupled);
                const double d = __dadd_rn(__dsub_rn(__dmul_rn(neg_drift, xi), c0c), __dmul_rn(alpha, eta));
                yi = __dadd_rn(yi, UDT ? d : __dmul_rn(dt, d));
                xi = __dadd_rn(xi, UDT ? yi : __dmul_rn(sdt, yi));
            }
            // y <- 0 where |x| > 1 (strict, SB only), then cwiseMax(-1).cwiseMin(1): both fire
            // exactly when |x| > 1 (never for NaN, which propagates), and the clamp is +-1
            // with x's sign
            if (fabs(xi) > 1.0) {
                if constexpr (VAR != 2) yi = 0.0;
                xi = __hiloint2double((__double2hiint(xi) & static_cast<int>(0x80000000u)) | 0x3FF00000, 0);
            }
            x[s] = xi;
            y[s] = yi;
        }
        __syncwarp(wmask);  // every lane has finished reading phi(t) and this step's words
#pragma unroll
        for (int s = 0; s < NQ; ++s) put_phi(s0 + s, x[s]);
        __syncwarp(wmask);  // phi(t+1) complete
    }

    // ---- read_spins + pack (solver.hpp:237-244, :288-297): bit i set iff !(x_i < 0)
    uint64_t word = 0;
    bool bad = false;
#pragma unroll
    for (int s = 0; s < NQ; ++s) {
        const int i = s0 + s;
        if (i < n) {
            word |= static_cast<uint64_t>(!(x[s] < 0.0)) << i;
            bad |= !isfinite(x[s]) || !isfinite(y[s]);  // check_finite (solver.hpp:138-143)
        }
    }
    word = lane_or<LANES>(wmask, word);
    if (h == 0) {
        const long long idx = (static_cast<long long>(run) * p.L + l) * p.batch + traj;
        p.words[idx - p.row0] = word;
    }
    // NaN (numerical failure) -> bit 1; noise-event buffer overflow (re-run on the exact
    // sequential path) -> bit 2
    if (bad) atomicOr(&p.nan_block[blockIdx.x], 1);
    if (overflow) atomicOr(&p.nan_block[blockIdx.x], 2 | ovf_code);
    if (p.block_end_ns && (tid & 31) == 0) atomicMax(&p.block_end_ns[blockIdx.x], globaltimer());
}

template <int NMAX, int LANES, int VAR, int DMAX, bool UDT>
int launch_small_u(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    using G = Geo<NMAX, LANES, VAR>;
    const int csr_bytes = DMAX == 0 ? ((G::kNP + 1) * 4 + 15) / 16 * 16 + p.nnz * 12
                          : (VAR == 1 ? G::kNP * (16 + 64) : G::kNP * 48);
    const int smem = G::csr + csr_bytes + 16;
    auto kern = sb_small_kernel<NMAX, LANES, VAR, DMAX, UDT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const long long kMaxGrid = 1ll << 30;
    for (long long b0 = 0; b0 < nblocks; b0 += kMaxGrid) {
        SamplerParams q = p;
        q.block_begin = p.block_begin + b0;
        const long long nb = nblocks - b0 < kMaxGrid ? nblocks - b0 : kMaxGrid;
        q.nan_block = p.nan_block + b0;
        if (p.block_end_ns) q.block_end_ns = p.block_end_ns + b0;
        kern<<<static_cast<unsigned>(nb), kThreads, smem, st>>>(q);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace sbimpl
}  // namespace momc_b200

#include "sampler_batch.cuh"

namespace momc_b200 {
namespace sbimpl {

inline bool force_step_kernel()
{
    static const bool v = [] {
        const char* e = std::getenv("MOMC_SAMPLER_STEP");
        return e && e[0] == '1';
    }();
    return v;
}

// n <= 42: batched resolution (sampler_batch.cuh); n <= 64: per-step resolution
template <int NMAX, int LANES, int VAR, int DMAX>
int launch_small(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    const bool udt = p.dt == 1.0 && p.s_dt_a0 == 1.0;
    if constexpr (NMAX <= 42) {
        if (!force_step_kernel()) {
            if (udt) return launch_batch_u<NMAX, LANES, VAR, DMAX, true>(p, nblocks, st);
            return launch_batch_u<NMAX, LANES, VAR, DMAX, false>(p, nblocks, st);
        }
    }
    if (udt) return launch_small_u<NMAX, LANES, VAR, DMAX, true>(p, nblocks, st);
    return launch_small_u<NMAX, LANES, VAR, DMAX, false>(p, nblocks, st);
}

template <int NMAX, int LANES, int DMAX>
int launch_variant(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    switch (p.variant) {
        case 0: return launch_small<NMAX, LANES, 0, DMAX>(p, nblocks, st);
        case 1: return launch_small<NMAX, LANES, 1, DMAX>(p, nblocks, st);
        default: return launch_small<NMAX, LANES, 2, DMAX>(p, nblocks, st);
    }
}

}  // namespace sbimpl

// instantiation units sampler_n<NMAX>_d<DMAX>.cu
#define MOMC_SB_DECL(N, D) int launch_small_n##N##_d##D(const SamplerParams&, long long, cudaStream_t);
MOMC_SB_DECL(16, 0)
MOMC_SB_DECL(32, 0)
MOMC_SB_DECL(42, 0)
MOMC_SB_DECL(64, 0)
MOMC_SB_DECL(16, 3)
MOMC_SB_DECL(32, 3)
MOMC_SB_DECL(42, 3)
MOMC_SB_DECL(64, 3)
#undef MOMC_SB_DECL

}  // namespace momc_b200
