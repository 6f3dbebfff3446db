#pragma once
// SB sampler, batched noise resolution (n <= 42; included by sampler_impl.cuh).
//
// Same B phase and rounding as sb_small_kernel (see sampler_impl.cuh): a CTA of 128 threads
// integrates 32 trajectories of one (run, weight), LANES = 4 lanes per trajectory (lanes t,
// t + 8, t + 16, t + 24 of a warp), each lane holding NQ spins in registers. What changes is who resolves the
// (trajectory, step) noise streams of fill_step_noise (solver.hpp:128-136, rng.hpp:156-185).
// sb_small_kernel resolves one step at a time: the four lanes of a trajectory walk the same
// stream redundantly and the warp waits for the slowest of its 8 streams every step. Here the
// steps come in batches of LANES: lane h resolves the stream of step tb + h of its own
// trajectory, alone, for the whole batch (phase R), then the trajectory's lanes run the LANES
// spin updates (phase B) from the resolved streams. A warp walks 32 streams at once, so it pays
// for the slowest of 32 streams once per 4 steps instead of the slowest of 8 streams every step,
// and the Philox blocks, the fast-path tests and the walk are done once per stream.
//
// R, per stream (lane-local, no shuffles):
//   * Philox blocks 0.. of the stream into the stream's word row (kC words), and a 64-bit
//     mask of the words whose ziggurat attempt would take the fast path (|hz| < kn[iz]);
//   * the walk over the slow words in stream order: a wedge attempt takes 3 words (the
//     normal, if accepted, is hz * wn[iz] of its first word, the fast formula), a tail
//     1 + 4k words (its value is stored into its last two words); each attempt adds its word
//     increase at the normal index from which it applies, as a byte in a lane-major table
//     (spin i -> byte 16 (i / NQ) + i % NQ), and tails set a bit of the lane's 16-bit mask;
//   * one byte-wise prefix sum (x (w + carry) * 0x01010101 per word) turns the increases into
//     each normal's word offset: normal i is word i + off(i) of the row (off <= kC - 1 words,
//     so a byte holds 4 off).
//   A stream that needs more than kC words (P ~ 1e-3 at n = 42) is resolved sequentially by
//   its lane instead (seq_resolve: the reference's next_normal loop, normals packed from word
//   0, a tail's value in two words), so no block leaves the kernel for that.
// B, per step: lane h reads its 16 offset bytes (one LDS.128) and its tail bits, then updates
//   its NQ spins exactly as sb_small_kernel's B phase (bit-identical).
#include <cuda_runtime.h>

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>

#include "sampler.cuh"

namespace momc_b200 {
namespace sbimpl {

// CTA shape of the batch kernel: 128 threads (32 trajectories), 4 CTAs per SM (123 registers,
// ~48 KB shared memory each): 16 resident warps. Measured at C2: (128, 5) and (192, 3) force
// 96 registers and spill x / y across the noise phase (7.51 / 7.56 ms), (192 threads, 112
// registers) ran 8.33 ms; this shape 7.31 ms.
constexpr int kBT = 128;
constexpr int kBMin = 4;

template <int NMAX, int LANES, int VAR, int BT = 128>
struct BGeo {
    static constexpr int kTPC = BT / LANES;           // trajectories per CTA
    static constexpr int kNQ = (NMAX + LANES - 1) / LANES;  // spins per lane
    static constexpr int kNP = kNQ * LANES;                 // integrated spins (>= n)
    static constexpr int kC = 56;                           // words per stream row
    // row strides: stream h's row at h * kSS, trajectory rows at kTS == 4 mod 32 (the 8 lanes
    // of an STS.128 phase, 8 trajectories with one h, hit distinct bank quads; B's reads at
    // 4 t + NQ h are distinct over the warp)
    static constexpr int kSS = kC;
    static constexpr int kTS = LANES * kSS + 4;
    // Philox blocks per stream row (kNBU unrolled at a time); more is sequential resolution
    static constexpr int kNB = (NMAX + 14 + 3) / 4 < kC / 4 ? (NMAX + 14 + 3) / 4 : kC / 4;
    static constexpr int kNBU = (kNB + 1) / 2;
    // offset table per stream: 16 words of lane-major offset bytes, 4 half-words of tail bits
    // (lane h's at half-word h), 2 pad; per trajectory LANES streams
    static constexpr int kWS = 20;
    static constexpr int kWT = LANES * kWS + 20;  // == 4 mod 32: the 8 lanes of a quarter-warp
                                                 // (8 trajectories, one h) read distinct quads
    static constexpr int kPhiW = VAR == 1 ? 4 : 8;
    static constexpr int kPStr = VAR == 1 ? (kNP + 27) / 32 * 32 + 4 : (kNP + 13) / 16 * 16 + 2;
    // dSB with padded rows (TAB) keeps phi as a sign mask in registers: no phi rows
    static constexpr bool kTab = VAR == 1;  // (with DMAX == 3, see the kernel)
    static constexpr int kMK = 5;           // sign of x_j at mask bit j + kMK (shift counts >= 0)
    static_assert(kNP + kMK <= 64, "sign mask fits 64 bits");
    // (the ziggurat tables live in static shared memory: their addresses are immediates)
    static constexpr int words = 0;                                 // kTPC x kTS u32
    static constexpr int wofs = words + kTPC * kTS * 4;             // kTPC x kWT u32
    static constexpr int phi = wofs + kTPC * kWT * 4;               // kTPC x kPStr phi entries
    static constexpr int csr = (phi + kTPC * kPStr * kPhiW + 15) / 16 * 16;
    static_assert(LANES == 4, "one stream per lane and step of a 4-step batch");
    static_assert(kNQ <= 16, "16 offset bytes per lane");
    static_assert(NMAX + 14 <= kC, "sequential resolution packs n normals and up to 14 tails");
    static_assert(kNB * 4 <= kC && kNB * 4 < 64, "generated blocks fit the row and the mask");
};

// OR over the LANES lanes of a trajectory (lanes t + 8 h, h < LANES)
template <int LANES>
__device__ __forceinline__ uint64_t traj_or(unsigned mask, uint64_t v)
{
#pragma unroll
    for (int o = 32 / LANES; o < 32; o <<= 1) v |= __shfl_xor_sync(mask, v, o);
    return v;
}

// Ziggurat tables of the batch kernel in static shared memory (their addresses are immediates),
// plus FP32 copies of wn / fn for the wedge and tail brackets.
struct BatchZig {
    uint32_t kn[128];
    double wn[128];
    double fn[128];
    float wnf[128];
    float fnf[128];
};
static __shared__ BatchZig g_bz;

// Wedge test of rng.hpp:164-168 for the attempt with words u, u1, u2: accept iff
// fn[iz] + u01 (fn[iz-1] - fn[iz]) < exp(-x^2 / 2), x = hz wn[iz], in FP64. Decided in FP32
// unless the two sides are within 4e-5 relative: the FP32 x carries <= 3 roundings (1.8e-7), so
// -x^2/2 (|.| <= r^2/2 < 6) is off by <= 3e-6 absolute and __expf adds <= 6e-7; the FP32 lhs
// (u01 truncated to 24 bits, fn rounded) is within 5e-7 relative (adjacent fn within a factor
// 2.2). Both sides are > 2e-3, so a 4e-5 band leaves a 10x margin.
__device__ __forceinline__ bool wedge_accept(uint32_t u, uint32_t u1, uint32_t u2)
{
    const uint32_t iz = u & 127u;
    const float xf = __int2float_rn(static_cast<int32_t>(u)) * g_bz.wnf[iz];
    const float ef = __expf(-0.5f * xf * xf);
    const float uf = __uint2float_rz(u2 >> 8) * 0x1.0p-24f;  // the top 24 bits of u01, exact
    const float lf = __fmaf_rn(uf, g_bz.fnf[iz - 1] - g_bz.fnf[iz], g_bz.fnf[iz]);
    if (lf < ef * (1.0f - 4e-5f)) return true;
    if (lf > ef * (1.0f + 4e-5f)) return false;
    const double xv = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), g_bz.wn[iz]);
    const double lhs =
        __dadd_rn(g_bz.fn[iz], __dmul_rn(u01_from(u1, u2), __dsub_rn(g_bz.fn[iz - 1], g_bz.fn[iz])));
    return lhs < exp(__dmul_rn(__dmul_rn(-0.5, xv), xv));
}

// One tail trial of rng.hpp:172-178 from words a0..a3: true (and the value r + x, signed by
// hz) on accept. The decision 2y >= x^2 is taken in FP32 unless within 1e-5 relative + 4e-6
// absolute (__logf of the 53-bit u01 rounded to FP32 is within ~4e-7 absolute); the accepted
// value is always the FP64 one.
__device__ __forceinline__ bool tail_trial(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t u,
                                           double& val)
{
    const double r = 3.442619855899;
    const uint64_t v1 = (static_cast<uint64_t>(a1) << 32) | a0, v2 = (static_cast<uint64_t>(a3) << 32) | a2;
    const float xf = -__logf(__ull2float_rn((v1 >> 11) + 1) * 0x1.0p-53f) * (1.0f / 3.442619855899f);
    const float yf = -__logf(__ull2float_rn((v2 >> 11) + 1) * 0x1.0p-53f);
    const float lf = yf + yf, rf = xf * xf;
    const float band = 1e-5f * (lf + rf) + 4e-6f;
    bool acc;
    if (lf - rf > band) acc = true;
    else if (rf - lf > band) acc = false;
    else {
        const double xx = __ddiv_rn(-log(u01_open_from(a0, a1)), r);
        const double yy = -log(u01_open_from(a2, a3));
        acc = __dadd_rn(yy, yy) >= __dmul_rn(xx, xx);
    }
    if (acc) {
        const double xx = __ddiv_rn(-log(u01_open_from(a0, a1)), r);
        val = static_cast<int32_t>(u) > 0 ? __dadd_rn(r, xx) : -__dadd_rn(r, xx);
    }
    return acc;
}

// Sequential resolution of one stream (the reference's next_normal loop, rng.hpp:156-185) for
// the rare stream that needs more than kC words: normal i's word goes to row word i + g(i),
// g(i) = tails among normals <= i (a tail's value takes two words, hi first); offsets and tail
// bits into the stream's table (zeroed by the caller). Returns false if the row overflows.
template <int NQ, int kC>
__device__ __noinline__ bool seq_resolve(uint32_t* us, uint32_t* wr, int n, uint32_t k0, uint32_t k1, uint32_t lo,
                                         uint32_t tr, uint32_t wl)
{
    uint32_t blk = 0, buf[4];
    int bp = 4;
    auto next = [&]() -> uint32_t {
        if (bp == 4) {
            const uint4 b = philox(k0, k1, blk++, lo, tr, wl);
            buf[0] = b.x;
            buf[1] = b.y;
            buf[2] = b.z;
            buf[3] = b.w;
            bp = 0;
        }
        return buf[bp++];
    };
    unsigned char* wb = reinterpret_cast<unsigned char*>(wr);
    unsigned short* tb = reinterpret_cast<unsigned short*>(wr + 16);
    int slot = 0;
    for (int i = 0; i < n; ++i) {
        if (slot + 2 > kC) return false;
        for (;;) {
            const uint32_t u = next();
            const uint32_t iz = u & 127u;
            if (zmag(u) < g_bz.kn[iz]) {
                us[slot++] = u;
                break;
            }
            if (iz == 0) {
                double v;
                for (;;) {
                    const uint32_t a0 = next(), a1 = next(), a2 = next(), a3 = next();
                    if (tail_trial(a0, a1, a2, a3, u, v)) break;
                }
                us[slot] = static_cast<uint32_t>(__double2hiint(v));
                us[slot + 1] = static_cast<uint32_t>(__double2loint(v));
                slot += 2;
                wb[i + (16 - NQ) * (i / NQ)] += 4;
                tb[i / NQ] |= static_cast<unsigned short>(1u << (i % NQ));
                break;
            }
            const uint32_t a = next(), b = next();
            if (wedge_accept(u, a, b)) {
                us[slot++] = u;
                break;
            }
        }
    }
    return true;
}

// phi-row bytes of the batch kernel (none for the sign-mask path)
template <int NMAX, int LANES, int VAR, int DMAX, int BT>
__host__ __device__ constexpr int batch_phi_bytes()
{
    using G = BGeo<NMAX, LANES, VAR, BT>;
    return VAR == 1 && DMAX == 3 ? 0 : G::kTPC * G::kPStr * G::kPhiW;
}

// (a & b) | c in one LOP3
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ double lds_f64(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <int NMAX, int LANES, int VAR, int DMAX, bool UDT, int BT, int MINB>
__device__ __forceinline__ void sb_batch_body(const SamplerParams& p)
{
    using G = BGeo<NMAX, LANES, VAR, BT>;
    constexpr int TPC = G::kTPC;
    constexpr int NQ = G::kNQ;
    constexpr int NP = G::kNP;
    constexpr int kC = G::kC;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* wbuf = reinterpret_cast<uint32_t*>(smem + G::words);
    uint32_t* wofs = reinterpret_cast<uint32_t*>(smem + G::wofs);
    unsigned char* phis = smem + G::phi;
    constexpr int kCsr = (G::phi + batch_phi_bytes<NMAX, LANES, VAR, DMAX, BT>() + 15) / 16 * 16;
    unsigned char* csr = smem + kCsr;
    // coupling records as in sb_small_kernel, except TAB: {sh0, sh1, sh2, -} with
    // sh_d = j_d + kMK - 3 - d, so (M >> sh_d) has x_{j_d}'s sign bit at bit 3 + d
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
    // lane 8 h + t of a warp: trajectory t of the warp's 8, spin block h. A half-warp then holds
    // two spin blocks whose coupling tables (spins 11 h + s) start 16 banks apart, so the
    // 16 table reads of an LDS.64 phase are conflict-free (lane 4 t + h put h = 0, 2 on the same
    // banks: 1.3e8 extra wavefronts per C2 launch)
    const int t_loc = (tid >> 5) * (32 / LANES) + (tid & (32 / LANES - 1));
    const int h = (tid & 31) / (32 / LANES);

    {  // CTA setup (identical to sb_small_kernel)
        static_assert(sizeof(ZigTables) == offsetof(BatchZig, wnf), "BatchZig extends ZigTables");
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.zig);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&g_bz);
        for (int i = tid; i < static_cast<int>(sizeof(ZigTables) / 4); i += BT) dst[i] = src[i];
        for (int i = tid; i < 128; i += BT) {
            g_bz.wnf[i] = static_cast<float>(p.zig->wn[i]);
            g_bz.fnf[i] = static_cast<float>(p.zig->fn[i]);
        }
        if constexpr (DMAX == 0) {
            for (int i = tid; i <= NP; i += BT) rp[i] = p.row_ptr[i < n ? i : n];
            const double* v = p.vals + static_cast<long long>(l) * p.nnz;
            for (int i = tid; i < p.nnz; i += BT) {
                cv[i] = v[i];
                cc[i] = p.col[i];
            }
        } else if constexpr (TAB) {
            const double* v = p.pad_vals + static_cast<long long>(l) * n * DMAX;
            const double c0l = p.c0[l];
            for (int i = tid; i < NP; i += BT) {
                int* ro = reinterpret_cast<int*>(csr + i * 16);
                for (int d = 0; d < 3; ++d) ro[d] = (i < n ? p.pad_col[i * 3 + d] : i) + G::kMK - 3 - d;
                ro[3] = 0;
            }
            double* tab = reinterpret_cast<double*>(csr + NP * 16);
            for (int e = tid; e < NP * 8; e += BT) {
                const int i = e >> 3, pat = e & 7;
                double coupled = 0.0;
                for (int d = 0; d < 3; ++d) {
                    const double jv = i < n ? v[i * 3 + d] : 0.0;
                    coupled = __dadd_rn(coupled, (pat >> d) & 1 ? -jv : jv);
                }
                tab[e] = __dmul_rn(c0l, coupled);
            }
        } else {
            const double* v = p.pad_vals + static_cast<long long>(l) * n * DMAX;
            for (int i = tid; i < NP; i += BT) {
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
    const unsigned wmask = __ballot_sync(0xffffffffu, traj < p.batch);
    if (traj >= p.batch) return;  // no CTA-wide barrier below this point

    const uint64_t key = run_key(p.seed, static_cast<uint32_t>(run));
    const uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
    const uint32_t wl = static_cast<uint32_t>(l), tr = static_cast<uint32_t>(traj);
    const double c0 = p.c0[l];
    const double alpha = p.alpha, dt = p.dt, sdt = p.s_dt_a0;
    const bool pos_init = p.init_scale > 0.0;
    const int s0 = h * NQ;

    // ---- init_state (solver.hpp:108-124), as sb_small_kernel
    double x[NQ];
    double y[NQ];
    {
        const bool par = s0 & 1;
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
            if (2 * c - 1 < NQ) {
                x[2 * c - 1] = init_val(par ? cx.x : px.z, par ? cx.y : px.w);
                y[2 * c - 1] = init_val(par ? cy.x : py.z, par ? cy.y : py.w);
            }
            if (2 * c < NQ) {
                x[2 * c] = init_val(par ? cx.z : cx.x, par ? cx.w : cx.y);
                y[2 * c] = init_val(par ? cy.z : cy.x, par ? cy.w : cy.y);
            }
            px = cx;
            py = cy;
        }
    }

    unsigned char* phb = phis + t_loc * G::kPStr * G::kPhiW;
    auto put_phi = [&](int j, double xv) {
        if constexpr (VAR == 1) reinterpret_cast<uint32_t*>(phb)[j] = xv < 0.0 ? 0x80000000u : 0u;
        else reinterpret_cast<double*>(phb)[j] = xv;
    };
    auto term = [&](double jv, int o) -> double {
        if constexpr (VAR == 1)
            return __longlong_as_double(__double_as_longlong(jv) ^
                                        (static_cast<long long>(*reinterpret_cast<const uint32_t*>(phb + o)) << 32));
        else return __dmul_rn(jv, *reinterpret_cast<const double*>(phb + o));
    };
    if constexpr (!TAB) {
#pragma unroll
        for (int s = 0; s < NQ; ++s) put_phi(s0 + s, x[s]);
    }

    const uint32_t* kn = g_bz.kn;
    const double* wn = g_bz.wn;
    uint32_t* trow = wbuf + t_loc * G::kTS;   // this trajectory's LANES stream rows
    uint32_t* twr = wofs + t_loc * G::kWT;    // and their offset tables
    const uint4* recs = reinterpret_cast<const uint4*>(csr) + s0 * (TAB ? 1 : 3);
    const unsigned char* tabl = csr + NP * 16 + s0 * 64;
    const uint32_t tabs = static_cast<uint32_t>(__cvta_generic_to_shared(tabl));  // 64-byte aligned
    bool overflow = false;
    int ovf_code = 0;
    __syncwarp(wmask);

    for (int tb = 0; tb < p.T; tb += LANES) {
        // ---- R: this lane resolves the stream of step tb + h
        if (tb + h < p.T) {
            uint32_t* us = trow + h * G::kSS;
            uint32_t* wr = twr + h * G::kWS;
            const uint32_t lo = tag_word(kTagStepNoise, static_cast<uint32_t>(tb + h));
#pragma unroll
            for (int c = 0; c < G::kWS / 4; ++c) reinterpret_cast<uint4*>(wr)[c] = make_uint4(0u, 0u, 0u, 0u);
            // Philox blocks 0 .. kNB-1 of the stream into the row, and the fast-path mask F
            // (bit p: word p's attempt would take the fast path); kNB * 4 words cover the
            // stream unless it needs more (P ~ 1e-3 at n = 42: sequential resolution below)
            uint64_t F = 0;
#pragma unroll 1
            constexpr int kU = G::kNBU;  // blocks per unrolled group
            for (int c = 0; c < G::kNB; c += kU) {
                uint32_t fc = 0;
#pragma unroll
                for (int b = 0; b < kU; ++b) {
                    if (c + b < G::kNB) {
                        const uint4 r = philox(k0, k1, static_cast<uint32_t>(c + b), lo, tr, wl);
                        *reinterpret_cast<uint4*>(us + 4 * (c + b)) = r;
                        // fast iff |hz| < kn[iz]: both <= 2^31 and kn >= 1, so the sign of the
                        // difference decides; shifted in from word 3 down to word 0
                        uint32_t f = (zmag(r.w) - kn[r.w & 127u]) >> 31;
                        f = __funnelshift_l(zmag(r.z) - kn[r.z & 127u], f, 1);
                        f = __funnelshift_l(zmag(r.y) - kn[r.y & 127u], f, 1);
                        f = __funnelshift_l(zmag(r.x) - kn[r.x & 127u], f, 1);
                        fc |= f << (4 * b);
                    }
                }
                F |= static_cast<uint64_t>(fc) << (4 * c);
            }
            constexpr int kGen = 4 * G::kNB;
            // slow words, and among them the attempt starts: a wedge attempt at q takes words q,
            // q+1, q+2 whatever its outcome, so the starts are the fixpoint Y = S & ~cov(Y) (a
            // slow word is a start iff no start lies 1 or 2 words before it; unique, found by
            // iteration from the left, converging in one or two rounds). Tails take 1 + 4k words
            // and restart the computation after them.
            const uint64_t S = ~F & ((1ull << kGen) - 1);
            auto starts = [](uint64_t s) {
                // round k settles every position whose chain of slow words 1-2 apart is shorter
                // than k, so this ends within kGen rounds
                uint64_t y = s & ~((s << 1) | (s << 2));
                for (;;) {
                    const uint64_t yn = s & ~((y << 1) | (y << 2));
                    if (yn == y) return y;
                    y = yn;
                }
            };
            uint64_t Y = starts(S);
            uint32_t ylo = static_cast<uint32_t>(Y), yhi = static_cast<uint32_t>(Y >> 32);

            unsigned char* wb = reinterpret_cast<unsigned char*>(wr);
            unsigned short* tbits = reinterpret_cast<unsigned short*>(wr + 16);
            int slow = 0;  // words taken by the slow attempts so far beyond their normals
            bool seq = false;
            for (;;) {
                int q;  // next attempt start
                if (ylo) {
                    q = __ffs(ylo) - 1;
                    ylo &= ylo - 1;
                } else if (yhi) {
                    q = 31 + __ffs(yhi);
                    yhi &= yhi - 1;
                } else {
                    break;
                }
                if (q > n - 1 + slow) break;  // the n normals end before this attempt
                if (q + 2 >= kGen) {
                    seq = true;
                    break;
                }
                const uint32_t u = us[q];
                const int i = q - slow;  // the attempt's normal index
                int e, d;
                if ((u & 127u) == 0) {  // tail: 4 words per trial
                    int qq = q + 1;
                    double sval = 0.0;
                    for (;;) {
                        if (qq + 4 > kGen) {
                            seq = true;
                            break;
                        }
                        const bool ok = tail_trial(us[qq], us[qq + 1], us[qq + 2], us[qq + 3], u, sval);
                        qq += 4;
                        if (ok) break;
                    }
                    if (seq) break;
                    // the value goes into the tail's last two words: B reads lo at the normal's
                    // word and hi just before it
                    us[qq - 1] = static_cast<uint32_t>(__double2loint(sval));
                    us[qq - 2] = static_cast<uint32_t>(__double2hiint(sval));
                    e = i;
                    d = qq - q - 1;
                    if (i < NP) tbits[i / NQ] |= static_cast<unsigned short>(1u << (i % NQ));
                    Y = qq >= 64 ? 0ull : starts(S & (~0ull << qq));
                    ylo = static_cast<uint32_t>(Y);
                    yhi = static_cast<uint32_t>(Y >> 32);
                } else {
                    const bool acc = wedge_accept(u, us[q + 1], us[q + 2]);
                    e = acc ? i + 1 : i;
                    d = acc ? 2 : 3;
                }
                slow += d;
                if (e < NP) {  // lane-major byte of normal e: 16 (e / NQ) + e % NQ
                    const uint32_t ue = static_cast<uint32_t>(e);
                    wb[ue + (16 - NQ) * (ue / NQ)] += static_cast<unsigned char>(4 * d);
                }
            }
            if (n - 1 + slow >= kGen) seq = true;  // the last normals lie past the generated words
            if (p.test_seq_every > 0 && (tr + static_cast<uint32_t>(tb + h)) % p.test_seq_every == 0) seq = true;
            if (seq) {
#pragma unroll
                for (int c = 0; c < G::kWS / 4; ++c) reinterpret_cast<uint4*>(wr)[c] = make_uint4(0u, 0u, 0u, 0u);
                if (!seq_resolve<NQ, kC>(us, wr, n, k0, k1, lo, tr, wl)) {
                    overflow = true;
                    ovf_code |= 4;
                }
            }
            // increases -> offsets: byte-wise prefix sum over the 64 lane-major bytes
            uint4* w4 = reinterpret_cast<uint4*>(wr);
            uint32_t carry = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint4 v = w4[c];
                v.x = (v.x + carry) * 0x01010101u;
                v.y = (v.y + (v.x >> 24)) * 0x01010101u;
                v.z = (v.z + (v.y >> 24)) * 0x01010101u;
                v.w = (v.w + (v.z >> 24)) * 0x01010101u;
                carry = v.w >> 24;
                w4[c] = v;
            }
        }
        __syncwarp(wmask);  // the trajectory's streams of this batch are resolved

        const int nj = p.T - tb < LANES ? p.T - tb : LANES;
        for (int j = 0; j < nj; ++j) {
            const int t = tb + j;
            const double neg_drift = p.sched[2 * t];
            const double pump = p.sched[2 * t + 1];
            const uint32_t* wrj = twr + j * G::kWS;
            const uint4 Wv = *reinterpret_cast<const uint4*>(wrj + 4 * h);
            const uint32_t specm = reinterpret_cast<const unsigned short*>(wrj + 16)[h];
            const uint32_t* ubs = trow + j * G::kSS + s0;
            uint64_t M = 0;  // TAB: phi(t) as signs, x_j < 0 at bit j + kMK
            if constexpr (TAB) {
                uint32_t lm = 0;
                if (pos_init) {
                    // init_scale > 0: x is never -0.0 (x_0 = s (2u - 1) gives +0.0 at most,
                    // x + y is -0.0 only if both are, the clamp gives +-1), so x < 0 is the
                    // sign bit (a NaN trajectory is reported as a failure either way)
#pragma unroll
                    for (int s = NQ - 1; s >= 0; --s) lm = __funnelshift_l(__double2hiint(x[s]), lm, 1);
                } else {
#pragma unroll
                    for (int s = 0; s < NQ; ++s) lm |= static_cast<uint32_t>(x[s] < 0.0) << s;
                }
                M = static_cast<uint64_t>(lm) << (s0 + G::kMK);
                M = traj_or<LANES>(wmask, M);
            }

            // ---- B: spin updates (sb_step solver.hpp:159-181 / simcim_step :196-210)
#pragma unroll
            for (int s = 0; s < NQ; ++s) {
                const uint32_t Wq = s < 4 ? Wv.x : s < 8 ? Wv.y : s < 12 ? Wv.z : Wv.w;
                const uint32_t boff = __byte_perm(Wq, 0u, 0x4440u + static_cast<uint32_t>(s & 3));
                const uint32_t* wp =
                    reinterpret_cast<const uint32_t*>(reinterpret_cast<const unsigned char*>(ubs + s) + boff);
                const uint32_t u = wp[0];
                double eta = __dmul_rn(static_cast<double>(static_cast<int32_t>(u)), wn[u & 127u]);
                if (specm & (1u << s)) {
                    asm volatile("");  // a branch, not predication: tails are rare
                    eta = __hiloint2double(static_cast<int>(wp[-1]), static_cast<int>(u));
                }
                double coupled = 0.0;
                double c0c = 0.0;
                if constexpr (TAB) {
                    // table entry f0 + 2 f1 + 4 f2 (f_d = x_{j_d} < 0) at byte 8 f0 + 16 f1 + 32 f2
                    const uint4 rc = recs[s];
                    uint32_t a = lop3_and_or(static_cast<uint32_t>(M >> rc.x), 8u, tabs);
                    a = lop3_and_or(static_cast<uint32_t>(M >> rc.y), 16u, a);
                    a = lop3_and_or(static_cast<uint32_t>(M >> rc.z), 32u, a);
                    c0c = lds_f64(a + s * 64);
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
                    const double d =
                        __dadd_rn(__dsub_rn(__dmul_rn(pump, xi), __dmul_rn(c0, coupled)), __dmul_rn(alpha, eta));
                    yi = __dadd_rn(__dmul_rn(0.9, yi), __dmul_rn(1.0 - 0.9, d));
                    xi = __dadd_rn(xi, UDT ? yi : __dmul_rn(dt, yi));
                } else {
                    if constexpr (!TAB) c0c = __dmul_rn(c0, coupled);
                    const double d = __dadd_rn(__dsub_rn(__dmul_rn(neg_drift, xi), c0c), __dmul_rn(alpha, eta));
                    yi = __dadd_rn(yi, UDT ? d : __dmul_rn(dt, d));
                    xi = __dadd_rn(xi, UDT ? yi : __dmul_rn(sdt, yi));
                }
                // y <- 0 where |x| > 1 (strict, SB only), then the clamp to +-1 with x's sign: both
                // fire exactly when |x| > 1 (never for NaN, which propagates). In place under one
                // predicate: x.hi = (x.hi & sign) | hi(1.0), x.lo = 0, y = 0
                {
                    uint32_t xl = static_cast<uint32_t>(__double2loint(xi)), xh = static_cast<uint32_t>(__double2hiint(xi));
                    uint32_t yl = static_cast<uint32_t>(__double2loint(yi)), yh = static_cast<uint32_t>(__double2hiint(yi));
                    if constexpr (VAR != 2) {
                        asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %4, 0d3FF0000000000000;\n\t"
                            "@p lop3.b32 %1, %1, 0x80000000, %5, 0xEA;\n\t@p mov.b32 %0, 0;\n\t"
                            "@p mov.b32 %2, 0;\n\t@p mov.b32 %3, 0;\n\t}"
                            : "+r"(xl), "+r"(xh), "+r"(yl), "+r"(yh)
                            : "d"(fabs(xi)), "r"(0x3FF00000u));
                    } else {
                        asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %2, 0d3FF0000000000000;\n\t"
                            "@p lop3.b32 %1, %1, 0x80000000, %3, 0xEA;\n\t@p mov.b32 %0, 0;\n\t}"
                            : "+r"(xl), "+r"(xh)
                            : "d"(fabs(xi)), "r"(0x3FF00000u));
                    }
                    xi = __hiloint2double(static_cast<int>(xh), static_cast<int>(xl));
                    yi = __hiloint2double(static_cast<int>(yh), static_cast<int>(yl));
                }
                x[s] = xi;
                y[s] = yi;
            }
            if constexpr (!TAB) {
                __syncwarp(wmask);  // every lane has finished reading phi(t)
#pragma unroll
                for (int s = 0; s < NQ; ++s) put_phi(s0 + s, x[s]);
                __syncwarp(wmask);  // phi(t+1) complete
            } else {
                __syncwarp(wmask);  // this batch's rows are read before the next R
            }
        }
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
    word = traj_or<LANES>(wmask, word);
    if (h == 0) {
        const long long idx = (static_cast<long long>(run) * p.L + l) * p.batch + traj;
        p.words[idx - p.row0] = word;
    }
    if (bad) atomicOr(&p.nan_block[blockIdx.x], 1);
    if (overflow) atomicOr(&p.nan_block[blockIdx.x], 2 | ovf_code);
    if (p.block_end_ns && (tid & 31) == 0) atomicMax(&p.block_end_ns[blockIdx.x], globaltimer());
}

template <int NMAX, int LANES, int VAR, int DMAX, bool UDT, int BT, int MINB>
__global__ void __launch_bounds__(BT, MINB) sb_batch_kernel(const SamplerParams p)
{
    sb_batch_body<NMAX, LANES, VAR, DMAX, UDT, BT, MINB>(p);
}

template <int NMAX, int LANES, int VAR, int DMAX, bool UDT, int BT, int MINB>
int launch_batch_c(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    using G = BGeo<NMAX, LANES, VAR, BT>;
    const int csr_bytes = DMAX == 0 ? ((G::kNP + 1) * 4 + 15) / 16 * 16 + p.nnz * 12
                          : (VAR == 1 ? G::kNP * (16 + 64) : G::kNP * 48);
    const int smem = (G::phi + batch_phi_bytes<NMAX, LANES, VAR, DMAX, BT>() + 15) / 16 * 16 + csr_bytes + 16;
    auto kern = sb_batch_kernel<NMAX, LANES, VAR, DMAX, UDT, BT, MINB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const long long kMaxGrid = 1ll << 30;
    for (long long b0 = 0; b0 < nblocks; b0 += kMaxGrid) {
        SamplerParams q = p;
        q.block_begin = p.block_begin + b0;
        const long long nb = nblocks - b0 < kMaxGrid ? nblocks - b0 : kMaxGrid;
        q.nan_block = p.nan_block + b0;
        if (p.block_end_ns) q.block_end_ns = p.block_end_ns + b0;
        kern<<<static_cast<unsigned>(nb), BT, smem, st>>>(q);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int NMAX, int LANES, int VAR, int DMAX, bool UDT>
int launch_batch_u(const SamplerParams& p, long long nblocks, cudaStream_t st)
{
    return launch_batch_c<NMAX, LANES, VAR, DMAX, UDT, kBT, kBMin>(p, nblocks, st);
}

}  // namespace sbimpl
}  // namespace momc_b200
