// Generic-n SB sampler: state in HBM, one wave of 128-trajectory blocks at a time. Used
// for n > 64 and as the exact sequential fallback for any block the register-resident
// kernel flags (noise-stream event overflow). Same arithmetic contract as
// sampler_impl.cuh: row i of J(c_l) summed over its CSR columns in ascending order from
// +0.0 with separately rounded products (equal to the shim's dense k-ordered GEMM, since
// the omitted zero products are exact no-ops), then the sb_step / simcim_step element
// update (solver.hpp:167-179, :199-210); noise drawn sequentially per rng.hpp:156-185.
// Layout of the state buffers: [spin i][wave trajectory] so that every per-spin access
// across a warp is a coalesced 256-B line.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "sampler.cuh"

namespace momc_b200 {

namespace {

struct WaveCtx {
    SamplerParams p;
    long long wave_block0;  // first block (relative to p.block_begin) of this wave
    long long wave_blocks;
    long long W;            // wave_blocks * p.block_traj
};

__device__ __forceinline__ void decode(const WaveCtx& w, long long wt, int& run, int& l, int& traj, bool& active)
{
    const int bt = w.p.block_traj;
    const long long gblock = w.p.block_begin + w.wave_block0 + wt / bt;
    const int chunk = static_cast<int>(gblock % w.p.chunks);
    const long long rl = gblock / w.p.chunks;
    l = static_cast<int>(rl % w.p.L);
    run = static_cast<int>(rl / w.p.L);
    traj = chunk * bt + static_cast<int>(wt % bt);
    active = traj < w.p.batch;
}

__global__ void gen_init(WaveCtx w, double* x, double* y)
{
    const long long wt = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (wt >= w.W) return;
    int run, l, traj;
    bool active;
    decode(w, wt, run, l, traj, active);
    if (!active) return;
    const uint64_t key = run_key(w.p.seed, static_cast<uint32_t>(run));
    DevStream sx, sy;
    sx.init(key, l, traj, tag_word(kTagInitX, 0));
    sy.init(key, l, traj, tag_word(kTagInitY, 0));
    const double h = w.p.init_scale;
    for (int i = 0; i < w.p.n; ++i) {
        const uint64_t v = sx.next_u64();
        const double u = static_cast<double>(v >> 11) * 0x1.0p-53;
        x[i * w.W + wt] = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, u), 1.0));
    }
    for (int i = 0; i < w.p.n; ++i) {
        const uint64_t v = sy.next_u64();
        const double u = static_cast<double>(v >> 11) * 0x1.0p-53;
        y[i * w.W + wt] = __dmul_rn(h, __dsub_rn(__dmul_rn(2.0, u), 1.0));
    }
}

__global__ void gen_noise(WaveCtx w, int t, double* noise)
{
    const long long wt = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (wt >= w.W) return;
    int run, l, traj;
    bool active;
    decode(w, wt, run, l, traj, active);
    if (!active) return;
    DevStream s;
    s.init(run_key(w.p.seed, static_cast<uint32_t>(run)), l, traj, tag_word(kTagStepNoise, static_cast<uint32_t>(t)));
    for (int i = 0; i < w.p.n; ++i) noise[i * w.W + wt] = normal_seq(s, w.p.zig);
}

// grid: (wave_blocks, n); block: 128 trajectories of one (run, weight); thread = (spin i, traj)
__global__ void gen_step(WaveCtx w, int t, const double* __restrict__ x, double* __restrict__ xn, double* y,
                         const double* __restrict__ noise)
{
    const long long wb = blockIdx.x;
    const int i = blockIdx.y;
    const long long wt = wb * w.p.block_traj + threadIdx.x;
    int run, l, traj;
    bool active;
    decode(w, wt, run, l, traj, active);
    if (!active) return;
    const double* Jv = w.p.vals + static_cast<long long>(l) * w.p.nnz;
    const bool dsb = w.p.variant == 1;
    double coupled = 0.0;
    for (int e = w.p.row_ptr[i]; e < w.p.row_ptr[i + 1]; ++e) {
        const double xj = x[w.p.col[e] * w.W + wt];
        const double phi = dsb ? (xj < 0.0 ? -1.0 : 1.0) : xj;
        coupled = __dadd_rn(coupled, __dmul_rn(Jv[e], phi));
    }
    const double c0 = w.p.c0[l];
    const double a_t = __ddiv_rn(static_cast<double>(t + 1), static_cast<double>(w.p.T));
    const bool noisy = w.p.alpha > 0.0;
    const double eta = noisy ? noise[i * w.W + wt] : 0.0;
    double xi = x[i * w.W + wt];
    double yi = y[i * w.W + wt];
    if (w.p.variant == 2) {
        const double pump = __dmul_rn(-0.5, __dsub_rn(1.0, a_t));
        double d = __dsub_rn(__dmul_rn(pump, xi), __dmul_rn(c0, coupled));
        if (noisy) d = __dadd_rn(d, __dmul_rn(w.p.alpha, eta));
        yi = __dadd_rn(__dmul_rn(0.9, yi), __dmul_rn(1.0 - 0.9, d));
        xi = __dadd_rn(xi, __dmul_rn(w.p.dt, yi));
    } else {
        const double neg_drift = -__dsub_rn(w.p.a0, a_t);
        double d = __dsub_rn(__dmul_rn(neg_drift, xi), __dmul_rn(c0, coupled));
        if (noisy) d = __dadd_rn(d, __dmul_rn(w.p.alpha, eta));
        yi = __dadd_rn(yi, __dmul_rn(w.p.dt, d));
        xi = __dadd_rn(xi, __dmul_rn(w.p.s_dt_a0, yi));
        yi = fabs(xi) > 1.0 ? 0.0 : yi;
    }
    xi = (xi < -1.0) ? -1.0 : xi;
    xi = (1.0 < xi) ? 1.0 : xi;
    xn[i * w.W + wt] = xi;
    y[i * w.W + wt] = yi;
    if (w.p.first_bad_step_task >= 0 && (!isfinite(xi) || !isfinite(yi)))
        atomicMin(&w.p.bad_step[w.wave_block0 + wb], t + 1);
}

// check_finite (solver.hpp:138-143) on the final state: a non-finite x never heals (NaN
// passes the clamp), and a non-finite y survives to the end for SimCIM (no reset); for SB the
// wall zeroes y whenever x overflowed, as in the reference's post-wall check.
__global__ void gen_readout(WaveCtx w, const double* __restrict__ x, const double* __restrict__ y)
{
    const long long wt = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (wt >= w.W) return;
    int run, l, traj;
    bool active;
    decode(w, wt, run, l, traj, active);
    if (!active) return;
    const int n = w.p.n;
    const int wpc = (n + 63) / 64;
    const long long idx = (static_cast<long long>(run) * w.p.L + l) * w.p.batch + traj;
    bool bad = false;
    for (int wd = 0; wd < wpc; ++wd) {
        uint64_t word = 0;
        for (int b = 0; b < 64 && wd * 64 + b < n; ++b) {
            const double v = x[(wd * 64 + b) * w.W + wt];
            word |= static_cast<uint64_t>(!(v < 0.0)) << b;
            bad |= !isfinite(v) || !isfinite(y[(wd * 64 + b) * w.W + wt]);
        }
        w.p.words[(idx - w.p.row0) * wpc + wd] = word;
    }
    const long long blk = w.wave_block0 + wt / w.p.block_traj;
    if (bad) w.p.nan_block[blk] = 1;
    if (w.p.block_end_ns && (threadIdx.x & 31) == 0) {
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        atomicMax(&w.p.block_end_ns[blk], tnow);
    }
}

}  // namespace

int launch_sampler_generic(const SamplerParams& p, long long nblocks, const GenericScratch& g, void* stream)
{
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long wave_cap = g.cap_traj / p.block_traj;
    if (wave_cap < 1) return cudaErrorInvalidValue;
    for (long long b0 = 0; b0 < nblocks; b0 += wave_cap) {
        WaveCtx w;
        w.p = p;
        w.wave_block0 = b0;
        w.wave_blocks = nblocks - b0 < wave_cap ? nblocks - b0 : wave_cap;
        w.W = w.wave_blocks * p.block_traj;
        const unsigned grid1 = static_cast<unsigned>((w.W + 127) / 128);
        gen_init<<<grid1, 128, 0, st>>>(w, g.x, g.y);
        double* xa = g.x;
        double* xb = g.xn;
        for (int t = 0; t < p.T; ++t) {
            if (p.alpha > 0.0) gen_noise<<<grid1, 128, 0, st>>>(w, t, g.noise);
            dim3 grid2(static_cast<unsigned>(w.wave_blocks), static_cast<unsigned>(p.n));
            gen_step<<<grid2, p.block_traj, 0, st>>>(w, t, xa, xb, g.y, g.noise);
            double* tmp = xa;
            xa = xb;
            xb = tmp;
        }
        gen_readout<<<grid1, 128, 0, st>>>(w, xa, g.y);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace momc_b200
