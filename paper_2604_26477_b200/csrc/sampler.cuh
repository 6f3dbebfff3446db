// Batched noise-injected SB sampler (bSB / dSB / SimCIM) on sm_100a.
// Restates momc::run_sampler (solver.hpp:439-529) / integrate_block (:221-234) /
// sb_step (:152-183) / simcim_step (:188-214) / init_state (:108-124) /
// fill_step_noise (:128-136) / read_spins (:237-244), FP64, in the reference's exact
// per-element operation order (no FMA contraction), so final spins are bit-identical
// to the oracle build of the reference.
#pragma once
#include <cstdint>

#include "rng.cuh"

namespace momc_b200 {

constexpr int kSampleBlock = 128;  // trajectories per block of the sequential (generic) path
constexpr int kMaxPadDeg = 4;      // max padded row length of the register-resident path

struct SamplerParams {
    int n;            // spins
    int nnz;          // CSR entries (2m)
    int T;            // n_iterations
    int variant;      // 0 bsb, 1 dsb, 2 simcim
    double dt, a0, alpha, init_scale, s_dt_a0;  // s_dt_a0 = dt * a0 (host-rounded, solver.hpp:176)
    int L, batch, runs, chunks;                 // chunks = ceil(batch / block_traj)
    int block_traj;                             // trajectories per block (sampler_block_traj)
    long long block_begin;                      // first flattened (run, weight, chunk) block
    uint64_t seed;
    const int* row_ptr;       // n + 1
    const int* col;           // nnz, ascending within a row
    const double* vals;       // L * nnz, J(c_l) in CSR order
    const double* c0;         // L
    const double* pad_vals;   // L * n * DMAX: rows padded with exact zeros (DMAX > 0 path)
    int pad_dmax;             // 0: runtime CSR rows; else the padded row length
    int pad_col[64 * kMaxPadDeg];  // padded column indices (pad = the row's own index)
    const ZigTables* zig;
    uint64_t* words;          // (runs * L * batch) * wpc, canonical order, from row row0
    long long row0;           // first pool row held by `words` (compact pipeline pools)
    const double* sched;      // 2 x T: {-(a0 - a_t), -0.5 (1 - a_t)} per step (register path)
    unsigned long long* block_end_ns;  // per launched block (optional)
    int* nan_block;           // per launched block: 1 if any trajectory went non-finite
    int first_bad_step_task;  // debug rerun: -1, else records first bad step per block
    int test_seq_every;       // test hook: > 0 resolves every k-th (trajectory, step) stream of the
                              // batch kernel sequentially (seq_resolve); 0 in production
    int* bad_step;            // per launched block: min first non-finite step (debug rerun)
};

// Trajectories per flattened block for this problem: the register-resident path
// (n <= 64, alpha > 0) uses 256 / lanes-per-trajectory, the sequential path 128.
int sampler_block_traj(int n, double alpha);
bool sampler_uses_register_path(int n, double alpha);

// Launch the register-resident path (n <= 64, alpha > 0); returns a CUDA error.
int launch_sampler(const SamplerParams& p, long long nblocks, void* stream);

// Generic path (any n; also the exact fallback for blocks flagged by the fast kernel).
// State buffers (x, y, noise) are owned by the caller.
struct GenericScratch {
    double* x;      // [chunk_traj][n]
    double* y;
    double* xn;     // next x (double buffer)
    double* noise;  // [chunk_traj][n]
    long long cap_traj;
};
int launch_sampler_generic(const SamplerParams& p, long long nblocks, const GenericScratch& g, void* stream);

}  // namespace momc_b200
