/*
 * momc_b200.h — C-ABI of the B200 (sm_100a) hot path of momc (arXiv 2604.26477).
 *
 * Plain C: pointers and sizes only, no C++/torch types. Implemented in
 * paper_2604_26477_b200/csrc/capi.cu, built into paper_2604_26477_b200/libmomc_b200.so.
 * The reference (/root/reference/proj/include/momc) is a header-only C++ library with no
 * FFI; each entry point below replaces the reference function cited beside it, and
 * include/momc_b200/momc_b200.hpp re-exports those functions with the reference's exact
 * C++ signatures on top of this ABI.
 *
 * Conventions
 *   - Return 0 on success, MOMC_EUSAGE (2) where the reference throws
 *     std::invalid_argument, MOMC_ERUNTIME (1) where it throws anything else (numerical
 *     failure, CUDA error). `err` (may be NULL) receives the reference's message text.
 *   - "host" buffers are ordinary CPU memory; "_dev" entry points take device pointers
 *     on the context's device and run on the context's stream (asynchronous unless noted).
 *   - Spin configurations are packed exactly like momc::SamplePool (solver.hpp:288-297):
 *     wpc = ceil(n/64) uint64 words per config, bit b of word b/64 set iff s_b = +1.
 *   - Objective values are cut values (maximised), K doubles per vector, row-major.
 */
#ifndef MOMC_B200_H
#define MOMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOMC_OK 0
#define MOMC_ERUNTIME 1
#define MOMC_EUSAGE 2

typedef struct momc_ctx momc_ctx; /* one device + one stream + resident buffers */

/* momc::SolverConfig (solver.hpp:46-67); `threads` is accepted and ignored. */
typedef struct {
    int variant; /* 0 bsb, 1 dsb, 2 simcim (SolverVariant, solver.hpp:26) */
    int n_iterations;
    double dt, a0, alpha;
    int batch_size;
    double init_scale;
    uint64_t seed;
    int threads;
} momc_solver_cfg;

/* momc::MultiObjectiveInstance (instance.hpp:102-172) as flat host arrays:
 * m edges (edge_i[e] < edge_j[e]), weights row-major m x k. */
typedef struct {
    int n, k, m;
    const int32_t* edge_i;
    const int32_t* edge_j;
    const double* w;
} momc_instance_view;

/* ---------------------------------------------------------------- context
 * No reference counterpart: the reference is stateless and run_sampler owns a transient
 * thread pool (solver.hpp:463-467). A context is one device, its streams and the resident
 * buffers (instance, lattice, pool, archive) the calls below share. */
int momc_b200_ctx_create(int device, momc_ctx** out, char* err, size_t errlen);
void momc_b200_ctx_destroy(momc_ctx* ctx);
int momc_b200_ctx_sync(momc_ctx* ctx, char* err, size_t errlen);
/* the cudaStream_t the context launches on (for external events / NCCL) */
void* momc_b200_ctx_stream(momc_ctx* ctx);
/* number of kernel launches issued by this context since creation */
long long momc_b200_ctx_launches(momc_ctx* ctx);
/* sampler blocks re-run on the exact sequential path (noise-event buffer overflow) */
long long momc_b200_ctx_fallback_blocks(momc_ctx* ctx);

/* Upload / validate the instance (MultiObjectiveInstance ctor checks, instance.hpp:104-123)
 * and build the CSR graph on the device. */
int momc_b200_set_instance(momc_ctx* ctx, const momc_instance_view* inst, char* err, size_t errlen);

/* generate_uniform_instance (instance.hpp:259-284) on the device and make it the resident
 * instance; kind 0 = WeightSpec::uniform_int(lo, hi), 1 = uniform_real(lo, hi). */
int momc_b200_generate_uniform_instance(momc_ctx* ctx, int n, double density, int k, int kind, double lo, double hi,
                                        uint64_t seed, int64_t* out_m, char* err, size_t errlen);
/* generate_correlated_instance (instance.hpp:364-458) on the device (K = 3: U{1..10} base
 * layers, third layer -lambda (w1 + w2) + sigma g with sigma bisected to target_rho over the
 * 2048-config probe pool); becomes the resident instance. */
int momc_b200_generate_correlated_instance(momc_ctx* ctx, int n, double density, double target_rho, uint64_t seed,
                                           int64_t* out_m, char* err, size_t errlen);
/* measured_correlation (instance.hpp:338-357) of the resident K = 3 instance */
int momc_b200_measured_correlation(momc_ctx* ctx, int pool_size, uint64_t seed, double* out, char* err, size_t errlen);
/* copy the resident instance out: edge_i, edge_j (m), w (m x k) */
int momc_b200_instance_get(momc_ctx* ctx, int32_t* edge_i, int32_t* edge_j, double* w, char* err, size_t errlen);
/* dSB with integer weights and |H*J(c)| <= 256 uses the fused tensor-core step (exact
 * int8 / bf16 contraction H*J(c).sgn(X), then one FP64 rounding of c0/H times it) when
 * n >= n_min (default 256; INT_MAX turns it off); smaller n keep the bit-exact FP64 order of
 * the reference. */
int momc_b200_set_dense_threshold(momc_ctx* ctx, int n_min);
/* Per-kernel device times (diagnostics for roofline figures; no reference counterpart).
 * With timing on, every launch of the register sampler (class 0), the dense tensor-core GEMM
 * (1), the dense FP64 update (2) and the tensor-core evaluate_cuts (3) is bracketed by CUDA
 * events on its stream. momc_b200_kernel_times synchronises the context's streams and
 * returns the summed milliseconds and launch counts per class (4 entries each; NULL skips),
 * zeroing them when `reset` is non-zero. */
int momc_b200_set_kernel_timing(momc_ctx* ctx, int on);
int momc_b200_kernel_times(momc_ctx* ctx, double* ms, long long* counts, int reset);
/* Which sampler produced the resident pool: 0 none yet, 1 register-resident (n <= 64,
 * bit-exact), 2 sequential generic (bit-exact), 3 fused tensor-core dSB with int8 H*J(c),
 * 4 the same with bf16 H*J(c). Paths 3 and 4 round J(c).sgn(X) once (not bit-exact; see
 * DESIGN.md §3). */
int momc_b200_sampler_path(momc_ctx* ctx);

/* Upload L interior weight vectors (numerators, row-major L x k, denominator H) and
 * scalarise every one on the device: build_block_system / scalarize
 * (scalarize.hpp:22-39, :62-71). Fails with MOMC_EUSAGE and the reference's message on a
 * degenerate normalisation. Synchronous. */
int momc_b200_set_weights(momc_ctx* ctx, const int32_t* nums, int L, int H, char* err, size_t errlen);
/* copy J(c_l) (dense n x n, row-major) and c0 of weight l to host (tests) */
int momc_b200_get_coupling(momc_ctx* ctx, int l, double* J, double* c0, char* err, size_t errlen);

/* ---------------------------------------------------------------- sampler (solver.hpp) */
/* run_sampler (solver.hpp:439-529) over the resident instance and weights for the
 * flattened task range [block_begin, block_end) of (run, weight, 128-trajectory chunk)
 * blocks (block_end < 0: all runs*L*ceil(batch/128) blocks). The pool stays on the
 * device in canonical order; timings: [0] sampling seconds (device events). */
int momc_b200_sample(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs, long long block_begin,
                     long long block_end, double* seconds, char* err, size_t errlen);
/* pool geometry and copies: size = runs*L*batch configs */
long long momc_b200_pool_size(momc_ctx* ctx);
int momc_b200_pool_get(momc_ctx* ctx, uint64_t* words, int64_t* stamps_ns, char* err, size_t errlen);
const uint64_t* momc_b200_pool_device(momc_ctx* ctx);

/* Host-to-host drop-in for run_sampler (solver.hpp:439-529): instance + weights + sample +
 * copy back; words / records in the reference's canonical order (solver.hpp:493-495). */
int momc_b200_run_sampler(momc_ctx* ctx, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                          const momc_solver_cfg* cfg, int runs, uint64_t* out_words, int64_t* out_stamps_ns,
                          double* out_seconds /* [model_construction, sampling] */, char* err, size_t errlen);


/* ---------------------------------------------------------------- Pareto stage (pareto.hpp) */
/* non_dominated_filter(pool, inst) (pareto.hpp:370-410) on the pool resident in the context
 * (after momc_b200_sample). The archive (lexicographically descending, one lex-smallest
 * configuration per vector) stays resident. seconds (nullable, 5 entries): dedup, eval,
 * collapse, front, archive order. Synchronous. */
int momc_b200_filter(momc_ctx* ctx, int64_t* out_F, double* seconds, char* err, size_t errlen);
/* the same over M host configs (M x wpc words) for the resident instance */
int momc_b200_filter_pool(momc_ctx* ctx, const uint64_t* words, size_t M, int64_t* out_F, double* filtering_s,
                          char* err, size_t errlen);
/* non_dominated_filter(vector<ObjectiveVector>) (pareto.hpp:253-293); sense 0 = cut (max),
 * 1 = hamiltonian (min). Host values M x k. */
int momc_b200_filter_values(momc_ctx* ctx, const double* vals, size_t M, int k, int sense, int64_t* out_F,
                            char* err, size_t errlen);
/* merge of configuration-carrying archives (multi-GPU allgather): device values M x k and
 * device configs M x wpc; equal vectors keep the lexicographically smallest config. */
int momc_b200_filter_values_dev(momc_ctx* ctx, const double* d_vals, const uint64_t* d_words, int wpc, size_t M,
                                int k, int64_t* out_F, char* err, size_t errlen);
/* resident archive (the ParetoArchive entries of non_dominated_filter, pareto.hpp:370-410):
 * size, host copy, device pointers, device-to-device copy */
int64_t momc_b200_archive_size(momc_ctx* ctx);
int momc_b200_archive_get(momc_ctx* ctx, double* vals, uint64_t* words, char* err, size_t errlen);
int momc_b200_archive_copy_device(momc_ctx* ctx, double* d_vals, uint64_t* d_words, char* err, size_t errlen);

/* hypervolume(archive, r) (pareto.hpp:540-552) of F host vectors, or of the resident archive */
int momc_b200_hypervolume(momc_ctx* ctx, const double* vals, int64_t F, int k, const double* r, double* out,
                          char* err, size_t errlen);
int momc_b200_archive_hypervolume(momc_ctx* ctx, const double* r, double* out, char* err, size_t errlen);
/* detail::evaluate_cuts (pareto.hpp:330-363): U host configs -> U x k cut values */
int momc_b200_evaluate_cuts(momc_ctx* ctx, const uint64_t* words, size_t U, double* out, char* err, size_t errlen);
/* reference_point_sampled (pareto.hpp:620-642) and clamp_reference under the resident archive (:647-655) */
int momc_b200_reference_point_sampled(momc_ctx* ctx, int count, uint64_t seed, double* r, char* err, size_t errlen);
int momc_b200_clamp_reference(momc_ctx* ctx, double* r, char* err, size_t errlen);

/* brute_force_pareto (oracle.hpp:25-77) of the resident instance into the resident archive:
 * exact front over all configurations with s_0 = +1, equal vectors on the lex-smallest
 * configuration, entries lex-descending. Replaces the reference's 2^(n-1) Gray walk
 * (enumerate.hpp:38-83) by a vertex-separator decomposition, so the n <= 22 cap
 * (enumerate.hpp:17) becomes n <= 64 for graphs with a small separator (heavy-hex 42: under a
 * second). Integer weights only (usage error otherwise). r_exact (K, may be NULL) receives
 * reference_point_exact. */
int momc_b200_brute_force_pareto(momc_ctx* ctx, int64_t* out_F, double* r_exact, char* err, size_t errlen);
/* reference_point_exact (pareto.hpp:603-617): componentwise minimum of the cut values over
 * every configuration, by the same decomposition (no front). */
int momc_b200_reference_point_exact(momc_ctx* ctx, double* r, char* err, size_t errlen);

/* samples_to_reach (pareto.hpp:763-781) for M host configs in canonical order on the
 * resident instance: first 1-based count whose running archive reaches target_hv within
 * 1e-9 relative; *out = -1 when never reached. */
int momc_b200_samples_to_reach(momc_ctx* ctx, const uint64_t* words, size_t M, const double* r, double target_hv,
                               int64_t* out, char* err, size_t errlen);
/* convergence_trace (pareto.hpp:716-757): replay by timestamp (stable), HV of the running
 * archive at `checkpoints` evenly spaced milestones; outputs are `checkpoints` long. */
int momc_b200_convergence_trace(momc_ctx* ctx, const uint64_t* words, const int64_t* stamps_ns, size_t M,
                                const double* r, int checkpoints, double* elapsed_s, double* hv, int64_t* samples,
                                char* err, size_t errlen);

/* Self-test of the hand-written tcgen05 int8 blocks: D (128 x 128 int32, row-major) =
 * A (128 x K int8, row-major) . B (128 x K int8, row-major)^T, K a multiple of 128. */
int momc_b200_tc_i8_selftest(momc_ctx* ctx, const int8_t* A, const int8_t* B, int K, int32_t* D, char* err,
                             size_t errlen);

/* Roofline calibration (no reference counterpart): normals/s of a kernel doing
 * only the sampler's per-word noise work (Philox block per 4 words, rng.hpp:113-121; the
 * ziggurat fast test and eta = hz * wn[iz], rng.hpp:156-163). */
int momc_b200_rng_calibrate(momc_ctx* ctx, int blocks_per_thread, double* normals_per_s, char* err, size_t errlen);
/* Philox4x32-10 (rng.hpp:16-39) on the device, through the routine every sampler kernel uses:
 * out[4i..4i+3] = block(keys[i], ctrs[4i..4i+3]) (known-answer tests, test_rng.cpp:14-27) */
int momc_b200_philox_blocks(momc_ctx* ctx, const uint64_t* keys, const uint32_t* ctrs, size_t count, uint32_t* out,
                            char* err, size_t errlen);

/* ---------------------------------------------------------------- pool CSV (solver.hpp:357-432) */
/* The record rows of save_pool_csv, formatted on the device: for each of M records
 * "run,weight,trajectory,timestamp_ns,<16 hex nibbles per word>\n". With out == NULL only
 * *out_len (bytes) is computed; otherwise cap must be >= that. The two header lines are the
 * caller's (they carry the pool's timings). */
int momc_b200_format_pool_rows(momc_ctx* ctx, const uint32_t* run, const uint32_t* weight, const uint32_t* trajectory,
                               const int64_t* stamps_ns, const uint64_t* words, size_t M, int n, char* out, size_t cap,
                               size_t* out_len, char* err, size_t errlen);
/* load_pool_csv's record loop on the device: `text` = the file bytes after the two header
 * lines (the first of them is line first_lineno); empty lines are skipped; the first bad
 * line raises the reference's "<path>:<line>: malformed pool record" / "bad spin field
 * width" (code 1). The records stay on the context: *out_M, then momc_b200_parsed_pool_get. */
int momc_b200_parse_pool_rows(momc_ctx* ctx, const char* text, size_t len, int n, int first_lineno, const char* path,
                              size_t* out_M, char* err, size_t errlen);
int momc_b200_parsed_pool_get(momc_ctx* ctx, uint32_t* run, uint32_t* weight, uint32_t* trajectory, int64_t* stamps_ns,
                              uint64_t* words, char* err, size_t errlen);

/* ---------------------------------------------------------------- pipeline (pipeline.hpp:309-393) */
typedef struct {
    double model_construction_s; /* instance + lattice scalarisation (build_block_system) */
    double sampling_s;           /* run_sampler integration + readout (device events) */
    double pareto_filtering_s;   /* dedup + eval + collapse + front + order + reference + HV */
    double end_to_end_s;         /* wall clock of the whole call, host copies included */
    int64_t pool_size, unique_configs, unique_vectors, archive_size;
    double hv;
    double reference[16];
    double dedup_s, eval_s, collapse_s, front_s, order_s, reference_s, hv_s;
    int front_method; /* 1 compressed grid, 2 all-pairs */
    int sampler_path; /* momc_b200_sampler_path() of the sampling stage */
} momc_bench_report;

/* bench(): instance -> scalarise L weight vectors -> sample runs*L*batch -> filter ->
 * reference point (sampled:ref_count with the solver seed, clamped under the archive, or
 * `fixed_ref` when non-NULL) -> hypervolume. The pool is copied to out_pool when non-NULL
 * (momc::BenchResult::pool); the archive stays resident (momc_b200_archive_get). */
int momc_b200_bench(momc_ctx* ctx, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                    const momc_solver_cfg* cfg, int runs, int ref_count, const double* fixed_ref, uint64_t* out_pool,
                    momc_bench_report* report, char* err, size_t errlen);

/* The same pipeline on the resident instance + weights (no host copies besides scalars):
 * scalarise -> sample blocks [block_begin, block_end) -> filter -> (if do_hv) reference
 * point + hypervolume. Used for device-resident throughput and per-rank shards. The pool
 * holds only the rows of the sampled blocks afterwards (momc_b200_pool_size / pool_get /
 * pool_device see that contiguous canonical slice), so a streaming caller can sample run r
 * of a long job without a pool sized for all r runs. */
int momc_b200_pipeline(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs, long long block_begin,
                       long long block_end, int do_hv, int ref_count, const double* fixed_ref,
                       momc_bench_report* report, char* err, size_t errlen);
/* Streaming (time-to-optimal; the running archive of archive_insert pareto.hpp:702-710 and
 * samples_to_reach :763-781, kept on the device): a running archive on the context. stream_step samples
 * blocks [block_begin, block_end) of a `runs`-run job (compact pool), filters them into the
 * resident archive (unordered) and, with merge != 0, merges that front into the running
 * archive and (r, hv non-NULL) returns the running archive's hypervolume at r. running_merge_values merges device rows (another context's or
 * another rank's front) the same way. running_to_archive makes the running archive the
 * resident archive (archive order) for momc_b200_archive_get. */
int momc_b200_running_reset(momc_ctx* ctx, char* err, size_t errlen);
int momc_b200_stream_step(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs, long long block_begin,
                          long long block_end, int merge, const double* r, double* hv, int64_t* running_F,
                          momc_bench_report* report, char* err, size_t errlen);
/* device pointers of the resident archive (valid until the next call that replaces it) */
int momc_b200_archive_device_ptrs(momc_ctx* ctx, const double** vals, const uint64_t** words, int64_t* F);
int momc_b200_running_merge_values(momc_ctx* ctx, const double* d_vals, const uint64_t* d_words, int wpc, size_t M,
                                   int k, const double* r, double* hv, int64_t* running_F, char* err, size_t errlen);
int momc_b200_running_to_archive(momc_ctx* ctx, int64_t* out_F, char* err, size_t errlen);
/* flattened (run, weight, chunk) block count of a run configuration on this context: the
 * sharding unit (the reference's (run, weight, 512-trajectory) tasks, solver.hpp:455-499) */
long long momc_b200_num_blocks(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs);

/* ---------------------------------------------------------------- device groups (several GPUs)
 * Replaces the reference's task pool (run_sampler solver.hpp:455-522: (run, weight,
 * 512-trajectory chunk) tasks on `threads` host threads) by one context per device. Blocks
 * are split into contiguous shares (the RNG streams are position-independent,
 * solver.hpp:86-94, so the pool is the single-device pool bit for bit); each device filters
 * its share to a local front; the fronts are gathered on member 0 (NCCL all-gather when the
 * devices are distinct, peer copies otherwise) and merged by the same filter, so the archive
 * equals the single-device one (lex-min owners, pareto.hpp:390-398). */
typedef struct momc_group momc_group;
#define MOMC_GROUP_SINGLE 0 /* one device */
#define MOMC_GROUP_NCCL 1   /* ncclCommInitAll over the devices, ncclAllGather of the fronts */
#define MOMC_GROUP_COPY 2   /* cudaMemcpyPeer into member 0 (repeated devices, MOMC_GROUP_TRANSPORT=copy) */
/* devices == NULL or ndev <= 0: from MOMC_GPUS ("N" = devices 0..N-1, or a list "0,2,5");
 * unset: device 0 */
int momc_b200_group_create(const int* devices, int ndev, momc_group** out, char* err, size_t errlen);
void momc_b200_group_destroy(momc_group* g);
int momc_b200_group_size(momc_group* g);
momc_ctx* momc_b200_group_ctx(momc_group* g, int i); /* member i's context (per-device calls) */
int momc_b200_group_transport(momc_group* g);       /* MOMC_GROUP_* */
int momc_b200_group_set_instance(momc_group* g, const momc_instance_view* inst, char* err, size_t errlen);
int momc_b200_group_set_weights(momc_group* g, const int32_t* nums, int L, int H, char* err, size_t errlen);
/* momc_b200_run_sampler over the group: the whole pool in canonical order (each shard's
 * timestamps count from its own device's start) */
int momc_b200_group_run_sampler(momc_group* g, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                                const momc_solver_cfg* cfg, int runs, uint64_t* out_words, int64_t* out_stamps_ns,
                                double* out_seconds, char* err, size_t errlen);
/* momc_b200_filter_pool over the group: row shares filtered per device, fronts merged; the
 * archive is resident on member 0 (momc_b200_archive_get(momc_b200_group_ctx(g, 0), ...)) */
int momc_b200_group_filter_pool(momc_group* g, const uint64_t* words, size_t M, int64_t* out_F, double* filtering_s,
                                char* err, size_t errlen);
/* momc_b200_bench over the group (pool and stamps copied out when non-NULL); the archive is
 * resident on member 0; sampling_s and the stage times are the slowest member's */
int momc_b200_group_bench(momc_group* g, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                          const momc_solver_cfg* cfg, int runs, int ref_count, const double* fixed_ref,
                          uint64_t* out_pool, int64_t* out_stamps_ns, momc_bench_report* report, char* err,
                          size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* MOMC_B200_H */
