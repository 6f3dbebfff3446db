// Pareto stage on the device: dedup -> cut evaluation -> collapse -> non-dominated front
// -> archive order -> reference point -> hypervolume. Restates pareto.hpp:253-410, 540-655.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "ctx.cuh"

namespace momc_b200 {

// Device-resident archive / value set produced by the Pareto stage.
struct DevArchive {
    long long F = 0;  // entries
    int K = 0;
    int wpc = 0;      // 0 for objective-only archives
    DevBuf<double> vals;     // F x K, lexicographically descending
    DevBuf<uint64_t> words;  // F x wpc
};

struct ParetoTimings {
    double dedup_s = 0, eval_s = 0, collapse_s = 0, front_s = 0, order_s = 0;
    long long unique_configs = 0, unique_vectors = 0;
    int front_method = 0;  // 1 grid, 2 pairwise
};

// non_dominated_filter(pool, inst) (pareto.hpp:370-410) over M configs resident on the
// device (d_words, M x wpc). The result replaces `out`. Synchronous.
void filter_pool_device(Ctx& c, const uint64_t* d_words, long long M, DevArchive& out, ParetoTimings* tm);

// non_dominated_filter(vector<ObjectiveVector>) (pareto.hpp:253-293), cut sense; d_vals M x K.
// With d_words != nullptr (wpc words per vector), equal vectors keep the lex-smallest
// config (the cross-shard merge of pool archives, pareto.hpp:383-387).
void filter_values_device(Ctx& c, const double* d_vals, const uint64_t* d_words, int wpc, int n_spins,
                          long long M, int K, DevArchive& out, ParetoTimings* tm);

// exact equality of two sets of distinct vectors (streaming: did the running archive change?)
bool same_value_set(Ctx& c, const double* a, long long Fa, const double* b, long long Fb, int K);

// front of (M pool configs U X extra rows xv/xw) into `out` in one pass (streaming merge);
// all_vals receives the combined values, the X extra rows first. True when the fused pool
// pass ran (all_vals then holds only the X old rows)
bool filter_pool_merge_device(Ctx& c, const uint64_t* d_words, long long M, const double* xv, const uint64_t* xw,
                              long long X, DevArchive& out, DevBuf<double>& all_vals);

// detail::evaluate_cuts (pareto.hpp:330-363) for U configs: d_out U x K.
void evaluate_cuts_device(Ctx& c, const uint64_t* d_words, long long U, double* d_out);
// the same for rows idx[0..U) of d_words
void evaluate_cuts_rows(Ctx& c, const uint64_t* d_words, const uint32_t* idx, long long U, double* d_out);

// reference_point_sampled (pareto.hpp:620-642)
std::vector<double> reference_point_sampled_device(Ctx& c, int count, uint64_t seed, const double* clamp_vals = nullptr,
                                                   long long clamp_rows = 0);

// hypervolume (pareto.hpp:540-552) of F x K values (device) against r (host); validates r
// (pareto.hpp:103-118) and throws the reference's messages.
// reuse_front_grid: the archive is the output of the last filter on this context, whose front
// grid (if the grid method ran and nothing rebuilt a grid since) covers it
double hypervolume_device(Ctx& c, const double* d_vals, long long F, int K, const std::vector<double>& r,
                          bool reuse_front_grid = false);

// reference_point_sampled clamped under the archive (pareto.hpp:620-655) and the hypervolume
// at it, with r kept on the device between the two: one host round trip; r_out receives r
double hv_sampled_reference_device(Ctx& c, const double* d_vals, long long F, int K, int count, uint64_t seed,
                                   std::vector<double>& r_out, bool reuse_front_grid = false);

}  // namespace momc_b200
