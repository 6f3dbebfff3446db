// Context object behind momc_b200.h: one device, one stream, resident device buffers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "rng.cuh"
#include "sampler.cuh"

namespace momc_b200 {

// Error carrying the C-ABI code (2 = usage / std::invalid_argument, 1 = runtime).
struct ApiError : std::runtime_error {
    int code;
    ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void usage(const std::string& m) { throw ApiError(2, m); }
[[noreturn]] inline void runtime(const std::string& m) { throw ApiError(1, m); }

inline void ck(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) runtime(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// Stream of the context the calling thread is working for (set by bind()). Device
// buffers are stream-ordered allocations on it from the device's default memory pool
// (release threshold raised at context creation), so per-call scratch costs neither a
// cudaMalloc nor the implicit device synchronisation of cudaFree.
inline thread_local cudaStream_t g_alloc_stream = nullptr;

// Growable device buffer.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
    void reserve(size_t n)
    {
        if (n <= cap) return;
        release();
        const size_t bytes = sizeof(T) * (n ? n : 1);
        if (g_alloc_stream) ck(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, g_alloc_stream), "cudaMallocAsync");
        else ck(cudaMalloc(&p, bytes), "cudaMalloc");
        cap = n;
    }
    void release()
    {
        if (p) {
            if (g_alloc_stream) cudaFreeAsync(p, g_alloc_stream);
            else cudaFree(p);
        }
        p = nullptr;
        cap = 0;
    }
};

// Optional per-kernel-class device timing (momc_b200_set_kernel_timing): an event pair around
// each timed launch on its own stream, summed after the caller's synchronisation. Off by
// default; bench.py turns it on for a separate roofline pass, never for the timed value.
enum KernelClass { kKSampler = 0, kKDenseGemm = 1, kKDenseUpdate = 2, kKEvalGemm = 3, kKClasses = 4 };
struct KernelTimer {
    bool on = false;
    std::vector<cudaEvent_t> ev;  // 2 per recorded launch
    std::vector<int> cls;
    size_t used = 0;
    double ms[kKClasses] = {};
    long long count[kKClasses] = {};
    int begin(cudaStream_t st)
    {
        if (!on) return -1;
        if (2 * used + 2 > ev.size()) {
            cudaEvent_t a, b;
            ck(cudaEventCreate(&a), "event");
            ck(cudaEventCreate(&b), "event");
            ev.push_back(a);
            ev.push_back(b);
            cls.push_back(0);
        }
        ck(cudaEventRecord(ev[2 * used], st), "event");
        return static_cast<int>(used++);
    }
    void end(int i, int k, cudaStream_t st)
    {
        if (i < 0) return;
        cls[static_cast<size_t>(i)] = k;
        ck(cudaEventRecord(ev[2 * static_cast<size_t>(i) + 1], st), "event");
    }
    // call after the launches' stream has been synchronised
    void collect()
    {
        for (size_t i = 0; i < used; ++i) {
            float t = 0;
            ck(cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]), "event");
            ms[cls[i]] += t;
            count[cls[i]]++;
        }
        used = 0;
    }
    ~KernelTimer()
    {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;         // highest priority: everything but the register sampler
    cudaStream_t sample_stream = nullptr;  // lowest priority: the register sampler (other contexts' Pareto
                                           // kernels take freed SM slots first)
    cudaEvent_t ev_dep = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long launches = 0;
    long long fallback_blocks = 0;  // sampler blocks re-run on the sequential path
    int last_path = 0;              // momc_b200_sampler_path of the resident pool
    int fallback_reasons = 0;

    // instance
    int n = 0, k = 0, m = 0, nnz = 0;
    long long inst_gen = 0;     // bumped by every set_instance (caches keyed on the instance)
    long long weights_gen = 0;  // bumped when set_weights changes the lattice (caches keyed on it)
    long long weights_inst = -1;          // inst_gen the current lattice was set for
    std::vector<int32_t> h_nums_last;     // the current lattice's numerators (change detection)
    int h_H_last = 0;
    bool integer_weights = false;  // every weight integral and sum |w| < 2^31 (exact int32 cut path)
    bool cut_pack = false;         // cut values of all K objectives fit one 64-bit key (offsets)
    std::vector<long long> cut_lo; // per objective: smallest possible cut value
    std::vector<int> cut_bits;     // per objective: key bits
    bool values_are_cuts = false;  // the filter in progress orders this instance's cut values
    std::vector<int> h_ei, h_ej;
    std::vector<double> h_w;
    DevBuf<int> d_ei, d_ej, d_rowptr, d_col, d_eidx;
    DevBuf<double> d_w;
    DevBuf<double> d_wsum;          // per-objective totals of the edge weights (weight_totals())
    long long wsum_gen = -1;
    DevBuf<int> d_wi;  // integer weights (m x k) when integer_weights

    // weights / scalarisation
    int L = 0, H = 0;
    DevBuf<int> d_nums;
    DevBuf<double> d_vals, d_c0, d_padv;
    int pad_dmax = 0;               // padded row length of the register-resident sampler (0: CSR rows)
    std::vector<int> h_pad_col;     // 64 * kMaxPadDeg padded column indices
    DevBuf<ZigTables> d_zig;

    // pool
    long long pool_size = 0;
    int pool_runs = 0, pool_batch = 0;
    long long pool_block_begin = 0, pool_blocks = 0;
    int pool_block_traj = 128;
    long long pool_row0 = 0;  // first canonical row held in d_words (compact pipeline pools)
    DevBuf<uint64_t> d_words;
    DevBuf<int> d_nan, d_badstep;
    DevBuf<unsigned long long> d_block_end, d_t0;
    DevBuf<double> d_gx, d_gy, d_gxn, d_gnoise;  // generic-n scratch
    DevBuf<double> d_sched;                      // pump schedule table (register sampler)
    DevBuf<uint64_t> d_upload;                   // host pools uploaded for filtering
    std::shared_ptr<void> pareto_scratch;         // pareto.cu working buffers
    std::shared_ptr<void> dense_scratch;          // dense.cu working buffers
    int dense_min_n = 256;                        // dense int8 tensor path for dSB at n >= this
    std::shared_ptr<void> csv_scratch;            // csv.cu parsed pool
    std::shared_ptr<void> archive;
    std::shared_ptr<void> running;                // streaming: running archive (unordered)
    double running_hv = 0.0;                      // its HV at running_hv_ref (cached)
    std::vector<double> running_hv_ref;
    bool skip_order = false;                      // fronts for internal use: no archive order
    // the compressed grid in pareto_scratch (built by the front of the last filter) covers the
    // archive at (grid_archive, grid_rows): its dominated region is the archive's, so the
    // hypervolume reuses it instead of rebuilding one (pareto.cu); any other grid build bumps
    // grid_gen and invalidates it
    // page-locked staging for the small host <-> device transfers of the Pareto stage (a
    // pageable cudaMemcpyAsync stages through a driver buffer and blocks); see pinned_buf()
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    unsigned long long grid_gen = 0, front_grid_gen = ~0ull;
    const double* grid_archive = nullptr;
    long long grid_rows = -1;
    // momc_b200_pipeline with HV: the archive's lexicographic order runs on order_stream
    // beside the reference point and HV on `stream` (which read the unordered front, the same
    // value set); the pipeline joins it before returning
    cudaStream_t order_stream = nullptr;
    cudaEvent_t ev_order_fork = nullptr, ev_order_done = nullptr;
    bool order_async = false;    // the next finish_archive orders on order_stream
    bool order_pending = false;  // an order is in flight on order_stream
    const double* order_front = nullptr;  // its unordered front rows (the same value set)
    KernelTimer ktimer;                           // optional per-kernel-class device times

    ~Ctx();
};

// At least `bytes` of ctx's page-locked staging buffer (grown on demand; contents not kept).
inline void* pinned_buf(Ctx& c, size_t bytes)
{
    if (c.pinned_bytes < bytes) {
        if (c.pinned) {
            cudaStreamSynchronize(c.stream);
            cudaFreeHost(c.pinned);
            c.pinned = nullptr;
            c.pinned_bytes = 0;
        }
        size_t b = 256 * 1024;
        while (b < bytes) b <<= 1;
        if (cudaMallocHost(&c.pinned, b) != cudaSuccess) throw std::runtime_error("cudaMallocHost failed");
        c.pinned_bytes = b;
    }
    return c.pinned;
}

// Device array of the K per-objective sums of all edge weights, W_k = sum_e w_ek in edge
// order (evaluate_cuts' constant, pareto.hpp:346-361), computed once per instance.
inline const double* weight_totals(Ctx& c)
{
    if (c.wsum_gen != c.inst_gen) {
        std::vector<double> W(static_cast<size_t>(c.k), 0.0);
        for (int e = 0; e < c.m; ++e)
            for (int q = 0; q < c.k; ++q) W[static_cast<size_t>(q)] += c.h_w[static_cast<size_t>(e) * c.k + q];
        c.d_wsum.reserve(static_cast<size_t>(c.k));
        if (cudaMemcpyAsync(c.d_wsum.p, W.data(), sizeof(double) * c.k, cudaMemcpyHostToDevice, c.stream) != cudaSuccess ||
            cudaStreamSynchronize(c.stream) != cudaSuccess)
            throw std::runtime_error("weight totals upload failed");
        c.wsum_gen = c.inst_gen;
    }
    return c.d_wsum.p;
}

// Makes ctx's device current and its stream the allocation stream of this thread.
inline void bind(Ctx& c)
{
    ck(cudaSetDevice(c.device), "cudaSetDevice");
    g_alloc_stream = c.stream;
}

// dense.cu
struct SamplerParams;
bool dense_path_ok(Ctx& c, int variant);
int dense_path_kind(Ctx& c, int variant);  // 0 none, 1 int8, 2 bf16
int dense_block_traj();                      // trajectories per block of the dense path
void sample_dense(Ctx& c, const SamplerParams& p, long long b0, long long nblocks);
bool eval_gemm_ok(const Ctx& c);
void evaluate_cuts_gemm(Ctx& c, const uint64_t* d_words, const uint32_t* d_idx, long long U, double* d_out);
// enumerate.cu: exact front (resident archive) and/or exact reference point
void brute_force_device(Ctx& c, std::vector<double>* r_exact, bool front);
// trace.cu: samples_to_reach / convergence_trace over M device configs
std::optional<long long> samples_to_reach_device(Ctx& c, const uint64_t* d_words, long long M,
                                                 const std::vector<double>& r, double target);
void convergence_trace_device(Ctx& c, const uint64_t* d_words, const int64_t* h_stamps, long long M,
                              const std::vector<double>& r, int checkpoints, double* elapsed, double* hv,
                              long long* samples);
// csv.cu: pool CSV record rows (save_pool_csv / load_pool_csv bodies)
size_t format_pool_rows(Ctx& c, const uint32_t* run, const uint32_t* wt, const uint32_t* tr, const int64_t* ts,
                        const uint64_t* words, long long M, int n, char* out, size_t cap);
long long parse_pool_rows(Ctx& c, const char* text, size_t len, int n, int first_lineno, const std::string& path);
void parsed_pool_get(Ctx& c, uint32_t* run, uint32_t* wt, uint32_t* tr, int64_t* ts, uint64_t* words);
// tc_selftest.cu: D = A . B^T (128 x 128, int8 -> int32) through the hand-written tcgen05 path
void tc_i8_selftest(Ctx& c, const int8_t* hA, const int8_t* hB, int K, int32_t* hD);
// calib.cu: normals/s of the RNG-only calibration kernel
double rng_calibrate(Ctx& c, int blocks_per_thread);
// calib.cu: Philox4x32-10 blocks of (key, counter) pairs on the device (known-answer tests)
void philox_blocks(Ctx& c, const uint64_t* keys, const uint32_t* ctrs, long long count, uint32_t* out);
// capi.cu: the ziggurat tables on the device (uploaded once)
const ZigTables* device_zig(Ctx& c);
// instance_gen.cu
void generate_correlated_device(Ctx& c, int n, double density, double target_rho, uint64_t seed, std::vector<int>& ei,
                                std::vector<int>& ej, std::vector<double>& w);
double measured_correlation_device(Ctx& c, int pool_size, uint64_t seed);
void generate_uniform_device(Ctx& c, int n, double density, int k, int kind, double lo, double hi, uint64_t seed,
                             std::vector<int>& ei, std::vector<int>& ej, std::vector<double>& w);

}  // namespace momc_b200
