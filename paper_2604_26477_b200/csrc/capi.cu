// C-ABI (include/momc_b200.h): context, instance, scalarisation, sampler entry points.
// Host-side orchestration only; all per-sample arithmetic runs in the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/momc_b200.h"
#include "capi_internal.cuh"
#include "ctx.cuh"
#include "pareto.cuh"
#include "sampler.cuh"

using namespace momc_b200;

namespace momc_b200 {

// out row i = -(in row F - 1 - i) (the Hamiltonian-sense archive order, momc_b200_filter_values)
__global__ void k_negate_reverse_rows(const double* __restrict__ in, long long F, int K, double* __restrict__ out)
{
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < F * K;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = q / K, k = q % K;
        out[q] = -in[(F - 1 - i) * K + k];
    }
}

Ctx::~Ctx()
{
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    g_alloc_stream = nullptr;  // synchronous frees from here on (the stream goes away below)
    for (auto* b : {&d_ei, &d_ej, &d_rowptr, &d_col, &d_eidx, &d_wi, &d_nums, &d_nan, &d_badstep}) b->release();
    for (auto* b : {&d_w, &d_vals, &d_c0, &d_padv, &d_gx, &d_gy, &d_gxn, &d_gnoise, &d_sched}) b->release();
    d_zig.release();
    d_words.release();
    d_block_end.release();
    d_t0.release();
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_dep) cudaEventDestroy(ev_dep);
    if (order_stream) cudaStreamSynchronize(order_stream);
    if (ev_order_fork) cudaEventDestroy(ev_order_fork);
    if (ev_order_done) cudaEventDestroy(ev_order_done);
    if (order_stream) cudaStreamDestroy(order_stream);
    if (sample_stream) cudaStreamDestroy(sample_stream);
    if (stream) cudaStreamDestroy(stream);
    if (pinned) cudaFreeHost(pinned);
}

DevArchive& resident_archive(Ctx& c)
{
    if (!c.archive) c.archive = std::shared_ptr<void>(new DevArchive(), [](void* p) {
        auto* a = static_cast<DevArchive*>(p);
        a->vals.release();
        a->words.release();
        delete a;
    });
    return *static_cast<DevArchive*>(c.archive.get());
}

DevArchive& running_archive(Ctx& c)
{
    if (!c.running) c.running = std::shared_ptr<void>(new DevArchive(), [](void* p) {
        auto* a = static_cast<DevArchive*>(p);
        a->vals.release();
        a->words.release();
        delete a;
    });
    return *static_cast<DevArchive*>(c.running.get());
}

// running <- front(running U (vals, words)); unordered (internal use); returns the new size.
// *changed: whether the running archive's value set changed (its HV can only change then).
long long running_merge(Ctx& c, const double* d_vals, const uint64_t* d_words, long long M, int K, int wpc,
                        bool* changed = nullptr)
{
    DevArchive& R = running_archive(c);
    if (changed) *changed = M > 0;
    if (M <= 0) return R.F;
    if (R.F == 0) {  // first front: copy
        R.F = M;
        R.K = K;
        R.wpc = wpc;
        R.vals.reserve(static_cast<size_t>(M) * K);
        R.words.reserve(static_cast<size_t>(M) * wpc + 1);
        ck(cudaMemcpyAsync(R.vals.p, d_vals, sizeof(double) * M * K, cudaMemcpyDeviceToDevice, c.stream), "D2D");
        if (wpc)
            ck(cudaMemcpyAsync(R.words.p, d_words, sizeof(uint64_t) * M * wpc, cudaMemcpyDeviceToDevice, c.stream),
               "D2D");
        return R.F;
    }
    if (R.K != K || R.wpc != wpc) usage("running archive shape mismatch");
    const long long T = R.F + M;
    DevBuf<double> cv;
    DevBuf<uint64_t> cw;
    cv.reserve(static_cast<size_t>(T) * K);
    cw.reserve(static_cast<size_t>(T) * wpc + 1);
    ck(cudaMemcpyAsync(cv.p, R.vals.p, sizeof(double) * R.F * K, cudaMemcpyDeviceToDevice, c.stream), "D2D");
    ck(cudaMemcpyAsync(cv.p + R.F * K, d_vals, sizeof(double) * M * K, cudaMemcpyDeviceToDevice, c.stream), "D2D");
    if (wpc) {
        ck(cudaMemcpyAsync(cw.p, R.words.p, sizeof(uint64_t) * R.F * wpc, cudaMemcpyDeviceToDevice, c.stream), "D2D");
        ck(cudaMemcpyAsync(cw.p + R.F * wpc, d_words, sizeof(uint64_t) * M * wpc, cudaMemcpyDeviceToDevice, c.stream),
           "D2D");
    }
    const long long F_old = R.F;
    const bool so = c.skip_order;
    c.skip_order = true;
    try {
        filter_values_device(c, cv.p, wpc ? cw.p : nullptr, wpc, c.n, T, K, R, nullptr);
    } catch (...) {
        c.skip_order = so;
        throw;
    }
    c.skip_order = so;
    if (changed) *changed = !same_value_set(c, cv.p, F_old, R.vals.p, R.F, K);  // old rows lead cv
    cv.release();
    cw.release();
    return R.F;
}

// rng.hpp:62-89 ZigguratTables, same libm calls in the same order (bit-identical tables).
ZigTables host_ziggurat()
{
    ZigTables z;
    const double m1 = 2147483648.0;
    const double vn = 9.91256303526217e-3;
    double dn = 3.442619855899, tn = dn;
    const double q = vn / std::exp(-0.5 * dn * dn);
    z.kn[0] = static_cast<uint32_t>((dn / q) * m1);
    z.kn[1] = 0;
    z.wn[0] = q / m1;
    z.wn[127] = dn / m1;
    z.fn[0] = 1.0;
    z.fn[127] = std::exp(-0.5 * dn * dn);
    for (int i = 126; i >= 1; --i) {
        dn = std::sqrt(-2.0 * std::log(vn / dn + std::exp(-0.5 * dn * dn)));
        z.kn[i + 1] = static_cast<uint32_t>((dn / tn) * m1);
        tn = dn;
        z.fn[i] = std::exp(-0.5 * dn * dn);
        z.wn[i] = dn / m1;
    }
    return z;
}

// ---- K1 scalarise (scalarize.hpp:22-39), one CTA per weight vector
__global__ void scalarize_kernel(int n, int k, int nnz, int H, const int* __restrict__ nums, const double* __restrict__ w,
                                 const int* __restrict__ rowptr, const int* __restrict__ eidx, double* vals,
                                 double* rowsum_scratch, double* c0, int* degenerate)
{
    const int l = blockIdx.x;
    const int* num = nums + static_cast<long long>(l) * k;
    double* v = vals + static_cast<long long>(l) * nnz;
    for (int s = threadIdx.x; s < nnz; s += blockDim.x) {
        const int e = eidx[s];
        double acc = 0;  // `double w = 0; for k: w += c[k] * e.w[k]`, c[k] = num_k / H
        for (int q = 0; q < k; ++q)
            acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(static_cast<double>(num[q]), static_cast<double>(H)),
                                           w[static_cast<long long>(e) * k + q]));
        v[s] = acc;
    }
    __syncthreads();
    double* rs = rowsum_scratch + static_cast<long long>(l) * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0.0;  // J.rowwise().sum(): j ascending (zeros of the dense row are exact no-ops)
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) s = __dadd_rn(s, v[e]);
        rs[i] = fabs(s);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // .cwiseAbs().maxCoeff() as the running fold m = max(m, a_i) from a_0
        double m = rs[0];
        for (int i = 1; i < n; ++i) m = (m < rs[i]) ? rs[i] : m;
        if (!(m > 0.0) || !isfinite(m)) {
            degenerate[l] = 1;
            c0[l] = 0.0;
        } else {
            degenerate[l] = 0;
            c0[l] = __ddiv_rn(1.0, m);
        }
    }
}

// Large instances: the same three stages as separate grid-wide kernels (CSR values over all
// (weight, slot) pairs, row sums over all (weight, row) pairs, then the per-weight fold), so
// C4's 55 weights x 4e6 slots use the whole GPU. c_k = num_k / H is formed once per value.
__global__ void k_scal_vals(int k, long long nnz, int L, int H, const int* __restrict__ nums,
                            const double* __restrict__ w, const int* __restrict__ eidx, double* vals)
{
    const long long total = nnz * L;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int l = static_cast<int>(q / nnz);
        const long long sl = q % nnz;
        const int e = eidx[sl];
        const int* num = nums + static_cast<long long>(l) * k;
        double acc = 0;
        for (int j = 0; j < k; ++j)
            acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(static_cast<double>(num[j]), static_cast<double>(H)),
                                           w[static_cast<long long>(e) * k + j]));
        vals[q] = acc;
    }
}

__global__ void k_scal_rowsum(int n, long long nnz, int L, const int* __restrict__ rowptr,
                              const double* __restrict__ vals, double* rs)
{
    // one warp per (weight, row): lanes add strided partial sums? No: the fold is sequential
    // in column order, so a row is one thread; rows of a warp are adjacent (coalescing is
    // poor for dense rows, but the slots are read once)
    const long long total = static_cast<long long>(n) * L;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int l = static_cast<int>(q / n), i = static_cast<int>(q % n);
        const double* v = vals + static_cast<long long>(l) * nnz;
        double s = 0.0;
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) s = __dadd_rn(s, v[e]);
        rs[q] = fabs(s);
    }
}

__global__ void k_scal_c0(int n, const double* __restrict__ rs, double* c0, int* degenerate)
{
    const int l = blockIdx.x;
    const double* r = rs + static_cast<long long>(l) * n;
    // .cwiseAbs().maxCoeff() as the fold m = max(m, a_i) from a_0: NaN a_0 poisons the fold,
    // NaN a_i (i > 0) is skipped; both are degenerate through the finiteness check below
    // unless a_0 is finite, where the max over the finite a_i is order-free
    __shared__ double part[256];
    double m = -1.0;
    bool nan_rest = false;
    for (int i = 1 + threadIdx.x; i < n; i += blockDim.x) {
        const double a = r[i];
        if (a != a) nan_rest = true;
        else m = a > m ? a : m;
    }
    (void)nan_rest;
    part[threadIdx.x] = m;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) part[threadIdx.x] = part[threadIdx.x + o] > part[threadIdx.x] ? part[threadIdx.x + o]
                                                                                            : part[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double a0 = r[0];
        double mm = a0;
        if (a0 == a0 && part[0] > mm) mm = part[0];
        if (!(mm > 0.0) || !isfinite(mm)) {
            degenerate[l] = 1;
            c0[l] = 0.0;
        } else {
            degenerate[l] = 0;
            c0[l] = __ddiv_rn(1.0, mm);
        }
    }
}

// rows of J(c_l) padded to `dmax` entries with exact zeros (sampler DMAX > 0 path)
__global__ void pad_rows_kernel(int n, int nnz, int dmax, const int* __restrict__ rowptr,
                                const double* __restrict__ vals, double* padv)
{
    const int l = blockIdx.x;
    for (int s = threadIdx.x; s < n * dmax; s += blockDim.x) {
        const int i = s / dmax, d = s % dmax;
        const int e = rowptr[i] + d;
        padv[static_cast<long long>(l) * n * dmax + s] = e < rowptr[i + 1] ? vals[static_cast<long long>(l) * nnz + e] : 0.0;
    }
}

// per-block sampler flags -> {OR of all flags, first block with bit 1 (or INT_MAX)} at
// flags[n], flags[n + 1], so the host reads two words instead of one per block
__global__ void k_flag_summary(int* flags, long long n)
{
    int acc = 0, first = 0x7fffffff;
    for (long long b = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; b < n;
         b += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int f = flags[b];
        acc |= f;
        if ((f & 1) && b < first) first = static_cast<int>(b);
    }
    acc = __reduce_or_sync(0xffffffffu, acc);
    first = __reduce_min_sync(0xffffffffu, first);
    if ((threadIdx.x & 31) == 0) {
        if (acc) atomicOr(flags + n, acc);
        if (first != 0x7fffffff) atomicMin(flags + n + 1, first);
    }
}

__global__ void stamp_t0(unsigned long long* t0)
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *t0 = t;
}

void validate_cfg(const momc_solver_cfg* c)
{  // SolverConfig::validate (solver.hpp:57-66)
    if (c->n_iterations < 1) usage("n_iterations must be >= 1");
    if (!(c->dt > 0.0)) usage("dt must be positive");
    if (!(c->a0 > 0.0)) usage("a0 must be positive");
    if (c->alpha < 0.0) usage("alpha must be non-negative");
    if (c->batch_size < 1) usage("batch_size must be >= 1");
    if (c->init_scale < 0.0) usage("init_scale must be non-negative");
    if (c->threads < 0) usage("threads must be non-negative");
    if (c->variant < 0 || c->variant > 2) usage("unknown solver variant");
}

void set_instance(Ctx& c, const momc_instance_view* iv)
{
    ++c.inst_gen;
    // MultiObjectiveInstance ctor (instance.hpp:104-123)
    if (iv->n < 1) usage("vertex count must be positive");
    if (iv->k < 1) usage("objective count must be positive");
    if (iv->m < 0) usage("edge count must be non-negative");
    bool sorted = true;  // strictly increasing (i, j): duplicates are impossible, CSR needs no sort
    for (int e = 0; e < iv->m; ++e) {
        const int i = iv->edge_i[e], j = iv->edge_j[e];
        if (i == j) usage("self-loop edge");
        if (i < 0 || j < 0 || i >= iv->n || j >= iv->n || i >= j) usage("edge endpoints must satisfy 0 <= i < j < n");
        if (e > 0) {
            const int pi = iv->edge_i[e - 1], pj = iv->edge_j[e - 1];
            if (!(pi < i || (pi == i && pj < j))) sorted = false;
        }
    }
    if (!sorted) {
        std::unordered_set<long long> seen;
        seen.reserve(static_cast<size_t>(iv->m) * 2 + 1);
        for (int e = 0; e < iv->m; ++e)
            if (!seen.insert(static_cast<long long>(iv->edge_i[e]) * iv->n + iv->edge_j[e]).second) usage("duplicate edge");
    }
    c.n = iv->n;
    c.k = iv->k;
    c.m = iv->m;
    c.h_ei.assign(iv->edge_i, iv->edge_i + iv->m);
    c.h_ej.assign(iv->edge_j, iv->edge_j + iv->m);
    c.h_w.assign(iv->w, iv->w + static_cast<size_t>(iv->m) * iv->k);
    // exact-integer cut path: all weights integral, |sum| < 2^31 per layer
    bool integral = true;
    std::vector<double> absum(static_cast<size_t>(c.k), 0.0);
    for (int e = 0; e < c.m; ++e)
        for (int q = 0; q < c.k; ++q) {
            const double v = c.h_w[static_cast<size_t>(e) * c.k + q];
            if (!(std::floor(v) == v) || !std::isfinite(v)) integral = false;
            absum[static_cast<size_t>(q)] += std::fabs(v);
        }
    for (double a : absum)
        if (!(a < 2147483647.0)) integral = false;
    c.integer_weights = integral;
    // cut value ranges (a cut sums a subset of the edges' weights): with integer weights and
    // at most 64 bits for all K offsets, archive orders sort one packed key
    c.cut_pack = false;
    c.cut_lo.assign(static_cast<size_t>(c.k), 0);
    c.cut_bits.assign(static_cast<size_t>(c.k), 0);
    if (integral) {
        int total = 0;
        for (int q = 0; q < c.k; ++q) {
            long long lo = 0, hi = 0;
            for (int e = 0; e < c.m; ++e) {
                const long long w = static_cast<long long>(c.h_w[static_cast<size_t>(e) * c.k + q]);
                (w < 0 ? lo : hi) += w;
            }
            int bits = 1;
            while (bits < 62 && (1ll << bits) <= hi - lo) ++bits;
            c.cut_lo[static_cast<size_t>(q)] = lo;
            c.cut_bits[static_cast<size_t>(q)] = bits;
            total += bits;
        }
        c.cut_pack = total <= 64;
    }
    // CSR of the symmetric graph, rows i, columns ascending; eidx maps a slot to its edge
    c.nnz = 2 * c.m;
    std::vector<int> deg(static_cast<size_t>(c.n) + 1, 0);
    for (int e = 0; e < c.m; ++e) {
        ++deg[static_cast<size_t>(c.h_ei[e])];
        ++deg[static_cast<size_t>(c.h_ej[e])];
    }
    std::vector<int> rowptr(static_cast<size_t>(c.n) + 1, 0);
    for (int i = 0; i < c.n; ++i) rowptr[static_cast<size_t>(i) + 1] = rowptr[static_cast<size_t>(i)] + deg[static_cast<size_t>(i)];
    std::vector<int> col(static_cast<size_t>(c.nnz)), eidx(static_cast<size_t>(c.nnz));
    if (sorted) {  // visiting (i, j) in order appends ascending columns to every row
        std::vector<int> fill(rowptr.begin(), rowptr.end() - 1);
        for (int e = 0; e < c.m; ++e) {
            const int i = c.h_ei[static_cast<size_t>(e)], j = c.h_ej[static_cast<size_t>(e)];
            col[static_cast<size_t>(fill[static_cast<size_t>(i)])] = j;
            eidx[static_cast<size_t>(fill[static_cast<size_t>(i)]++)] = e;
            col[static_cast<size_t>(fill[static_cast<size_t>(j)])] = i;
            eidx[static_cast<size_t>(fill[static_cast<size_t>(j)]++)] = e;
        }
    } else {
        std::vector<std::vector<std::pair<int, int>>> rows(static_cast<size_t>(c.n));
        for (int e = 0; e < c.m; ++e) {
            rows[static_cast<size_t>(c.h_ei[static_cast<size_t>(e)])].push_back({c.h_ej[static_cast<size_t>(e)], e});
            rows[static_cast<size_t>(c.h_ej[static_cast<size_t>(e)])].push_back({c.h_ei[static_cast<size_t>(e)], e});
        }
        for (int i = 0; i < c.n; ++i) {
            auto& r = rows[static_cast<size_t>(i)];
            std::sort(r.begin(), r.end());
            for (size_t q = 0; q < r.size(); ++q) {
                col[static_cast<size_t>(rowptr[static_cast<size_t>(i)]) + q] = r[q].first;
                eidx[static_cast<size_t>(rowptr[static_cast<size_t>(i)]) + q] = r[q].second;
            }
        }
    }
    int maxdeg = 0;
    for (int i = 0; i < c.n; ++i) maxdeg = std::max(maxdeg, deg[static_cast<size_t>(i)]);
    c.pad_dmax = (c.n <= 64 && maxdeg <= 3) ? 3 : 0;  // instantiated padded row length
    c.h_pad_col.assign(64 * kMaxPadDeg, 0);
    if (c.pad_dmax > 0) {
        for (int i = 0; i < c.n; ++i)
            for (int d = 0; d < c.pad_dmax; ++d)
                c.h_pad_col[static_cast<size_t>(i * c.pad_dmax + d)] =
                    d < deg[static_cast<size_t>(i)] ? col[static_cast<size_t>(rowptr[static_cast<size_t>(i)] + d)] : i;
    }
    const size_t mk = static_cast<size_t>(c.m) * c.k;
    c.d_ei.reserve(static_cast<size_t>(c.m));
    c.d_ej.reserve(static_cast<size_t>(c.m));
    c.d_w.reserve(mk);
    c.d_rowptr.reserve(static_cast<size_t>(c.n) + 1);
    c.d_col.reserve(static_cast<size_t>(c.nnz));
    c.d_eidx.reserve(static_cast<size_t>(c.nnz));
    ck(cudaMemcpyAsync(c.d_ei.p, c.h_ei.data(), sizeof(int) * c.m, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(c.d_ej.p, c.h_ej.data(), sizeof(int) * c.m, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(c.d_w.p, c.h_w.data(), sizeof(double) * mk, cudaMemcpyHostToDevice, c.stream), "H2D");
    if (integral) {
        std::vector<int> wi(mk);
        for (size_t q = 0; q < mk; ++q) wi[q] = static_cast<int>(c.h_w[q]);
        c.d_wi.reserve(mk);
        ck(cudaMemcpyAsync(c.d_wi.p, wi.data(), sizeof(int) * mk, cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cudaStreamSynchronize(c.stream), "sync");
    }
    ck(cudaMemcpyAsync(c.d_rowptr.p, rowptr.data(), sizeof(int) * (c.n + 1), cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(c.d_col.p, col.data(), sizeof(int) * c.nnz, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(c.d_eidx.p, eidx.data(), sizeof(int) * c.nnz, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaStreamSynchronize(c.stream), "sync");
    c.L = 0;  // weights must be re-scalarised against the new instance
}

void set_weights(Ctx& c, const int32_t* nums, int L, int H)
{
    if (c.n == 0) usage("no instance set");
    if (L < 1) usage("block system needs at least one weight vector");
    if (H < 1) usage("lattice resolution must be positive");
    for (int l = 0; l < L; ++l) {  // WeightVector ctor (weights.hpp:28-40)
        long long s = 0;
        for (int q = 0; q < c.k; ++q) {
            if (nums[static_cast<size_t>(l) * c.k + q] < 0) usage("weight numerators must be non-negative");
            s += nums[static_cast<size_t>(l) * c.k + q];
        }
        if (s != H) usage("weight numerators must sum to the resolution");
    }
    {  // a new lattice (or a new instance) invalidates lattice-keyed caches; re-scalarising
       // the same lattice (every pipeline call) does not
        const bool same = c.weights_inst == c.inst_gen && c.h_H_last == H &&
                          c.h_nums_last.size() == static_cast<size_t>(L) * c.k &&
                          std::equal(c.h_nums_last.begin(), c.h_nums_last.end(), nums);
        if (!same) {
            ++c.weights_gen;
            c.weights_inst = c.inst_gen;
            c.h_H_last = H;
            c.h_nums_last.assign(nums, nums + static_cast<size_t>(L) * c.k);
        }
    }
    c.L = L;
    c.H = H;
    c.d_nums.reserve(static_cast<size_t>(L) * c.k);
    c.d_vals.reserve(static_cast<size_t>(L) * (c.nnz ? c.nnz : 1));
    c.d_c0.reserve(static_cast<size_t>(L));
    DevBuf<double> rs;
    rs.reserve(static_cast<size_t>(L) * c.n);
    DevBuf<int> degen;
    degen.reserve(static_cast<size_t>(L));
    ck(cudaMemcpyAsync(c.d_nums.p, nums, sizeof(int) * L * c.k, cudaMemcpyHostToDevice, c.stream), "H2D");
    if (static_cast<long long>(c.nnz) * L <= (1ll << 20)) {  // small: one CTA per weight
        scalarize_kernel<<<L, 256, 0, c.stream>>>(c.n, c.k, c.nnz, H, c.d_nums.p, c.d_w.p, c.d_rowptr.p, c.d_eidx.p,
                                                  c.d_vals.p, rs.p, c.d_c0.p, degen.p);
        ++c.launches;
    } else {
        const long long tv = static_cast<long long>(c.nnz) * L, tr = static_cast<long long>(c.n) * L;
        k_scal_vals<<<static_cast<unsigned>(std::min<long long>((tv + 255) / 256, 148ll * 64)), 256, 0, c.stream>>>(
            c.k, c.nnz, L, H, c.d_nums.p, c.d_w.p, c.d_eidx.p, c.d_vals.p);
        k_scal_rowsum<<<static_cast<unsigned>(std::min<long long>((tr + 127) / 128, 148ll * 64)), 128, 0, c.stream>>>(
            c.n, c.nnz, L, c.d_rowptr.p, c.d_vals.p, rs.p);
        k_scal_c0<<<L, 256, 0, c.stream>>>(c.n, rs.p, c.d_c0.p, degen.p);
        c.launches += 3;
    }
    ck(cudaGetLastError(), "scalarize_kernel");
    std::vector<int> h_degen(static_cast<size_t>(L));
    ck(cudaMemcpyAsync(h_degen.data(), degen.p, sizeof(int) * L, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "sync");
    rs.release();
    degen.release();
    for (int l = 0; l < L; ++l) {
        if (h_degen[static_cast<size_t>(l)]) {
            c.L = 0;
            usage("degenerate scalarized coupling: normalization undefined");
        }
    }
    if (c.pad_dmax > 0) {
        c.d_padv.reserve(static_cast<size_t>(L) * c.n * c.pad_dmax);
        pad_rows_kernel<<<L, 128, 0, c.stream>>>(c.n, c.nnz, c.pad_dmax, c.d_rowptr.p, c.d_vals.p, c.d_padv.p);
        ++c.launches;
        ck(cudaGetLastError(), "pad_rows_kernel");
        ck(cudaStreamSynchronize(c.stream), "sync");
    }
}

// canonical pool rows [r0, r1) covered by sampler blocks [b0, b1)
std::pair<long long, long long> rows_of_blocks(int batch, int bt, long long b0, long long b1)
{
    if (b1 <= b0) return {0, 0};
    const int chunks = (batch + bt - 1) / bt;
    const long long r0 = (b0 / chunks) * batch + (b0 % chunks) * static_cast<long long>(bt);
    const long long last = b1 - 1;
    const long long r1 = (last / chunks) * batch + std::min<long long>((last % chunks + 1) * static_cast<long long>(bt), batch);
    return {r0, r1};
}

// compact: d_words holds only the rows of the sampled blocks (pool_row0 = first row)
void sample(Ctx& c, const momc_solver_cfg* cfg, int runs, long long b_begin, long long b_end, double* seconds,
            bool compact)
{
    validate_cfg(cfg);
    if (c.n == 0) usage("no instance set");
    if (c.L < 1) usage("run_sampler needs at least one weight vector");
    if (runs < 1) usage("runs must be >= 1");
    const int batch = cfg->batch_size;
    const bool regpath = sampler_uses_register_path(c.n, cfg->alpha);
    const int dkind = regpath ? 0 : dense_path_kind(c, cfg->variant);
    const int bt = dkind ? dense_block_traj() : sampler_block_traj(c.n, cfg->alpha);
    const int chunks = (batch + bt - 1) / bt;
    const long long total_blocks = static_cast<long long>(runs) * c.L * chunks;
    if (b_end < 0 || b_end > total_blocks) b_end = total_blocks;
    if (b_begin < 0 || b_begin > b_end) usage("invalid block range");
    const long long nblocks = b_end - b_begin;
    const int wpc = (c.n + 63) / 64;
    c.pool_size = static_cast<long long>(runs) * c.L * batch;
    c.pool_row0 = 0;
    if (compact) {
        const auto rr = rows_of_blocks(batch, bt, b_begin, b_end);
        c.pool_row0 = rr.first;
        c.pool_size = rr.second - rr.first;
    }
    c.pool_runs = runs;
    c.pool_batch = batch;
    c.pool_block_begin = b_begin;
    c.pool_blocks = nblocks;
    c.pool_block_traj = bt;
    c.d_words.reserve(static_cast<size_t>(c.pool_size) * wpc);
    c.d_nan.reserve(static_cast<size_t>(nblocks) + 2);
    c.d_badstep.reserve(static_cast<size_t>(nblocks) + 1);
    c.d_block_end.reserve(static_cast<size_t>(nblocks) + 1);
    c.d_t0.reserve(2);
    device_zig(c);
    ck(cudaMemsetAsync(c.d_nan.p, 0, sizeof(int) * (nblocks + 1), c.stream), "memset");
    ck(cudaMemsetAsync(c.d_nan.p + nblocks + 1, 0x7f, sizeof(int), c.stream), "memset");
    ck(cudaMemsetAsync(c.d_block_end.p, 0, sizeof(unsigned long long) * (nblocks + 1), c.stream), "memset");

    SamplerParams p{};
    p.n = c.n;
    p.nnz = c.nnz;
    p.T = cfg->n_iterations;
    p.variant = cfg->variant;
    p.dt = cfg->dt;
    p.a0 = cfg->a0;
    p.alpha = cfg->alpha;
    p.init_scale = cfg->init_scale;
    p.s_dt_a0 = cfg->dt * cfg->a0;
    p.L = c.L;
    p.batch = batch;
    p.runs = runs;
    p.chunks = chunks;
    p.block_traj = bt;
    p.block_begin = b_begin;
    p.seed = cfg->seed;
    p.row_ptr = c.d_rowptr.p;
    p.col = c.d_col.p;
    p.vals = c.d_vals.p;
    p.c0 = c.d_c0.p;
    p.pad_vals = c.d_padv.p;
    p.pad_dmax = c.pad_dmax;
    std::copy(c.h_pad_col.begin(), c.h_pad_col.end(), p.pad_col);
    p.zig = c.d_zig.p;
    p.words = c.d_words.p;
    p.row0 = c.pool_row0;
    {  // pump schedule per step (solver.hpp:70-76), same IEEE operations as the device formula
        std::vector<double> sched(2 * static_cast<size_t>(cfg->n_iterations));
        for (int t = 0; t < cfg->n_iterations; ++t) {
            const double a_t = static_cast<double>(t + 1) / static_cast<double>(cfg->n_iterations);
            sched[2 * static_cast<size_t>(t)] = -(cfg->a0 - a_t);
            sched[2 * static_cast<size_t>(t) + 1] = -0.5 * (1.0 - a_t);
        }
        c.d_sched.reserve(sched.size());
        ck(cudaMemcpyAsync(c.d_sched.p, sched.data(), sizeof(double) * sched.size(), cudaMemcpyHostToDevice, c.stream),
           "H2D");
        p.sched = c.d_sched.p;
    }
    p.block_end_ns = c.d_block_end.p;
    p.nan_block = c.d_nan.p;
    p.first_bad_step_task = -1;
    p.bad_step = c.d_badstep.p;
    {  // test hook: MOMC_TEST_SEQ_STREAMS=k resolves every k-th noise stream of the batch
       // kernel on its sequential in-kernel path (the words must be identical)
        const char* f = std::getenv("MOMC_TEST_SEQ_STREAMS");
        p.test_seq_every = f ? std::atoi(f) : 0;
    }

    auto scratch = [&](long long blocks) {
        long long cap = std::min<long long>(blocks, 4096) * bt;
        if (cap < bt) cap = bt;
        c.d_gx.reserve(static_cast<size_t>(cap) * c.n);
        c.d_gy.reserve(static_cast<size_t>(cap) * c.n);
        c.d_gxn.reserve(static_cast<size_t>(cap) * c.n);
        c.d_gnoise.reserve(static_cast<size_t>(cap) * c.n);
        return GenericScratch{c.d_gx.p, c.d_gy.p, c.d_gxn.p, c.d_gnoise.p, cap};
    };
    GenericScratch g{};
    const bool densepath = dkind != 0;
    if (!regpath && !densepath) g = scratch(nblocks);
    c.last_path = regpath ? 1 : densepath ? 2 + dkind : 2;

    // the register sampler runs on the low-priority stream, after everything queued so far
    cudaStream_t ss = c.stream;
    if (regpath && nblocks > 0) {
        ss = c.sample_stream;
        ck(cudaEventRecord(c.ev_dep, c.stream), "event");
        ck(cudaStreamWaitEvent(ss, c.ev_dep, 0), "event wait");
    }
    stamp_t0<<<1, 1, 0, ss>>>(c.d_t0.p);
    ++c.launches;
    ck(cudaEventRecord(c.ev0, ss), "event");
    if (nblocks > 0) {
        if (densepath) {
            sample_dense(c, p, b_begin, nblocks);  // tensor-core J sgn(X) (dense.cu)
        } else {
            const int kt = regpath ? c.ktimer.begin(ss) : -1;
            const int rc = regpath ? launch_sampler(p, nblocks, ss) : launch_sampler_generic(p, nblocks, g, c.stream);
            c.ktimer.end(kt, kKSampler, ss);
            ck(static_cast<cudaError_t>(rc), "sampler launch");
            c.launches += regpath ? 1 : 2 + (long long)p.T * (cfg->alpha > 0 ? 2 : 1);
        }
    }
    ck(cudaEventRecord(c.ev1, ss), "event");
    // Per-block flags: bit 2 = the register path's noise-event buffer overflowed (re-run the
    // block on the exact sequential path); bit 1 = some trajectory went non-finite. Reduced on
    // the device; the per-block words come back only when some block raised a flag.
    std::vector<int> flags;
    int summary[2] = {0, 0x7f7f7f7f};
    if (nblocks > 0) {
        k_flag_summary<<<static_cast<unsigned>(std::min<long long>((nblocks + 255) / 256, 148)), 256, 0, ss>>>(c.d_nan.p,
                                                                                                          nblocks);
        ++c.launches;
        auto* ph = static_cast<int*>(pinned_buf(c, 2 * sizeof(int)));
        ck(cudaMemcpyAsync(ph, c.d_nan.p + nblocks, 2 * sizeof(int), cudaMemcpyDeviceToHost, ss), "D2H");
        ck(cudaStreamSynchronize(ss), "sampler");
        summary[0] = ph[0];
        summary[1] = ph[1];
    } else {
        ck(cudaStreamSynchronize(ss), "sampler");
    }
    const char* force_fb = regpath ? std::getenv("MOMC_TEST_FORCE_FALLBACK") : nullptr;
    if (summary[0] != 0 || force_fb) {
        flags.resize(static_cast<size_t>(nblocks));
        ck(cudaMemcpy(flags.data(), c.d_nan.p, sizeof(int) * nblocks, cudaMemcpyDeviceToHost), "D2H");
    }
    const long long nflags = static_cast<long long>(flags.size());  // 0: no block raised a flag
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, c.ev0, c.ev1), "event");
    c.ktimer.collect();
    // test hook: MOMC_TEST_FORCE_FALLBACK=k re-runs every k-th register-path block on the
    // sequential path (its words must be identical); never set in production
    if (force_fb) {
        const long long every = std::atoll(force_fb);
        if (every > 0)
            for (long long b = 0; b < nflags; b += every) flags[static_cast<size_t>(b)] |= 2;
    }
    bool refixed = false;
    for (long long b = 0; b < nflags; ++b) {
        if (!(flags[static_cast<size_t>(b)] & 2)) continue;
        if (!refixed) g = scratch(1);
        refixed = true;
        SamplerParams q = p;
        q.block_begin = b_begin + b;
        q.block_end_ns = nullptr;
        q.nan_block = c.d_nan.p + b;
        ck(cudaMemsetAsync(q.nan_block, 0, sizeof(int), c.stream), "memset");
        ck(static_cast<cudaError_t>(launch_sampler_generic(q, 1, g, c.stream)), "sampler fallback");
        c.launches += 3 + 2ll * p.T;
        ++c.fallback_blocks;
        c.fallback_reasons |= flags[static_cast<size_t>(b)];
        ck(cudaMemcpyAsync(&flags[static_cast<size_t>(b)], q.nan_block, sizeof(int), cudaMemcpyDeviceToHost, c.stream),
           "D2H");
    }
    if (refixed) ck(cudaStreamSynchronize(c.stream), "sampler fallback");
    if (seconds) seconds[0] = ms * 1e-3;
    // numerical failure (solver.hpp:138-143, :503-523): NaN is sticky through the wall and
    // the clamp, so a final-state scan finds every failing trajectory; the step index is
    // recovered by re-running the first failing 512-trajectory task with per-step checks.
    long long h_first = -1;
    for (long long b = 0; b < nflags; ++b)
        if (flags[static_cast<size_t>(b)] & 1) {
            h_first = b;
            break;
        }
    if (h_first >= 0) {
        const long long gb = b_begin + h_first;
        const int chunkb = static_cast<int>(gb % chunks);
        const long long rl = gb / chunks;
        const int l = static_cast<int>(rl % c.L), run = static_cast<int>(rl / c.L);
        // re-run the reference tasks (512 trajectories, kTrajectoryChunk solver.hpp:99) that
        // overlap the failing block, in order, on the sequential path in 128-trajectory blocks
        const int gbt = kSampleBlock, gchunks = (batch + gbt - 1) / gbt, per512 = 512 / gbt;
        const int tf = chunkb * bt, tl = std::min(tf + bt, batch) - 1;
        int step = 0x7f7f7f7f;
        for (int task = tf / 512; task <= tl / 512 && step == 0x7f7f7f7f; ++task) {
            const long long rb = rl * gchunks + static_cast<long long>(per512) * task;
            const long long re = std::min<long long>(rl * gchunks + gchunks, rb + per512);
            SamplerParams q = p;
            q.block_traj = gbt;
            q.chunks = gchunks;
            q.block_begin = rb;
            q.first_bad_step_task = 1;
            q.block_end_ns = nullptr;
            c.d_badstep.reserve(static_cast<size_t>(re - rb));
            ck(cudaMemsetAsync(c.d_badstep.p, 0x7f, sizeof(int) * (re - rb), c.stream), "memset");
            // scratch outputs so the pool / flags of the real run are untouched
            DevBuf<uint64_t> wtmp;
            const auto tr = rows_of_blocks(batch, gbt, rb, re);
            q.row0 = tr.first;
            wtmp.reserve(static_cast<size_t>(tr.second - tr.first) * wpc + 1);
            DevBuf<int> ntmp;
            ntmp.reserve(static_cast<size_t>(re - rb));
            q.words = wtmp.p;
            q.nan_block = ntmp.p;
            const long long cap = (re - rb) * gbt;  // the sequential path carries the per-step finiteness check
            c.d_gx.reserve(static_cast<size_t>(cap) * c.n);
            c.d_gy.reserve(static_cast<size_t>(cap) * c.n);
            c.d_gxn.reserve(static_cast<size_t>(cap) * c.n);
            c.d_gnoise.reserve(static_cast<size_t>(cap) * c.n);
            const GenericScratch gs{c.d_gx.p, c.d_gy.p, c.d_gxn.p, c.d_gnoise.p, cap};
            const int rc = launch_sampler_generic(q, re - rb, gs, c.stream);
            ck(static_cast<cudaError_t>(rc), "sampler debug launch");
            std::vector<int> bs(static_cast<size_t>(re - rb));
            ck(cudaMemcpyAsync(bs.data(), c.d_badstep.p, sizeof(int) * (re - rb), cudaMemcpyDeviceToHost, c.stream), "D2H");
            ck(cudaStreamSynchronize(c.stream), "sync");
            step = *std::min_element(bs.begin(), bs.end());
        }
        runtime("numerical failure at step " + std::to_string(step) + " (run " + std::to_string(run) + ", weight " +
                std::to_string(l) + ")");
    }
}

void pool_get(Ctx& c, uint64_t* words, int64_t* stamps)
{
    const int wpc = (c.n + 63) / 64;
    if (words)
        ck(cudaMemcpyAsync(words, c.d_words.p, sizeof(uint64_t) * c.pool_size * wpc, cudaMemcpyDeviceToHost, c.stream),
           "D2H");
    if (stamps) {
        std::vector<unsigned long long> be(static_cast<size_t>(c.pool_blocks) + 1);
        unsigned long long t0 = 0;
        ck(cudaMemcpyAsync(be.data(), c.d_block_end.p, sizeof(unsigned long long) * c.pool_blocks,
                           cudaMemcpyDeviceToHost, c.stream),
           "D2H");
        ck(cudaMemcpyAsync(&t0, c.d_t0.p, sizeof t0, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "sync");
        const int bt = c.pool_block_traj;
        const int chunks = (c.pool_batch + bt - 1) / bt;
        for (long long i = 0; i < c.pool_size; ++i) stamps[i] = 0;
        for (long long b = 0; b < c.pool_blocks; ++b) {
            const long long gb = c.pool_block_begin + b;
            const int chunk = static_cast<int>(gb % chunks);
            const long long rl = gb / chunks;
            const long long base = rl * c.pool_batch + static_cast<long long>(chunk) * bt;
            const long long stamp = be[static_cast<size_t>(b)] > t0 ? static_cast<long long>(be[static_cast<size_t>(b)] - t0) : 0;
            for (int t = 0; t < bt && chunk * bt + t < c.pool_batch; ++t) stamps[base + t - c.pool_row0] = stamp;
        }
    }
    ck(cudaStreamSynchronize(c.stream), "sync");
}

void upload_words(Ctx& c, const uint64_t* words, size_t M)
{
    const int wpc = (c.n + 63) / 64;
    c.d_upload.reserve(M * wpc + 1);
    ck(cudaMemcpyAsync(c.d_upload.p, words, sizeof(uint64_t) * M * wpc, cudaMemcpyHostToDevice, c.stream), "H2D");
}

const ZigTables* device_zig(Ctx& c)
{
    if (!c.d_zig.p) {
        c.d_zig.reserve(1);
        const ZigTables z = host_ziggurat();
        ck(cudaMemcpyAsync(c.d_zig.p, &z, sizeof z, cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cudaStreamSynchronize(c.stream), "sync");
    }
    return c.d_zig.p;
}

}  // namespace momc_b200

extern "C" {

int momc_b200_ctx_create(int device, momc_ctx** out, char* err, size_t errlen)
{
    *out = nullptr;
    return guarded(err, errlen, [&] {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1)
            runtime("no CUDA device available: the momc_b200 path has no CPU fallback");
        if (device < 0 || device >= count) usage("device index out of range");
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10) runtime("momc_b200 is built for sm_100a (B200); device is sm_" +
                                      std::to_string(prop.major) + std::to_string(prop.minor));
        auto* c = new momc_ctx();
        c->device = device;
        int least = 0, greatest = 0;
        ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "stream priorities");
        ck(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, greatest), "stream");
        ck(cudaStreamCreateWithPriority(&c->sample_stream, cudaStreamNonBlocking, least), "stream");
        ck(cudaEventCreateWithFlags(&c->ev_dep, cudaEventDisableTiming), "event");
        cudaMemPool_t pool;
        ck(cudaDeviceGetDefaultMemPool(&pool, device), "cudaDeviceGetDefaultMemPool");
        uint64_t keep = ~0ull;  // keep freed blocks cached in the pool
        ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
        ck(cudaEventCreate(&c->ev0), "event");
        ck(cudaEventCreate(&c->ev1), "event");
        *out = c;
    });
}

void momc_b200_ctx_destroy(momc_ctx* ctx) { delete ctx; }

int momc_b200_ctx_sync(momc_ctx* ctx, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] { ck(cudaStreamSynchronize(ctx->stream), "sync"); });
}

void* momc_b200_ctx_stream(momc_ctx* ctx) { return ctx->stream; }
long long momc_b200_ctx_launches(momc_ctx* ctx) { return ctx->launches; }
long long momc_b200_ctx_fallback_blocks(momc_ctx* ctx) { return ctx->fallback_blocks | (static_cast<long long>(ctx->fallback_reasons) << 40); }

int momc_b200_set_instance(momc_ctx* ctx, const momc_instance_view* inst, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        set_instance(*ctx, inst);
    });
}

int momc_b200_set_weights(momc_ctx* ctx, const int32_t* nums, int L, int H, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        set_weights(*ctx, nums, L, H);
    });
}

int momc_b200_get_coupling(momc_ctx* ctx, int l, double* J, double* c0, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        if (l < 0 || l >= ctx->L) usage("weight index out of range");
        const int n = ctx->n, nnz = ctx->nnz;
        std::vector<double> v(static_cast<size_t>(nnz));
        std::vector<int> rp(static_cast<size_t>(n) + 1), col(static_cast<size_t>(nnz));
        ck(cudaMemcpyAsync(v.data(), ctx->d_vals.p + static_cast<size_t>(l) * nnz, sizeof(double) * nnz,
                           cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaMemcpyAsync(rp.data(), ctx->d_rowptr.p, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaMemcpyAsync(col.data(), ctx->d_col.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaMemcpyAsync(c0, ctx->d_c0.p + l, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        std::fill(J, J + static_cast<size_t>(n) * n, 0.0);
        for (int i = 0; i < n; ++i)
            for (int e = rp[static_cast<size_t>(i)]; e < rp[static_cast<size_t>(i) + 1]; ++e)
                J[static_cast<size_t>(i) * n + col[static_cast<size_t>(e)]] = v[static_cast<size_t>(e)];
    });
}

int momc_b200_sample(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs, long long block_begin, long long block_end,
                     double* seconds, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        sample(*ctx, cfg, runs, block_begin, block_end, seconds);
    });
}

long long momc_b200_pool_size(momc_ctx* ctx) { return ctx->pool_size; }

int momc_b200_pool_get(momc_ctx* ctx, uint64_t* words, int64_t* stamps_ns, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] { pool_get(*ctx, words, stamps_ns); });
}

const uint64_t* momc_b200_pool_device(momc_ctx* ctx) { return ctx->d_words.p; }

int momc_b200_run_sampler(momc_ctx* ctx, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                          const momc_solver_cfg* cfg, int runs, uint64_t* out_words, int64_t* out_stamps_ns,
                          double* out_seconds, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        validate_cfg(cfg);
        if (L < 1) usage("run_sampler needs at least one weight vector");
        if (runs < 1) usage("runs must be >= 1");
        const auto t0 = std::chrono::steady_clock::now();
        set_instance(*ctx, inst);
        set_weights(*ctx, nums, L, H);
        const auto t1 = std::chrono::steady_clock::now();
        double s = 0;
        sample(*ctx, cfg, runs, 0, -1, &s);
        pool_get(*ctx, out_words, out_stamps_ns);
        const auto t2 = std::chrono::steady_clock::now();
        if (out_seconds) {
            out_seconds[0] = std::chrono::duration<double>(t1 - t0).count();
            out_seconds[1] = std::chrono::duration<double>(t2 - t1).count();
        }
    });
}

int momc_b200_filter(momc_ctx* ctx, int64_t* out_F, double* seconds, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->pool_size <= 0) usage("non-dominated filter needs a non-empty pool");
        ParetoTimings tm;
        DevArchive& a = resident_archive(*ctx);
        filter_pool_device(*ctx, ctx->d_words.p, ctx->pool_size, a, &tm);
        if (out_F) *out_F = a.F;
        if (seconds) {
            seconds[0] = tm.dedup_s;
            seconds[1] = tm.eval_s;
            seconds[2] = tm.collapse_s;
            seconds[3] = tm.front_s;
            seconds[4] = tm.order_s;
        }
    });
}

int momc_b200_filter_pool(momc_ctx* ctx, const uint64_t* words, size_t M, int64_t* out_F, double* filtering_s,
                          char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (M == 0) usage("non-dominated filter needs a non-empty pool");
        const auto t0 = std::chrono::steady_clock::now();
        upload_words(*ctx, words, M);
        DevArchive& a = resident_archive(*ctx);
        filter_pool_device(*ctx, ctx->d_upload.p, static_cast<long long>(M), a, nullptr);
        if (out_F) *out_F = a.F;
        if (filtering_s) *filtering_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

int momc_b200_filter_values(momc_ctx* ctx, const double* vals, size_t M, int k, int sense, int64_t* out_F,
                            char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (M == 0) usage("non-dominated filter needs a non-empty pool");
        if (k < 1) usage("objective vector must be non-empty");
        std::vector<double> v(vals, vals + M * static_cast<size_t>(k));
        if (sense) for (double& x : v) x = -x;  // filter in maximisation space (pareto.hpp:267-271)
        DevBuf<double> dv;
        dv.reserve(v.size());
        ck(cudaMemcpyAsync(dv.p, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, ctx->stream), "H2D");
        DevArchive& a = resident_archive(*ctx);
        filter_values_device(*ctx, dv.p, nullptr, 0, 0, static_cast<long long>(M), k, a, nullptr);
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        dv.release();
        if (sense && a.F > 0) {
            // back to Hamiltonian values, archive ordered by them (pareto.hpp:283-289): negating
            // reverses the lexicographic order, so the lex-descending front in maximisation
            // space becomes lex-descending in Hamiltonian values by negating every value and
            // reversing the rows (rows are distinct)
            DevBuf<double> t;
            t.reserve(static_cast<size_t>(a.F) * k);
            k_negate_reverse_rows<<<(static_cast<unsigned>(a.F * k) + 255) / 256, 256, 0, ctx->stream>>>(a.vals.p, a.F,
                                                                                                       k, t.p);
            ck(cudaMemcpyAsync(a.vals.p, t.p, sizeof(double) * a.F * k, cudaMemcpyDeviceToDevice, ctx->stream), "D2D");
            ck(cudaStreamSynchronize(ctx->stream), "sync");
            t.release();
        }
        if (out_F) *out_F = a.F;
    });
}

int momc_b200_filter_values_dev(momc_ctx* ctx, const double* d_vals, const uint64_t* d_words, int wpc, size_t M,
                                int k, int64_t* out_F, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        DevArchive& a = resident_archive(*ctx);
        filter_values_device(*ctx, d_vals, d_words, wpc, ctx->n, static_cast<long long>(M), k, a, nullptr);
        if (out_F) *out_F = a.F;
    });
}

int64_t momc_b200_archive_size(momc_ctx* ctx) { return ctx->archive ? resident_archive(*ctx).F : 0; }

int momc_b200_archive_get(momc_ctx* ctx, double* vals, uint64_t* words, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        DevArchive& a = resident_archive(*ctx);
        if (vals && a.F)
            ck(cudaMemcpyAsync(vals, a.vals.p, sizeof(double) * a.F * a.K, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        if (words && a.F && a.wpc)
            ck(cudaMemcpyAsync(words, a.words.p, sizeof(uint64_t) * a.F * a.wpc, cudaMemcpyDeviceToHost, ctx->stream),
               "D2H");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int momc_b200_archive_copy_device(momc_ctx* ctx, double* d_vals, uint64_t* d_words, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        DevArchive& a = resident_archive(*ctx);
        if (d_vals && a.F)
            ck(cudaMemcpyAsync(d_vals, a.vals.p, sizeof(double) * a.F * a.K, cudaMemcpyDeviceToDevice, ctx->stream),
               "D2D");
        if (d_words && a.F && a.wpc)
            ck(cudaMemcpyAsync(d_words, a.words.p, sizeof(uint64_t) * a.F * a.wpc, cudaMemcpyDeviceToDevice,
                               ctx->stream),
               "D2D");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int momc_b200_hypervolume(momc_ctx* ctx, const double* vals, int64_t F, int k, const double* r, double* out,
                          char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (F <= 0) usage("hypervolume of an empty archive");
        DevBuf<double> dv;
        dv.reserve(static_cast<size_t>(F) * k);
        ck(cudaMemcpyAsync(dv.p, vals, sizeof(double) * F * k, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        *out = hypervolume_device(*ctx, dv.p, F, k, std::vector<double>(r, r + k));
        dv.release();
    });
}

int momc_b200_archive_hypervolume(momc_ctx* ctx, const double* r, double* out, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        DevArchive& a = resident_archive(*ctx);
        *out = hypervolume_device(*ctx, a.vals.p, a.F, a.K, std::vector<double>(r, r + a.K));
    });
}

int momc_b200_evaluate_cuts(momc_ctx* ctx, const uint64_t* words, size_t U, double* out, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->n == 0) usage("no instance set");
        if (U == 0) return;
        upload_words(*ctx, words, U);
        DevBuf<double> d;
        d.reserve(U * ctx->k);
        evaluate_cuts_device(*ctx, ctx->d_upload.p, static_cast<long long>(U), d.p);
        ck(cudaMemcpyAsync(out, d.p, sizeof(double) * U * ctx->k, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        d.release();
    });
}

int momc_b200_reference_point_sampled(momc_ctx* ctx, int count, uint64_t seed, double* r, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->n == 0) usage("no instance set");
        const auto v = reference_point_sampled_device(*ctx, count, seed);
        std::copy(v.begin(), v.end(), r);
    });
}

int momc_b200_brute_force_pareto(momc_ctx* ctx, int64_t* out_F, double* r_exact, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->n == 0) usage("no instance set");
        std::vector<double> r;
        brute_force_device(*ctx, &r, true);
        if (r_exact) std::copy(r.begin(), r.end(), r_exact);
        if (out_F) *out_F = resident_archive(*ctx).F;
    });
}

int momc_b200_reference_point_exact(momc_ctx* ctx, double* r, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->n == 0) usage("no instance set");
        std::vector<double> v;
        brute_force_device(*ctx, &v, false);
        std::copy(v.begin(), v.end(), r);
    });
}

int momc_b200_samples_to_reach(momc_ctx* ctx, const uint64_t* words, size_t M, const double* r, double target_hv,
                               int64_t* out, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->n == 0) usage("no instance set");
        if (M == 0) usage("empty pool");
        upload_words(*ctx, words, M);
        const auto hit = samples_to_reach_device(*ctx, ctx->d_upload.p, static_cast<long long>(M),
                                                 std::vector<double>(r, r + ctx->k), target_hv);
        *out = hit ? *hit : -1;
    });
}

int momc_b200_convergence_trace(momc_ctx* ctx, const uint64_t* words, const int64_t* stamps_ns, size_t M,
                                const double* r, int checkpoints, double* elapsed_s, double* hv, int64_t* samples,
                                char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->n == 0) usage("no instance set");
        if (M == 0) usage("convergence trace needs a non-empty pool");
        if (checkpoints < 1) usage("checkpoints must be >= 1");
        upload_words(*ctx, words, M);
        std::vector<long long> smp(static_cast<size_t>(checkpoints));
        convergence_trace_device(*ctx, ctx->d_upload.p, stamps_ns, static_cast<long long>(M),
                                 std::vector<double>(r, r + ctx->k), checkpoints, elapsed_s, hv, smp.data());
        for (int i = 0; i < checkpoints; ++i) samples[i] = smp[static_cast<size_t>(i)];
    });
}

int momc_b200_format_pool_rows(momc_ctx* ctx, const uint32_t* run, const uint32_t* weight, const uint32_t* trajectory,
                               const int64_t* stamps_ns, const uint64_t* words, size_t M, int n, char* out, size_t cap,
                               size_t* out_len, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        *out_len = format_pool_rows(*ctx, run, weight, trajectory, stamps_ns, words, static_cast<long long>(M), n, out, cap);
    });
}

int momc_b200_parse_pool_rows(momc_ctx* ctx, const char* text, size_t len, int n, int first_lineno, const char* path,
                              size_t* out_M, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        *out_M = static_cast<size_t>(parse_pool_rows(*ctx, text, len, n, first_lineno, path ? path : ""));
    });
}

int momc_b200_parsed_pool_get(momc_ctx* ctx, uint32_t* run, uint32_t* weight, uint32_t* trajectory, int64_t* stamps_ns,
                              uint64_t* words, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        parsed_pool_get(*ctx, run, weight, trajectory, stamps_ns, words);
    });
}

int momc_b200_running_reset(momc_ctx* ctx, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        DevArchive& R = running_archive(*ctx);
        R.F = 0;
        ctx->running_hv_ref.clear();
    });
}

int momc_b200_stream_step(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs, long long block_begin,
                          long long block_end, int merge, const double* r, double* hv, int64_t* running_F,
                          momc_bench_report* rep, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        validate_cfg(cfg);
        if (ctx->n == 0) usage("no instance set");
        if (ctx->L < 1) usage("run_sampler needs at least one weight vector");
        momc_bench_report local{};
        momc_bench_report* rp = rep ? rep : &local;
        std::memset(rp, 0, sizeof *rp);
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        double ss = 0;
        sample(*ctx, cfg, runs, block_begin, block_end, &ss, true);
        rp->sampling_s = ss;
        rp->pool_size = ctx->pool_size;
        const auto tf = clk::now();
        const bool so = ctx->skip_order;
        ctx->skip_order = true;  // internal fronts: no archive order
        struct Restore {
            Ctx& c;
            bool v;
            ~Restore() { c.skip_order = v; }
        } restore{*ctx, so};
        if (!merge) {  // the run's front into the resident archive (unordered)
            DevArchive& a = resident_archive(*ctx);
            ParetoTimings tm;
            filter_pool_device(*ctx, ctx->d_words.p, ctx->pool_size, a, &tm);
            rp->unique_configs = tm.unique_configs;
            rp->unique_vectors = tm.unique_vectors;
            rp->archive_size = a.F;
            ck(cudaStreamSynchronize(ctx->stream), "stream front");
            rp->pareto_filtering_s = std::chrono::duration<double>(clk::now() - tf).count();
            rp->end_to_end_s = std::chrono::duration<double>(clk::now() - t0).count();
            return;
        }
        // one collapse + front over (this run's configs U the running archive)
        DevArchive& R = running_archive(*ctx);
        const long long X = R.F;
        DevBuf<double> all;
        const bool fused = filter_pool_merge_device(*ctx, ctx->d_words.p, ctx->pool_size, R.vals.p, R.words.p, X, R, all);
        R.K = ctx->k;
        R.wpc = (ctx->n + 63) / 64;
        // the fused merge recomputes the HV every step: a value-set comparison (two kernels and
        // a read-back) costs about as much as the HV, and the set changes on most steps
        const bool changed = fused || X == 0 || !same_value_set(*ctx, all.p, X, R.vals.p, R.F, ctx->k);
        all.release();
        rp->archive_size = R.F;
        if (running_F) *running_F = R.F;
        if (r && hv) {
            // the HV of an unchanged value set at the same r is the cached one
            const std::vector<double> rv(r, r + ctx->k);
            if (changed || rv != ctx->running_hv_ref) {
                ctx->running_hv = hypervolume_device(*ctx, R.vals.p, R.F, R.K, rv, true);
                ctx->running_hv_ref = rv;
            }
            *hv = ctx->running_hv;
            rp->hv = *hv;
        }
        rp->pareto_filtering_s = std::chrono::duration<double>(clk::now() - tf).count();
        rp->end_to_end_s = std::chrono::duration<double>(clk::now() - t0).count();
    });
}

int momc_b200_running_merge_values(momc_ctx* ctx, const double* d_vals, const uint64_t* d_words, int wpc, size_t M,
                                   int k, const double* r, double* hv, int64_t* running_F, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        bool changed = true;
        const long long F = running_merge(*ctx, d_vals, d_words, static_cast<long long>(M), k, wpc, &changed);
        if (running_F) *running_F = F;
        if (r && hv) {
            const std::vector<double> rv(r, r + k);
            if (changed || rv != ctx->running_hv_ref) {
                const DevArchive& R = running_archive(*ctx);
                ctx->running_hv = hypervolume_device(*ctx, R.vals.p, R.F, R.K, rv, true);
                ctx->running_hv_ref = rv;
            }
            *hv = ctx->running_hv;
        }
        ck(cudaStreamSynchronize(ctx->stream), "running merge");
    });
}

int momc_b200_archive_device_ptrs(momc_ctx* ctx, const double** vals, const uint64_t** words, int64_t* F)
{
    DevArchive& a = resident_archive(*ctx);
    *vals = a.vals.p;
    *words = a.words.p;
    *F = a.F;
    return MOMC_OK;
}

int momc_b200_running_to_archive(momc_ctx* ctx, int64_t* out_F, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        DevArchive& R = running_archive(*ctx);
        DevArchive& a = resident_archive(*ctx);
        if (R.F == 0) {
            a.F = 0;
        } else {  // ordered copy (the filter of a front is the front itself, now in archive order)
            filter_values_device(*ctx, R.vals.p, R.wpc ? R.words.p : nullptr, R.wpc, ctx->n, R.F, R.K, a, nullptr);
        }
        if (out_F) *out_F = a.F;
    });
}

int momc_b200_tc_i8_selftest(momc_ctx* ctx, const int8_t* A, const int8_t* B, int K, int32_t* D, char* err,
                             size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        tc_i8_selftest(*ctx, A, B, K, D);
    });
}

int momc_b200_philox_blocks(momc_ctx* ctx, const uint64_t* keys, const uint32_t* ctrs, size_t count, uint32_t* out,
                            char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        philox_blocks(*ctx, keys, ctrs, static_cast<long long>(count), out);
    });
}

int momc_b200_rng_calibrate(momc_ctx* ctx, int blocks_per_thread, double* normals_per_s, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (blocks_per_thread < 1) usage("blocks_per_thread must be positive");
        *normals_per_s = rng_calibrate(*ctx, blocks_per_thread);
    });
}

int momc_b200_clamp_reference(momc_ctx* ctx, double* r, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        DevArchive& a = resident_archive(*ctx);
        std::vector<double> f(static_cast<size_t>(a.F) * a.K);
        if (a.F)
            ck(cudaMemcpyAsync(f.data(), a.vals.p, sizeof(double) * f.size(), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        for (long long i = 0; i < a.F; ++i)  // clamp_reference (pareto.hpp:647-655)
            for (int l = 0; l < a.K; ++l) r[l] = std::min(r[l], f[static_cast<size_t>(i * a.K + l)]);
    });
}

namespace {
// With HV, a filter's archive order (finish_archive with order_async) runs on
// ctx.order_stream beside the reference point and HV, which read the unordered front (the same
// value set). The order is joined into ctx.stream when this leaves scope, also on error.
struct OrderJoin {
    Ctx& c;
    bool ordering = false;
    OrderJoin(Ctx& cc, bool async) : c(cc) { c.order_async = async; }
    // the values the HV reads: the unordered front while the order runs
    const double* hv_vals(const DevArchive& a)
    {
        c.order_async = false;
        ordering = c.order_pending;
        return ordering ? c.order_front : a.vals.p;
    }
    // after the HV: the archive is complete when its order is
    void complete(const DevArchive& a, const double* hv_vals, momc_bench_report* rep)
    {
        if (!ordering) return;
        ck(cudaEventSynchronize(c.ev_order_done), "archive order");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, c.ev_order_fork, c.ev_order_done), "event");
        rep->order_s = ms * 1e-3;
        if (c.grid_archive == hv_vals) c.grid_archive = a.vals.p;  // the same value set
    }
    ~OrderJoin()
    {
        c.order_async = false;
        if (c.order_pending) {
            cudaStreamWaitEvent(c.stream, c.ev_order_done, 0);
            c.order_pending = false;
        }
    }
};
}  // namespace

int momc_b200_bench(momc_ctx* ctx, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                    const momc_solver_cfg* cfg, int runs, int ref_count, const double* fixed_ref, uint64_t* out_pool,
                    momc_bench_report* rep, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (runs < 1) usage("runs must be >= 1");
        validate_cfg(cfg);
        std::memset(rep, 0, sizeof *rep);
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        set_instance(*ctx, inst);
        set_weights(*ctx, nums, L, H);
        rep->model_construction_s = std::chrono::duration<double>(clk::now() - t0).count();
        double ss = 0;
        sample(*ctx, cfg, runs, 0, -1, &ss);
        rep->sampling_s = ss;
        rep->pool_size = ctx->pool_size;
        // the pool's read-back runs on the (now idle) sampler stream's copy engine while the
        // Pareto stage reads the same words on the compute stream
        if (out_pool)
            ck(cudaMemcpyAsync(out_pool, ctx->d_words.p, sizeof(uint64_t) * ctx->pool_size * ((ctx->n + 63) / 64),
                               cudaMemcpyDeviceToHost, ctx->sample_stream),
               "D2H");
        const auto tf = clk::now();
        ParetoTimings tm;
        DevArchive& a = resident_archive(*ctx);
        OrderJoin order_join(*ctx, true);
        filter_pool_device(*ctx, ctx->d_words.p, ctx->pool_size, a, &tm);
        const double* hv_vals = order_join.hv_vals(a);
        rep->unique_configs = tm.unique_configs;
        rep->unique_vectors = tm.unique_vectors;
        rep->archive_size = a.F;
        rep->dedup_s = tm.dedup_s;
        rep->eval_s = tm.eval_s;
        rep->collapse_s = tm.collapse_s;
        rep->front_s = tm.front_s;
        rep->order_s = tm.order_s;
        rep->front_method = tm.front_method;
        rep->sampler_path = ctx->last_path;
        const auto tr = clk::now();
        std::vector<double> r(static_cast<size_t>(ctx->k));
        if (fixed_ref) {
            r.assign(fixed_ref, fixed_ref + ctx->k);
            rep->hv = hypervolume_device(*ctx, hv_vals, a.F, a.K, r, true);
        } else {
            // sampled reference clamped under the archive, kept on the device for the HV: one
            // read-back for both (reference_s is then folded into hv_s)
            rep->hv = hv_sampled_reference_device(*ctx, hv_vals, a.F, a.K, ref_count, cfg->seed, r, true);
        }
        order_join.complete(a, hv_vals, rep);
        const auto te = clk::now();
        rep->reference_s = 0;
        rep->hv_s = std::chrono::duration<double>(te - tr).count();
        for (int l = 0; l < ctx->k && l < 16; ++l) rep->reference[l] = r[static_cast<size_t>(l)];
        rep->pareto_filtering_s = std::chrono::duration<double>(te - tf).count();
        if (out_pool) ck(cudaStreamSynchronize(ctx->sample_stream), "pool read-back");
        rep->end_to_end_s = std::chrono::duration<double>(clk::now() - t0).count();
    });
}


int momc_b200_pipeline(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs, long long block_begin, long long block_end,
                       int do_hv, int ref_count, const double* fixed_ref, momc_bench_report* rep, char* err,
                       size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        validate_cfg(cfg);
        if (ctx->n == 0) usage("no instance set");
        if (ctx->L < 1) usage("run_sampler needs at least one weight vector");
        std::memset(rep, 0, sizeof *rep);
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        // model construction: re-scalarise the resident lattice (build_block_system)
        std::vector<int32_t> nums(static_cast<size_t>(ctx->L) * ctx->k);
        ck(cudaMemcpyAsync(nums.data(), ctx->d_nums.p, sizeof(int32_t) * nums.size(), cudaMemcpyDeviceToHost,
                           ctx->stream), "D2H");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        set_weights(*ctx, nums.data(), ctx->L, ctx->H);
        rep->model_construction_s = std::chrono::duration<double>(clk::now() - t0).count();
        double ss = 0;
        // compact pool: only the rows of the sampled blocks, which are all fresh
        sample(*ctx, cfg, runs, block_begin, block_end, &ss, true);
        rep->sampling_s = ss;
        const auto tf = clk::now();
        ParetoTimings tm;
        DevArchive& a = resident_archive(*ctx);
        OrderJoin order_join(*ctx, do_hv != 0);
        filter_pool_device(*ctx, ctx->d_words.p, ctx->pool_size, a, &tm);
        const double* hv_vals = order_join.hv_vals(a);
        rep->pool_size = ctx->pool_size;
        rep->unique_configs = tm.unique_configs;
        rep->unique_vectors = tm.unique_vectors;
        rep->archive_size = a.F;
        rep->dedup_s = tm.dedup_s;
        rep->eval_s = tm.eval_s;
        rep->collapse_s = tm.collapse_s;
        rep->front_s = tm.front_s;
        rep->order_s = tm.order_s;
        rep->front_method = tm.front_method;
        rep->sampler_path = ctx->last_path;
        if (do_hv) {
            const auto tr = clk::now();
            std::vector<double> r(static_cast<size_t>(ctx->k));
            if (fixed_ref) {
                r.assign(fixed_ref, fixed_ref + ctx->k);
                rep->hv = hypervolume_device(*ctx, hv_vals, a.F, a.K, r, true);
            } else {
                // sampled reference clamped under the archive, kept on the device for the HV:
                // one read-back for both (reference_s is then folded into hv_s)
                rep->hv = hv_sampled_reference_device(*ctx, hv_vals, a.F, a.K, ref_count, cfg->seed, r, true);
            }
            rep->reference_s = 0;
            rep->hv_s = std::chrono::duration<double>(clk::now() - tr).count();
            for (int l = 0; l < ctx->k && l < 16; ++l) rep->reference[l] = r[static_cast<size_t>(l)];
        }
        order_join.complete(a, hv_vals, rep);
        rep->pareto_filtering_s = std::chrono::duration<double>(clk::now() - tf).count();
        rep->end_to_end_s = std::chrono::duration<double>(clk::now() - t0).count();
    });
}

long long momc_b200_num_blocks(momc_ctx* ctx, const momc_solver_cfg* cfg, int runs)
{
    if (!ctx || !cfg || cfg->batch_size < 1 || runs < 1 || ctx->L < 1) return 0;
    bind(*ctx);
    const bool regpath = sampler_uses_register_path(ctx->n, cfg->alpha);
    const int bt = !regpath && dense_path_kind(*ctx, cfg->variant) ? dense_block_traj() : sampler_block_traj(ctx->n, cfg->alpha);
    return static_cast<long long>(runs) * ctx->L * ((cfg->batch_size + bt - 1) / bt);
}


int momc_b200_generate_uniform_instance(momc_ctx* ctx, int n, double density, int k, int kind, double lo, double hi,
                                        uint64_t seed, int64_t* out_m, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        std::vector<int> ei, ej;
        std::vector<double> w;
        generate_uniform_device(*ctx, n, density, k, kind, lo, hi, seed, ei, ej, w);
        momc_instance_view v{n, k, static_cast<int>(ei.size()), ei.data(), ej.data(), w.data()};
        set_instance(*ctx, &v);
        if (out_m) *out_m = static_cast<int64_t>(ei.size());
    });
}

int momc_b200_generate_correlated_instance(momc_ctx* ctx, int n, double density, double target_rho, uint64_t seed,
                                           int64_t* out_m, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        std::vector<int> ei, ej;
        std::vector<double> w;
        generate_correlated_device(*ctx, n, density, target_rho, seed, ei, ej, w);
        momc_instance_view v{n, 3, static_cast<int>(ei.size()), ei.data(), ej.data(), w.data()};
        set_instance(*ctx, &v);
        if (out_m) *out_m = static_cast<int64_t>(ei.size());
    });
}

int momc_b200_measured_correlation(momc_ctx* ctx, int pool_size, uint64_t seed, double* out, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        bind(*ctx);
        if (ctx->n == 0) usage("no instance set");
        *out = measured_correlation_device(*ctx, pool_size, seed);
    });
}

int momc_b200_instance_get(momc_ctx* ctx, int32_t* edge_i, int32_t* edge_j, double* w, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        std::copy(ctx->h_ei.begin(), ctx->h_ei.end(), edge_i);
        std::copy(ctx->h_ej.begin(), ctx->h_ej.end(), edge_j);
        std::copy(ctx->h_w.begin(), ctx->h_w.end(), w);
    });
}

int momc_b200_sampler_path(momc_ctx* ctx) { return ctx ? ctx->last_path : 0; }

int momc_b200_set_kernel_timing(momc_ctx* ctx, int on)
{
    if (!ctx) return MOMC_EUSAGE;
    ctx->ktimer.on = on != 0;
    return MOMC_OK;
}

int momc_b200_kernel_times(momc_ctx* ctx, double* ms, long long* counts, int reset)
{
    if (!ctx) return MOMC_EUSAGE;
    bind(*ctx);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess || cudaStreamSynchronize(ctx->sample_stream) != cudaSuccess)
        return MOMC_ERUNTIME;
    try {
        ctx->ktimer.collect();
    } catch (const std::exception&) {
        return MOMC_ERUNTIME;
    }
    for (int i = 0; i < kKClasses; ++i) {
        if (ms) ms[i] = ctx->ktimer.ms[i];
        if (counts) counts[i] = ctx->ktimer.count[i];
        if (reset) {
            ctx->ktimer.ms[i] = 0;
            ctx->ktimer.count[i] = 0;
        }
    }
    return MOMC_OK;
}

int momc_b200_set_dense_threshold(momc_ctx* ctx, int n_min)
{
    ctx->dense_min_n = n_min < 65 ? 65 : n_min;
    return MOMC_OK;
}

}  // extern "C"
