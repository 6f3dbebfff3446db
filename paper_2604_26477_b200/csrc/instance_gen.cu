// generate_uniform_instance (instance.hpp:259-284) on the device: every vertex pair (i, j)
// draws its presence from Stream(key, i, j, tag_word(edge_presence)) and, if present, K
// weights from Stream(key, i, j, tag_word(edge_weight)) via WeightSpec::draw
// (instance.hpp:230-237), key = derive_key(seed, 0x696E7374). Edges are emitted in (i, j)
// order, exactly as the reference's nested loop. Used for the C4 N=2000 instance
// (1,999,000 pairs), whose host generation dominates the reference's model construction.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "rng.cuh"

namespace momc_b200 {

namespace {

__device__ __forceinline__ uint64_t pair_offset(int n, int i) { return static_cast<uint64_t>(i) * n - static_cast<uint64_t>(i) * (i + 1) / 2; }

// row i per blockIdx.y; columns j > i over blockIdx.x * blockDim.x + threadIdx.x
__global__ void k_presence(int n, double density, uint64_t key, unsigned char* flag, int* row_count)
{
    const int i = blockIdx.y;
    const int j = i + 1 + blockIdx.x * blockDim.x + threadIdx.x;
    bool present = false;
    if (j < n) {
        DevStream s;
        s.init(key, static_cast<uint32_t>(i), static_cast<uint32_t>(j), tag_word(kTagEdgePresence, 0));
        const double u = static_cast<double>(s.next_u64() >> 11) * 0x1.0p-53;  // next_u01 (rng.hpp:131-134)
        present = !(u >= density);
        flag[pair_offset(n, i) + (j - i - 1)] = present;
    }
    const int c = __syncthreads_count(present);
    if (threadIdx.x == 0 && c) atomicAdd(&row_count[i], c);
}

// ordered compaction of row i (one CTA per row) + weight draws
__global__ void k_emit(int n, int k, int kind, double lo, double hi, uint64_t key, const unsigned char* flag,
                       const long long* row_start, int* ei, int* ej, double* w)
{
    const int i = blockIdx.x;
    const uint64_t base = pair_offset(n, i);
    const int len = n - i - 1;
    __shared__ int warp_sum[32];
    long long out = row_start[i];
    for (int j0 = 0; j0 < len; j0 += blockDim.x) {
        const int jj = j0 + threadIdx.x;
        const bool p = jj < len && flag[base + jj];
        const unsigned b = __ballot_sync(0xffffffffu, p);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0) warp_sum[wid] = __popc(b);
        __syncthreads();
        int before = 0, total = 0;
        for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
            if (q < wid) before += warp_sum[q];
            total += warp_sum[q];
        }
        if (p) {
            const long long e = out + before + __popc(b & ((1u << lane) - 1));
            const int j = i + 1 + jj;
            ei[e] = i;
            ej[e] = j;
            DevStream s;
            s.init(key, static_cast<uint32_t>(i), static_cast<uint32_t>(j), tag_word(kTagEdgeWeight, 0));
            for (int q = 0; q < k; ++q) {
                double v;
                if (kind == 0) {  // uniform_int: lo + next_below(hi - lo + 1)
                    const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
                    v = lo + static_cast<double>(__umul64hi(s.next_u64(), span));
                } else {  // uniform_real: lo + (hi - lo) * next_u01_open()
                    const double u = static_cast<double>((s.next_u64() >> 11) + 1) * 0x1.0p-53;
                    v = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
                }
                w[e * k + q] = v;
            }
        }
        out += total;
        __syncthreads();
    }
}

// correlation_noise normal of every edge (instance.hpp:380-386)
__global__ void k_edge_noise(const int* __restrict__ ei, const int* __restrict__ ej, int m, uint64_t key,
                             const ZigTables* __restrict__ z, double* noise)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    DevStream s;
    s.init(key, static_cast<uint32_t>(ei[e]), static_cast<uint32_t>(ej[e]), tag_word(kTagCorrelationNoise, 0));
    noise[e] = normal_seq(s, z);
}

// probe_pool config c (instance.hpp:315-331) as packed words: bit i set iff s_i = +1
__device__ __forceinline__ void probe_words(uint64_t key, int c, int n, uint64_t* w)
{
    DevStream s;
    s.init(key, static_cast<uint32_t>(c), 0, tag_word(kTagProbePool, 0));
    for (int i = 0; i < n; i += 64) w[i / 64] = s.next_u64();
}

__device__ __forceinline__ bool cut_edge(const uint64_t* w, int i, int j)
{
    return ((w[i >> 6] >> (i & 63)) ^ (w[j >> 6] >> (j & 63))) & 1ull;
}

constexpr int kMaxProbeN = 4096;

// x_c = sum over cut edges of (w1 + w2), b_c = sum over cut edges of noise, in edge order
// (instance.hpp:392-402); one thread per probe configuration
__global__ void k_probe_xb(const int* __restrict__ ei, const int* __restrict__ ej, const double* __restrict__ w2, int m,
                           const double* __restrict__ noise, int n, int pool, uint64_t key, double* x, double* b)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= pool) return;
    uint64_t w[kMaxProbeN / 64];
    probe_words(key, c, n, w);
    double xc = 0, bc = 0;
    for (int e = 0; e < m; ++e) {
        if (cut_edge(w, ei[e], ej[e])) {
            xc = __dadd_rn(xc, __dadd_rn(w2[2 * e], w2[2 * e + 1]));
            bc = __dadd_rn(bc, noise[e]);
        }
    }
    x[c] = xc;
    b[c] = bc;
}

// measured_correlation's samples (instance.hpp:338-357): x = C_1 + C_2, y = C_3 with
// cut_values (instance.hpp:183-207, per-layer sums in edge order)
__global__ void k_probe_cuts(const int* __restrict__ ei, const int* __restrict__ ej, const double* __restrict__ w3, int m,
                             int n, int pool, uint64_t key, double* x, double* y)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= pool) return;
    uint64_t w[kMaxProbeN / 64];
    probe_words(key, c, n, w);
    double c0 = 0, c1 = 0, c2 = 0;
    for (int e = 0; e < m; ++e) {
        if (cut_edge(w, ei[e], ej[e])) {
            c0 = __dadd_rn(c0, w3[3 * e]);
            c1 = __dadd_rn(c1, w3[3 * e + 1]);
            c2 = __dadd_rn(c2, w3[3 * e + 2]);
        }
    }
    x[c] = __dadd_rn(c0, c1);
    y[c] = c2;
}

}  // namespace

// generate_correlated_instance (instance.hpp:364-458): the uniform base, the per-edge
// noise and the probe-pool sums on the device; the closed-form bisection for sigma on the
// host (a few hundred scalar steps, same expressions as the reference).
void generate_correlated_device(Ctx& c, int n, double density, double target_rho, uint64_t seed, std::vector<int>& ei,
                                std::vector<int>& ej, std::vector<double>& w)
{
    if (n < 4) usage("vertex count must be at least 4");
    if (!(density > 0.0) || density > 1.0) usage("density must lie in (0, 1]");
    if (!(target_rho > -1.0) || !(target_rho < 0.0)) usage("target correlation must lie in (-1, 0)");
    if (n > kMaxProbeN) usage("correlated generation on the device supports n <= 4096");
    std::vector<double> w2;
    generate_uniform_device(c, n, density, 2, 0, 1.0, 10.0, seed, ei, ej, w2);  // WeightSpec{} = U{1..10}
    const uint64_t key = derive_key(seed, 0x696E7374u);
    const int m = static_cast<int>(ei.size());
    if (m < 2) runtime("correlated generation failed: too few edges");
    constexpr int kPool = 2048;       // kCorrelationPoolSize
    constexpr double kLambda = 0.5;   // kCorrelationLambda
    DevBuf<int> dei, dej;
    DevBuf<double> dw, dnoise, dx, db;
    dei.reserve(static_cast<size_t>(m));
    dej.reserve(static_cast<size_t>(m));
    dw.reserve(static_cast<size_t>(m) * 2);
    dnoise.reserve(static_cast<size_t>(m));
    dx.reserve(kPool);
    db.reserve(kPool);
    ck(cudaMemcpyAsync(dei.p, ei.data(), sizeof(int) * m, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(dej.p, ej.data(), sizeof(int) * m, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(dw.p, w2.data(), sizeof(double) * m * 2, cudaMemcpyHostToDevice, c.stream), "H2D");
    const ZigTables* z = device_zig(c);
    k_edge_noise<<<(m + 127) / 128, 128, 0, c.stream>>>(dei.p, dej.p, m, key, z, dnoise.p);
    k_probe_xb<<<(kPool + 63) / 64, 64, 0, c.stream>>>(dei.p, dej.p, dw.p, m, dnoise.p, n, kPool, key, dx.p, db.p);
    c.launches += 2;
    std::vector<double> noise(static_cast<size_t>(m)), x(kPool), b(kPool);
    ck(cudaMemcpyAsync(noise.data(), dnoise.p, sizeof(double) * m, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(x.data(), dx.p, sizeof(double) * kPool, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(b.data(), db.p, sizeof(double) * kPool, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "correlated generator");
    for (auto* q : {&dei, &dej}) q->release();
    for (auto* q : {&dw, &dnoise, &dx, &db}) q->release();

    const double np = static_cast<double>(kPool);
    double mx = 0, mb = 0;
    for (int q = 0; q < kPool; ++q) {
        mx += x[static_cast<size_t>(q)];
        mb += b[static_cast<size_t>(q)];
    }
    mx /= np;
    mb /= np;
    double vx = 0, vb = 0, cxb = 0;
    for (int q = 0; q < kPool; ++q) {
        const double dx2 = x[static_cast<size_t>(q)] - mx;
        const double db2 = b[static_cast<size_t>(q)] - mb;
        vx += dx2 * dx2;
        vb += db2 * db2;
        cxb += dx2 * db2;
    }
    if (vx <= 0 || vb <= 0) runtime("correlated generation failed: degenerate probe pool");
    const double lambda = kLambda;
    const auto rho_of = [&](double sigma) {
        const double cov = -lambda * vx + sigma * cxb;
        const double vy = lambda * lambda * vx - 2.0 * lambda * sigma * cxb + sigma * sigma * vb;
        return cov / std::sqrt(vx * vy);
    };
    double lo = 0.0, hi = 1.0;
    int doublings = 0;
    while (rho_of(hi) < target_rho) {
        hi *= 2.0;
        if (++doublings > 200)
            runtime("correlated generation failed to bracket target rho; achieved " + std::to_string(rho_of(hi)));
    }
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        (rho_of(mid) < target_rho ? lo : hi) = mid;
    }
    const double sigma = 0.5 * (lo + hi);
    const double achieved = rho_of(sigma);
    if (std::abs(achieved - target_rho) > 0.005)
        runtime("correlated generation failed to reach target rho; achieved " + std::to_string(achieved));
    w.resize(static_cast<size_t>(m) * 3);
    for (int e = 0; e < m; ++e) {
        const double a = w2[static_cast<size_t>(e) * 2], bb = w2[static_cast<size_t>(e) * 2 + 1];
        w[static_cast<size_t>(e) * 3] = a;
        w[static_cast<size_t>(e) * 3 + 1] = bb;
        w[static_cast<size_t>(e) * 3 + 2] = -lambda * (a + bb) + sigma * noise[static_cast<size_t>(e)];
    }
}

// measured_correlation (instance.hpp:338-357) of the resident K=3 instance
double measured_correlation_device(Ctx& c, int pool_size, uint64_t seed)
{
    if (c.k != 3) usage("correlation measure requires K=3");
    if (c.n > kMaxProbeN) usage("correlation measure on the device supports n <= 4096");
    if (pool_size < 2) usage("pearson requires two samples of equal size >= 2");
    const uint64_t key = derive_key(seed, 0x696E7374u);
    DevBuf<double> dx, dy;
    dx.reserve(static_cast<size_t>(pool_size));
    dy.reserve(static_cast<size_t>(pool_size));
    k_probe_cuts<<<(pool_size + 63) / 64, 64, 0, c.stream>>>(c.d_ei.p, c.d_ej.p, c.d_w.p, c.m, c.n, pool_size, key,
                                                             dx.p, dy.p);
    c.launches++;
    std::vector<double> x(static_cast<size_t>(pool_size)), y(static_cast<size_t>(pool_size));
    ck(cudaMemcpyAsync(x.data(), dx.p, sizeof(double) * pool_size, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(y.data(), dy.p, sizeof(double) * pool_size, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "measured correlation");
    dx.release();
    dy.release();
    // pearson (instance.hpp:286-310)
    const double nn = static_cast<double>(pool_size);
    double mx = 0, my = 0;
    for (int i = 0; i < pool_size; ++i) {
        mx += x[static_cast<size_t>(i)];
        my += y[static_cast<size_t>(i)];
    }
    mx /= nn;
    my /= nn;
    double sxx = 0, syy = 0, sxy = 0;
    for (int i = 0; i < pool_size; ++i) {
        const double dx2 = x[static_cast<size_t>(i)] - mx;
        const double dy2 = y[static_cast<size_t>(i)] - my;
        sxx += dx2 * dx2;
        syy += dy2 * dy2;
        sxy += dx2 * dy2;
    }
    if (sxx <= 0 || syy <= 0) usage("pearson undefined for zero-variance sample");
    return sxy / std::sqrt(sxx * syy);
}

// Generates the instance on the device and returns it on the host (edge arrays).
void generate_uniform_device(Ctx& c, int n, double density, int k, int kind, double lo, double hi, uint64_t seed,
                             std::vector<int>& ei, std::vector<int>& ej, std::vector<double>& w)
{
    if (n < 2) usage("vertex count must be at least 2");
    if (!(density > 0.0) || density > 1.0) usage("density must lie in (0, 1]");
    if (k < 2) usage("objective count must be at least 2");
    if (kind == 0 && lo > hi) usage("empty integer weight range");
    if (kind != 0 && !(lo < hi)) usage("empty real weight range");
    const uint64_t key = derive_key(seed, 0x696E7374u);
    const long long pairs = static_cast<long long>(n) * (n - 1) / 2;
    DevBuf<unsigned char> flag;
    flag.reserve(static_cast<size_t>(pairs) + 1);
    DevBuf<int> rc;
    rc.reserve(static_cast<size_t>(n));
    ck(cudaMemsetAsync(rc.p, 0, sizeof(int) * n, c.stream), "memset");
    const int T = 256;
    k_presence<<<dim3(static_cast<unsigned>((n + T - 1) / T), static_cast<unsigned>(n)), T, 0, c.stream>>>(
        n, density, key, flag.p, rc.p);
    c.launches++;
    std::vector<int> counts(static_cast<size_t>(n));
    ck(cudaMemcpyAsync(counts.data(), rc.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "presence");
    std::vector<long long> start(static_cast<size_t>(n) + 1, 0);
    for (int i = 0; i < n; ++i) start[static_cast<size_t>(i) + 1] = start[static_cast<size_t>(i)] + counts[static_cast<size_t>(i)];
    const long long m = start[static_cast<size_t>(n)];
    if (m > 0x7FFFFFFFll) usage("too many edges");
    DevBuf<long long> dstart;
    dstart.reserve(static_cast<size_t>(n) + 1);
    DevBuf<int> dei, dej;
    DevBuf<double> dw;
    dei.reserve(static_cast<size_t>(m) + 1);
    dej.reserve(static_cast<size_t>(m) + 1);
    dw.reserve(static_cast<size_t>(m) * k + 1);
    ck(cudaMemcpyAsync(dstart.p, start.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, c.stream), "H2D");
    k_emit<<<n, T, 0, c.stream>>>(n, k, kind, lo, hi, key, flag.p, dstart.p, dei.p, dej.p, dw.p);
    c.launches++;
    ei.resize(static_cast<size_t>(m));
    ej.resize(static_cast<size_t>(m));
    w.resize(static_cast<size_t>(m) * k);
    ck(cudaMemcpyAsync(ei.data(), dei.p, sizeof(int) * m, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(ej.data(), dej.p, sizeof(int) * m, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(w.data(), dw.p, sizeof(double) * m * k, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "emit");
    for (auto* b : {&flag}) b->release();
    rc.release();
    dstart.release();
    dei.release();
    dej.release();
    dw.release();
}

}  // namespace momc_b200
