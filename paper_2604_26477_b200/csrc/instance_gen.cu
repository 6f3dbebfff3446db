// generate_uniform_instance (instance.hpp:259-284) on the device: every vertex pair (i, j)
// draws its presence from Stream(key, i, j, tag_word(edge_presence)) and, if present, K
// weights from Stream(key, i, j, tag_word(edge_weight)) via WeightSpec::draw
// (instance.hpp:230-237), key = derive_key(seed, 0x696E7374). Edges are emitted in (i, j)
// order, exactly as the reference's nested loop. Used for the C4 N=2000 instance
// (1,999,000 pairs), whose host generation dominates the reference's model construction.
#include <cuda_runtime.h>

#include <cstdint>
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

}  // namespace

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
