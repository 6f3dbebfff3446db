// Convergence statistics of a pool on the device:
//   samples_to_reach   pareto.hpp:763-781  first canonical-order prefix whose running archive
//                                          reaches a target HV (tolerance 1e-9 relative)
//   convergence_trace  pareto.hpp:716-757  HV of the running archive at evenly spaced
//                                          milestones of the timestamp replay order
// The reference replays record by record through archive_insert (pareto.hpp:702-710) and
// recomputes the HV after every change. The running archive after p records is the
// non-dominated set of the distinct vectors that first appeared among those p records, so
// here every distinct vector gets its first replay position f(v) (hash table, atomicMin),
// the vectors are sorted by f, and the archive of any prefix is the front of a sorted
// prefix of that list. HV(prefix) never decreases, so samples_to_reach is a binary search
// over that list; the trace evaluates each milestone's prefix. Fronts and HVs use the same
// device filter / exact hypervolume as everything else, so values are bit-identical.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <optional>
#include <vector>

#include "ctx.cuh"
#include "pareto.cuh"

namespace momc_b200 {

namespace {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;

unsigned grid_for(long long n, int t = 256)
{
    long long b = (n + t - 1) / t;
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>(b, 148ll * 32)));
}

__device__ __forceinline__ uint64_t vhash(const double* v, int K)
{
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (int l = 0; l < K; ++l) {
        uint64_t b = static_cast<uint64_t>(__double_as_longlong(v[l] == 0.0 ? 0.0 : v[l]));  // -0 == +0
        h ^= b + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xBF58476D1CE4E5B9ull;
    }
    return h ^ (h >> 31);
}

// slot of each row's vector in an open-addressed table (first inserter owns the slot);
// minpos[slot] = min over rows with that vector of pos[row]
__global__ void k_first_pos(const double* __restrict__ vals, long long M, int K, const uint32_t* __restrict__ pos,
                            uint32_t* table, uint32_t* minpos, uint64_t mask)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < M;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double* v = vals + i * K;
        uint64_t s = vhash(v, K) & mask;
        for (;;) {
            uint32_t cur = table[s];
            if (cur == kEmpty) {
                cur = atomicCAS(&table[s], kEmpty, static_cast<uint32_t>(i));
                if (cur == kEmpty) cur = static_cast<uint32_t>(i);
            }
            const double* u = vals + static_cast<long long>(cur) * K;
            bool eq = true;
            for (int l = 0; l < K; ++l) eq &= u[l] == v[l];
            if (eq) {
                atomicMin(&minpos[s], pos ? pos[i] : static_cast<uint32_t>(i));
                break;
            }
            s = (s + 1) & mask;
        }
    }
}

// occupied slots -> (first position, owner row)
__global__ void k_slots(const uint32_t* __restrict__ table, const uint32_t* __restrict__ minpos, uint64_t size,
                        uint32_t* keys, uint32_t* rows, unsigned long long* count)
{
    for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < size;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (table[s] == kEmpty) continue;
        const unsigned long long q = atomicAdd(count, 1ull);
        keys[q] = minpos[s];
        rows[q] = table[s];
    }
}

__global__ void k_gather(const double* __restrict__ vals, const uint32_t* __restrict__ rows, long long V, int K,
                         double* out)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V * K;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = vals[static_cast<long long>(rows[i / K]) * K + i % K];
}

__global__ void k_iota(uint32_t* a, long long n)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        a[i] = static_cast<uint32_t>(i);
}

__global__ void k_scatter_rank(const uint32_t* __restrict__ order, long long n, uint32_t* rank)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        rank[order[i]] = static_cast<uint32_t>(i);
}

// Distinct vectors of the M configs on the device, sorted by first replay position.
struct FirstSeen {
    long long V = 0;
    std::vector<uint32_t> first;  // host copy of the sorted first positions
    DevBuf<double> vals;          // V x K, in that order
};

void first_seen(Ctx& c, const uint64_t* d_words, long long M, const uint32_t* d_pos, FirstSeen& fs)
{
    const int K = c.k;
    DevBuf<double> v;
    v.reserve(static_cast<size_t>(M) * K);
    evaluate_cuts_device(c, d_words, M, v.p);
    uint64_t size = 1;
    while (size < 2ull * static_cast<uint64_t>(M) + 16) size <<= 1;
    DevBuf<uint32_t> table, minpos, keys, rows, keys2, rows2;
    DevBuf<unsigned long long> cnt;
    table.reserve(size);
    minpos.reserve(size);
    cnt.reserve(1);
    ck(cudaMemsetAsync(table.p, 0xFF, sizeof(uint32_t) * size, c.stream), "memset");
    ck(cudaMemsetAsync(minpos.p, 0xFF, sizeof(uint32_t) * size, c.stream), "memset");
    ck(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), c.stream), "memset");
    k_first_pos<<<grid_for(M), 256, 0, c.stream>>>(v.p, M, K, d_pos, table.p, minpos.p, size - 1);
    keys.reserve(static_cast<size_t>(M));
    rows.reserve(static_cast<size_t>(M));
    k_slots<<<grid_for(static_cast<long long>(size)), 256, 0, c.stream>>>(table.p, minpos.p, size, keys.p, rows.p,
                                                                         cnt.p);
    c.launches += 2;
    unsigned long long V = 0;
    ck(cudaMemcpyAsync(&V, cnt.p, sizeof V, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "first positions");
    // sort by first position (unique per vector: two vectors cannot first appear at one record)
    keys2.reserve(static_cast<size_t>(V));
    rows2.reserve(static_cast<size_t>(V));
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys2.p, rows.p, rows2.p, static_cast<int>(V), 0, 32,
                                    c.stream);
    DevBuf<unsigned char> tmp;
    tmp.reserve(tb + 1);
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys2.p, rows.p, rows2.p, static_cast<int>(V), 0, 32,
                                       c.stream),
       "sort");
    fs.V = static_cast<long long>(V);
    fs.vals.reserve(static_cast<size_t>(V) * K + 1);
    k_gather<<<grid_for(static_cast<long long>(V) * K), 256, 0, c.stream>>>(v.p, rows2.p, static_cast<long long>(V), K,
                                                                            fs.vals.p);
    c.launches += 2;
    fs.first.resize(V);
    ck(cudaMemcpyAsync(fs.first.data(), keys2.p, sizeof(uint32_t) * V, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "first positions");
    for (auto* b : {&table, &minpos, &keys, &rows, &keys2, &rows2}) b->release();
    cnt.release();
    tmp.release();
    v.release();
}

// HV of the front of the first j sorted vectors
double prefix_hv(Ctx& c, const FirstSeen& fs, long long j, const std::vector<double>& r, DevArchive& tmp)
{
    filter_values_device(c, fs.vals.p, nullptr, 0, 0, j, c.k, tmp, nullptr);
    return hypervolume_device(c, tmp.vals.p, tmp.F, c.k, r);
}

}  // namespace

// samples_to_reach (pareto.hpp:763-781) over M configs on the device: nullopt when never reached
std::optional<long long> samples_to_reach_device(Ctx& c, const uint64_t* d_words, long long M,
                                                 const std::vector<double>& r, double target)
{
    if (M <= 0) usage("empty pool");
    if (M >= 0xFFFFFFFFll) usage("pool too large for one device pass (shard it)");
    FirstSeen fs;
    first_seen(c, d_words, M, nullptr, fs);
    const double tol = 1e-9 * std::max(1.0, std::abs(target));
    DevArchive tmp;
    // smallest j with HV(front(first j)) >= target - tol; HV is monotone in j
    long long lo = 1, hi = fs.V;
    std::optional<long long> ans;
    if (prefix_hv(c, fs, hi, r, tmp) >= target - tol) {
        while (lo < hi) {
            const long long mid = lo + (hi - lo) / 2;
            if (prefix_hv(c, fs, mid, r, tmp) >= target - tol) hi = mid;
            else lo = mid + 1;
        }
        ans = static_cast<long long>(fs.first[static_cast<size_t>(lo - 1)]) + 1;
    }
    tmp.vals.release();
    tmp.words.release();
    fs.vals.release();
    return ans;
}

// convergence_trace (pareto.hpp:716-757): stamps[i] = record i's timestamp_ns; outputs
// `checkpoints` points (elapsed_s, hv, samples)
void convergence_trace_device(Ctx& c, const uint64_t* d_words, const int64_t* h_stamps, long long M,
                              const std::vector<double>& r, int checkpoints, double* elapsed, double* hv,
                              long long* samples)
{
    if (M <= 0) usage("convergence trace needs a non-empty pool");
    if (checkpoints < 1) usage("checkpoints must be >= 1");
    if (M >= 0xFFFFFFFFll) usage("pool too large for one device pass (shard it)");
    // replay order: stable sort by timestamp (pareto.hpp:691-699)
    DevBuf<long long> ts, ts2;
    DevBuf<uint32_t> idx, order, rank;
    ts.reserve(static_cast<size_t>(M));
    ts2.reserve(static_cast<size_t>(M));
    idx.reserve(static_cast<size_t>(M));
    order.reserve(static_cast<size_t>(M));
    rank.reserve(static_cast<size_t>(M));
    k_iota<<<grid_for(M), 256, 0, c.stream>>>(idx.p, M);
    // signed keys: flip the sign bit so the unsigned radix order is the signed order
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, reinterpret_cast<const unsigned long long*>(ts.p),
                                    reinterpret_cast<unsigned long long*>(ts2.p), idx.p, order.p, static_cast<int>(M), 0,
                                    64, c.stream);
    DevBuf<unsigned char> tmpb;
    tmpb.reserve(tb + 1);
    {
        std::vector<long long> flipped(static_cast<size_t>(M));
        for (long long i = 0; i < M; ++i)
            flipped[static_cast<size_t>(i)] =
                static_cast<long long>(static_cast<unsigned long long>(h_stamps[i]) ^ 0x8000000000000000ull);
        ck(cudaMemcpyAsync(ts.p, flipped.data(), sizeof(long long) * M, cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cub::DeviceRadixSort::SortPairs(tmpb.p, tb, reinterpret_cast<const unsigned long long*>(ts.p),
                                           reinterpret_cast<unsigned long long*>(ts2.p), idx.p, order.p,
                                           static_cast<int>(M), 0, 64, c.stream),
           "sort");
        ck(cudaStreamSynchronize(c.stream), "sort");
    }
    k_scatter_rank<<<grid_for(M), 256, 0, c.stream>>>(order.p, M, rank.p);
    c.launches += 2;
    std::vector<uint32_t> h_order(static_cast<size_t>(M));
    ck(cudaMemcpyAsync(h_order.data(), order.p, sizeof(uint32_t) * M, cudaMemcpyDeviceToHost, c.stream), "D2H");
    FirstSeen fs;
    first_seen(c, d_words, M, rank.p, fs);
    DevArchive tmp;
    double hv_cache = 0;
    long long j_cache = -1;
    for (int i = 0; i < checkpoints; ++i) {
        const long long m = std::max<long long>(
            1, std::llround(static_cast<double>(M) * static_cast<double>(i + 1) / static_cast<double>(checkpoints)));
        // vectors first seen at replay positions < m
        const long long j = std::lower_bound(fs.first.begin(), fs.first.end(), static_cast<uint32_t>(m)) - fs.first.begin();
        if (j != j_cache) {
            hv_cache = prefix_hv(c, fs, j, r, tmp);
            j_cache = j;
        }
        elapsed[i] = static_cast<double>(h_stamps[h_order[static_cast<size_t>(m - 1)]]) * 1e-9;
        hv[i] = hv_cache;
        samples[i] = m;
    }
    for (auto* b : {&idx, &order, &rank}) b->release();
    ts.release();
    ts2.release();
    tmpb.release();
    tmp.vals.release();
    tmp.words.release();
    fs.vals.release();
}

}  // namespace momc_b200
