// Pareto stage kernels (pareto.cuh). Design:
//   K5 dedup      open-addressing hash set over packed configs (warp-aggregated compaction)
//   K4 eval       exact int32 edge loop when all weights are integral (every partial sum is
//                 an integer < 2^31, so it equals evaluate_cuts' FP64 GEMM result exactly);
//                 otherwise the shim's FP64 order of evaluate_cuts (pareto.hpp:346-359)
//   K6 collapse   hash map keyed by the objective vector; the owner is the lexicographically
//                 smallest spin configuration (instance.hpp:63-67), kept by a CAS loop
//   K7 front      "grid" method: coordinates compressed to ranks; a (K-1)-d table holds,
//                 per cell, the max last-coordinate rank; a suffix max along every axis then
//                 decides weak dominance of every vector in O(1) (exact, order-free);
//                 all-pairs fallback when the compressed grid would not fit
//   archive       rank sort, lexicographically descending (pareto.hpp:405-406)
//   K8 HV         the same compressed grid over the front: HV = sum over cells of
//                 (cell volume) x (max covering gain), accumulated exactly in __int128 when
//                 the values are integers (bit-equal to the reference's exact double result)
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "pareto.cuh"
#include "rng.cuh"

namespace momc_b200 {

namespace {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr int kMaxK = 16;
constexpr long long kGridCap = 1ll << 27;  // max cells of a compressed grid table
constexpr int kDistinctCap = 1 << 15;      // max distinct values per axis for the grid method

__device__ __forceinline__ uint64_t hash_words(const uint64_t* w, int wpc)
{  // WordSpanHash-like mixing (pareto.hpp:297-306), any good mixer works here
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (int i = 0; i < wpc; ++i) h ^= mix64(w[i] + h);
    return h;
}

// order-preserving key of a double (-0.0 canonicalised to +0.0); 0 is below every value
__host__ __device__ __forceinline__ uint64_t dkey(double v)
{
    v = v + 0.0;
    uint64_t b;
#ifdef __CUDA_ARCH__
    b = static_cast<uint64_t>(__double_as_longlong(v));
#else
    std::memcpy(&b, &v, 8);
#endif
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ uint64_t hash_vals(const double* v, int K)
{
    uint64_t h = 0x243F6A8885A308D3ull;
    for (int k = 0; k < K; ++k) h ^= mix64(dkey(v[k]) + h);
    return h;
}

__device__ __forceinline__ bool vals_equal(const double* a, const double* b, int K)
{
    for (int k = 0; k < K; ++k)
        if (!(a[k] == b[k])) return false;
    return true;
}

// SpinConfiguration operator< (instance.hpp:63-67): spins compared from index 0 with
// -1 < +1; for packed words that is numeric order of the bit-reversed words, word 0 first.
__device__ __forceinline__ bool config_less(const uint64_t* a, const uint64_t* b, int wpc)
{
    for (int i = 0; i < wpc; ++i) {
        const uint64_t x = __brevll(a[i]), y = __brevll(b[i]);
        if (x != y) return x < y;
    }
    return false;
}

__device__ __forceinline__ void warp_append(bool flag, uint32_t value, uint32_t* out, unsigned long long* count)
{
    const unsigned mask = __activemask();
    const unsigned b = __ballot_sync(mask, flag);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(b) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(count, static_cast<unsigned long long>(__popc(b)));
    base = __shfl_sync(mask, base, leader);
    if (flag) out[base + __popc(b & ((1u << lane) - 1))] = value;
}

// warp_append through a per-warp shared-memory buffer of CAP entries: one atomicAdd on the
// global count per flush instead of one per warp and iteration (a single counter taking
// millions of adds is serialised in L2: C5's 6.6e6 distinct configs). Every lane of the warp
// calls push (block-uniform loops) and flush once after the loop. Entries at or past `limit`
// raise *overflow instead of being stored.
template <int CAP>
struct WarpBuffer {
    uint32_t* buf;  // this warp's CAP entries
    int n;          // warp-uniform fill
    __device__ __forceinline__ void flush(uint32_t* out, unsigned long long* count, unsigned long long limit,
                                          unsigned long long* overflow)
    {
        __syncwarp();
        const int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == 0 && n) base = atomicAdd(count, static_cast<unsigned long long>(n));
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int j = lane; j < n; j += 32) {
            if (base + j < limit) out[base + j] = buf[j];
            else atomicExch(overflow, 1ull);
        }
        __syncwarp();
        n = 0;
    }
    __device__ __forceinline__ void push(bool flag, uint32_t v, uint32_t* out, unsigned long long* count,
                                         unsigned long long limit, unsigned long long* overflow)
    {
        const unsigned b = __ballot_sync(0xffffffffu, flag);
        const int nf = __popc(b);
        if (n + nf > CAP) flush(out, count, limit, overflow);
        if (flag) buf[n + __popc(b & ((1u << (threadIdx.x & 31)) - 1))] = v;
        n += nf;
    }
};
constexpr int kWBuf = 128;

// warp_append that returns each flagged lane's slot (undefined for the others)
__device__ __forceinline__ unsigned long long warp_append_index(bool flag, unsigned long long* count)
{
    const unsigned mask = __activemask();
    const unsigned b = __ballot_sync(mask, flag);
    if (!b) return 0;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(b) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(count, static_cast<unsigned long long>(__popc(b)));
    base = __shfl_sync(mask, base, leader);
    return base + __popc(b & ((1u << lane) - 1));
}

// ---- K5+K4+K6 fused, one word per config, n <= 63, integer weights (the C1 / C2 pools):
// dedup on the config words themselves (64-bit keys, empty = ~0, which no n <= 63 config
// equals), the cut values of each fresh config (exact int32, instance.hpp:183-194) evaluated
// by the thread that inserted it, then the value vector collapsed (table of rows into vals,
// pareto.hpp:383-387) with the lexicographically smallest config kept by a 64-bit atomicMin
// on the bit-reversed word (config_less order). Counts in cnt[0] (unique configs) and cnt[2]
// (distinct vectors); reps lists the distinct vectors' slots. The vals row is written and
// fenced before it is published in t2; readers go through L2 (__ldcg).
// shared-memory edge table of the fused kernel: per edge one int (ei | ej << 16) and KM
// weights (KM = 2, 4, 8 or 16 >= K, padded with zeros; 16-byte rows for KM >= 4)
template <int KM>
__device__ __forceinline__ void cut_values_int(uint64_t w, int m, const int* __restrict__ epair,
                                               const int* __restrict__ ew, int (&acc)[KM])
{
#pragma unroll
    for (int k = 0; k < KM; ++k) acc[k] = 0;
    for (int e = 0; e < m; ++e) {
        const int pr = epair[e];
        const uint64_t d = (w >> (pr & 0xFFFF)) ^ (w >> (pr >> 16));
        const int cut = -static_cast<int>(d & 1ull);
        if constexpr (KM >= 4) {
#pragma unroll
            for (int k = 0; k < KM; k += 4) {
                const int4 q = *reinterpret_cast<const int4*>(ew + e * KM + k);
                acc[k] += q.x & cut;
                acc[k + 1] += q.y & cut;
                acc[k + 2] += q.z & cut;
                acc[k + 3] += q.w & cut;
            }
        } else {
#pragma unroll
            for (int k = 0; k < KM; ++k) acc[k] += ew[e * KM + k] & cut;
        }
    }
}

template <int KM>
__global__ void __launch_bounds__(256) k_dedup_eval_collapse(
    const uint64_t* __restrict__ words, long long M, int m, int K, const int* __restrict__ ei,
    const int* __restrict__ ej, const int* __restrict__ wi, unsigned long long* t1, uint64_t m1, uint32_t* t2,
    unsigned long long* own, uint64_t m2, double* vals, uint32_t* reps, unsigned long long* cnt)
{
    extern __shared__ __align__(16) int sm[];  // weights (m x KM) | edge pairs (m)
    int* ew = sm;
    int* epair = sm + m * KM;
    for (int e = threadIdx.x; e < m; e += blockDim.x) epair[e] = ei[e] | (ej[e] << 16);
    for (int q = threadIdx.x; q < m * KM; q += blockDim.x) {
        const int e = q / KM, k = q % KM;
        ew[q] = k < K ? wi[e * K + k] : 0;
    }
    __syncthreads();
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < M;
         i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        bool fresh = false;
        uint64_t w = i < M ? words[i] : ~0ull;
        // lanes holding the same word (neighbouring trajectories often converge to the same
        // configuration): only the lowest of them probes the table
        const unsigned same = __match_any_sync(0xffffffffu, w);
        if (i < M && (threadIdx.x & 31) == __ffs(same) - 1) {
            uint64_t h = mix64(w) & m1;
            for (;;) {
                const unsigned long long old = atomicCAS(&t1[h], ~0ull, static_cast<unsigned long long>(w));
                if (old == ~0ull) {
                    fresh = true;
                    break;
                }
                if (old == w) break;
                h = (h + 1) & m1;
            }
        }
        const unsigned long long u = warp_append_index(fresh, cnt);
        bool vfresh = false;
        uint32_t slot = 0;
        if (fresh) {
            int acc[KM];
            cut_values_int<KM>(w, m, epair, ew, acc);
            double v[KM];
#pragma unroll
            for (int k = 0; k < KM; ++k)
                if (k < K) {
                    v[k] = static_cast<double>(acc[k]);
                    vals[u * K + k] = v[k];
                }
            __threadfence();
            uint64_t hv = 0x243F6A8885A308D3ull;
#pragma unroll
            for (int k = 0; k < KM; ++k)
                if (k < K) hv ^= mix64(dkey(v[k]) + hv);
            hv &= m2;
            for (;;) {
                const uint32_t sidx = atomicCAS(&t2[hv], kEmpty, static_cast<uint32_t>(u));
                if (sidx == kEmpty) {
                    vfresh = true;
                    break;
                }
                bool eq = true;
#pragma unroll
                for (int k = 0; k < KM; ++k)
                    if (k < K) eq &= __ldcg(vals + static_cast<long long>(sidx) * K + k) == v[k];
                if (eq) break;
                hv = (hv + 1) & m2;
            }
            atomicMin(&own[hv], static_cast<unsigned long long>(__brevll(w)));
            slot = static_cast<uint32_t>(hv);
        }
        warp_append(vfresh, slot, reps, cnt + 2);
    }
}

struct AxisBits {  // per objective: (1 << bits) - 1
    unsigned long long mask[kMaxK];
};

// packed cut-value key: objective k at bits [shift_k, shift_k + bits_k) as v_k - lo_k
struct PackGeo {
    long long lo[kMaxK];
    int shift[kMaxK];
};

// The fused kernel when the K cut values pack into at most 63 bits (cut_pack): the collapse
// table holds the packed vectors themselves (64-bit keys, empty = ~0), so no value row is
// written, fenced and re-read for the comparison; the distinct vectors are unpacked from the
// table afterwards. The unique-config count goes to 32 spread counters (cnt[32..63]).
template <int KM>
__global__ void __launch_bounds__(256) k_dedup_eval_collapse_packed(
    const uint64_t* __restrict__ words, long long M, int m, int K, const int* __restrict__ ei,
    const int* __restrict__ ej, const int* __restrict__ wi, unsigned long long* t1, uint64_t m1,
    unsigned long long* t2, unsigned long long* own, uint64_t m2, PackGeo g, uint32_t* reps, unsigned long long* cnt)
{
    extern __shared__ __align__(16) int sm[];  // weights (m x KM) | edge pairs (m)
    int* ew = sm;
    int* epair = sm + m * KM;
    for (int e = threadIdx.x; e < m; e += blockDim.x) epair[e] = ei[e] | (ej[e] << 16);
    for (int q = threadIdx.x; q < m * KM; q += blockDim.x) {
        const int e = q / KM, k = q % KM;
        ew[q] = k < K ? wi[e * K + k] : 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long* ucnt = cnt + 32 + ((blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) & 31);
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < M;
         i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        bool fresh = false;
        uint64_t w = 0;
        if (i < M) {
            w = words[i];
            uint64_t h = mix64(w) & m1;
            for (;;) {
                // a slot goes from empty to its key once: a plain L2 read settles repeats
                unsigned long long old = __ldcg(&t1[h]);
                if (old == ~0ull) old = atomicCAS(&t1[h], ~0ull, static_cast<unsigned long long>(w));
                if (old == ~0ull) {
                    fresh = true;
                    break;
                }
                if (old == w) break;
                h = (h + 1) & m1;
            }
        }
        const unsigned fb = __ballot_sync(0xffffffffu, fresh);
        if (lane == 0 && fb) atomicAdd(ucnt, static_cast<unsigned long long>(__popc(fb)));
        bool vfresh = false;
        uint32_t slot = 0;
        if (fresh) {
            int acc[KM];
            cut_values_int<KM>(w, m, epair, ew, acc);
            unsigned long long key = 0;
#pragma unroll
            for (int k = 0; k < KM; ++k)
                if (k < K) key |= static_cast<unsigned long long>(static_cast<long long>(acc[k]) - g.lo[k]) << g.shift[k];
            uint64_t hv = mix64(key) & m2;
            for (;;) {
                unsigned long long old = __ldcg(&t2[hv]);
                if (old == ~0ull) old = atomicCAS(&t2[hv], ~0ull, key);
                if (old == ~0ull) {
                    vfresh = true;
                    break;
                }
                if (old == key) break;
                hv = (hv + 1) & m2;
            }
            atomicMin(&own[hv], static_cast<unsigned long long>(__brevll(w)));
            slot = static_cast<uint32_t>(hv);
        }
        warp_append(vfresh, slot, reps, cnt + 2);
    }
}

// rows of a running archive (distinct value vectors with their lex-min configs, one word each)
// into the packed collapse table of k_dedup_eval_collapse_packed: a vector the pool also reached
// keeps the smaller config (the same atomicMin over bit-reversed words), a new one is appended
template <int KM>
__global__ void k_insert_rows_packed(const double* __restrict__ xv, const uint64_t* __restrict__ xw, long long X,
                                     int K, PackGeo g, unsigned long long* t2, unsigned long long* own, uint64_t m2,
                                     uint32_t* reps, unsigned long long* cnt)
{
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < X;
         i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        bool vfresh = false;
        uint32_t slot = 0;
        if (i < X) {
            unsigned long long key = 0;
#pragma unroll
            for (int k = 0; k < KM; ++k)
                if (k < K)
                    key |= static_cast<unsigned long long>(static_cast<long long>(xv[i * K + k]) - g.lo[k]) << g.shift[k];
            uint64_t hv = mix64(key) & m2;
            for (;;) {
                unsigned long long old = __ldcg(&t2[hv]);
                if (old == ~0ull) old = atomicCAS(&t2[hv], ~0ull, key);
                if (old == ~0ull) {
                    vfresh = true;
                    break;
                }
                if (old == key) break;
                hv = (hv + 1) & m2;
            }
            atomicMin(&own[hv], static_cast<unsigned long long>(__brevll(xw[i])));
            slot = static_cast<uint32_t>(hv);
        }
        warp_append(vfresh, slot, reps, cnt + 2);
    }
}

// distinct vectors of the packed fused path: values unpacked from the keys, lex-min config
template <int KM>
__global__ void k_slots_packed(const uint32_t* __restrict__ reps, const unsigned long long* __restrict__ dV,
                               const unsigned long long* __restrict__ t2, const unsigned long long* __restrict__ own,
                               int K, PackGeo g, AxisBits b, double* vv, uint64_t* cfg, uint32_t* ident)
{
    const long long V = static_cast<long long>(*dV);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint32_t sl = reps[i];
        const unsigned long long key = t2[sl];
        const unsigned long long ow = own[sl];
#pragma unroll
        for (int k = 0; k < KM; ++k)
            if (k < K)
                vv[i * K + k] =
                    static_cast<double>(g.lo[k] + static_cast<long long>((key >> g.shift[k]) & b.mask[k]));
        cfg[i] = __brevll(ow);
        ident[i] = static_cast<uint32_t>(i);
    }
}

// distinct vectors of the fused path -> (row into vals, lex-min config word, identity owner)
__global__ void k_slots_fused(const uint32_t* __restrict__ reps, const unsigned long long* __restrict__ dV,
                              const uint32_t* __restrict__ t2, const unsigned long long* __restrict__ own,
                              uint32_t* rows, uint64_t* cfg, uint32_t* ident)
{
    const long long V = static_cast<long long>(*dV);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint32_t sl = reps[i];
        rows[i] = t2[sl];
        cfg[i] = __brevll(own[sl]);
        ident[i] = static_cast<uint32_t>(i);
    }
}

// k_gather_vals with the row count on the device
__global__ void k_gather_vals_dev(const double* __restrict__ src, const uint32_t* __restrict__ rows,
                                  const unsigned long long* __restrict__ dV, int K, double* dst)
{
    const long long n = static_cast<long long>(*dV) * K;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[i] = src[static_cast<long long>(rows[i / K]) * K + i % K];
}

// ---- K5 for one-word configs with n <= 63: the config word is the key (empty = ~0, which no
// such config equals); one CAS per config and no re-read of the pool for the comparison
// A table smaller than the pool (L2-sized) may fill up: past `limit` keys or 256 probes the
// kernel raises ucount[1] and stops inserting; the host then redoes the dedup at full size.
constexpr int kDedupCache = 1024;  // keys per CTA (8 KB)
__global__ void k_dedup64(const uint64_t* __restrict__ words, long long M, unsigned long long* table, uint64_t tmask,
                          uint32_t* uniq, unsigned long long* ucount, unsigned long long limit)
{
    // most configs of a pool are repeats (1e8 samples, ~7e6 distinct at C5), and the popular
    // ones would send thousands of CASes to one slot, serialised in L2. A direct-mapped cache of
    // keys this CTA has already settled in the table screens them first; then one lane per
    // distinct key of the warp goes to the table, where a slot already holding the key is
    // found by a plain read (a slot goes from empty to its key once)
    __shared__ unsigned long long seen[kDedupCache];
    __shared__ uint32_t pend[8][kWBuf];  // 256 threads
    for (int q = threadIdx.x; q < kDedupCache; q += blockDim.x) seen[q] = ~0ull;
    __syncthreads();
    WarpBuffer<kWBuf> wb{pend[threadIdx.x >> 5], 0};
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < M;
         i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        bool fresh = false;
        uint64_t w = i < M ? words[i] : ~0ull;
        const uint32_t cs = static_cast<uint32_t>(w ^ (w >> 29)) & (kDedupCache - 1);
        if (i < M && seen[cs] == w) w = ~0ull;  // settled by this CTA before
        const unsigned peers = __match_any_sync(0xffffffffu, w);
        if (w != ~0ull && (threadIdx.x & 31) == __ffs(peers) - 1) {
            uint64_t h = mix64(w) & tmask;
            for (int probe = 0;; ++probe) {
                if (probe == 256) {
                    atomicExch(ucount + 1, 1ull);
                    break;
                }
                unsigned long long old = __ldcg(&table[h]);
                if (old == ~0ull) old = atomicCAS(&table[h], ~0ull, static_cast<unsigned long long>(w));
                if (old == ~0ull) {
                    fresh = true;
                    break;
                }
                if (old == w) break;
                h = (h + 1) & tmask;
            }
            seen[cs] = w;  // in the table now (a racing write leaves another settled key)
        }
        wb.push(fresh, static_cast<uint32_t>(i), uniq, ucount, limit, ucount + 1);  // past limit: redo
    }
    wb.flush(uniq, ucount, limit, ucount + 1);
}

// ---- K5: dedup of packed configs (pareto.hpp:309-326)
__global__ void k_dedup(const uint64_t* __restrict__ words, long long M, int wpc, uint32_t* table, uint64_t tmask,
                        uint32_t* uniq, unsigned long long* ucount)
{
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < M;
         i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        bool fresh = false;
        if (i < M) {
            const uint64_t* w = words + i * wpc;
            uint64_t h = hash_words(w, wpc) & tmask;
            for (;;) {
                uint32_t s = atomicAdd(&table[h], 0u);
                if (s == kEmpty) {
                    s = atomicCAS(&table[h], kEmpty, static_cast<uint32_t>(i));
                    if (s == kEmpty) {
                        fresh = true;
                        break;
                    }
                }
                bool eq = true;
                for (int q = 0; q < wpc; ++q) eq &= words[static_cast<long long>(s) * wpc + q] == w[q];
                if (eq) break;
                h = (h + 1) & tmask;
            }
        }
        warp_append(fresh, static_cast<uint32_t>(i), uniq, ucount);
    }
}

// ---- K4: exact integer cut values, instance.hpp:183-194 (== evaluate_cuts for integer weights);
// KM >= K objectives unrolled (2, 4, 8 or 16)
template <int KM>
__global__ void k_eval_int(const uint64_t* __restrict__ words, const uint32_t* __restrict__ idx, long long U, int wpc,
                           int m, int K, const int* __restrict__ ei, const int* __restrict__ ej,
                           const int* __restrict__ wi, double* out)
{
    extern __shared__ int sm[];
    const bool staged = m * (2 + K) <= 12000;
    if (staged) {
        for (int e = threadIdx.x; e < m; e += blockDim.x) {
            sm[e] = ei[e];
            sm[m + e] = ej[e];
        }
        for (int q = threadIdx.x; q < m * K; q += blockDim.x) sm[2 * m + q] = wi[q];
        __syncthreads();
    }
    const int* sei = staged ? sm : ei;
    const int* sej = staged ? sm + m : ej;
    const int* swi = staged ? sm + 2 * m : wi;
    for (long long u = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; u < U;
         u += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint64_t* w = words + static_cast<long long>(idx ? idx[u] : u) * wpc;
        int acc[KM];
#pragma unroll
        for (int k = 0; k < KM; ++k) acc[k] = 0;
        if (wpc == 1) {
            const uint64_t w0 = w[0];
            for (int e = 0; e < m; ++e) {
                const uint64_t d = (w0 >> sei[e]) ^ (w0 >> sej[e]);
                const int cut = -static_cast<int>(d & 1ull);  // all-ones when the edge is cut
#pragma unroll
                for (int k = 0; k < KM; ++k)
                    if (k < K) acc[k] += swi[e * K + k] & cut;
            }
        } else {
            for (int e = 0; e < m; ++e) {
                const int a = sei[e], b = sej[e];
                const uint64_t d = (w[a >> 6] >> (a & 63)) ^ (w[b >> 6] >> (b & 63));
                const int cut = -static_cast<int>(d & 1ull);
#pragma unroll
                for (int k = 0; k < KM; ++k)
                    if (k < K) acc[k] += swi[e * K + k] & cut;
            }
        }
#pragma unroll
        for (int k = 0; k < KM; ++k)
            if (k < K) out[u * K + k] = static_cast<double>(acc[k]);
    }
}


// ---- K4 general: evaluate_cuts' FP64 order in the shim (pareto.hpp:346-359):
//      JS_i = sum_j J_k(i,j) s_j (j ascending, from +0.0); h = 0.5 * sum_i s_i JS_i; C = 0.5 (W - h)
__global__ void k_eval_dbl(const uint64_t* __restrict__ words, const uint32_t* __restrict__ idx, long long U, int wpc,
                           int n, int K, const int* __restrict__ rowptr, const int* __restrict__ col,
                           const int* __restrict__ eidx, const double* __restrict__ w, const double* __restrict__ W,
                           double* out)
{
    for (long long u = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; u < U;
         u += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint64_t* cw = words + static_cast<long long>(idx ? idx[u] : u) * wpc;
        for (int k = 0; k < K; ++k) {
            double dot = 0.0;
            for (int i = 0; i < n; ++i) {
                double js = 0.0;
                for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                    const int j = col[e];
                    const double sj = (cw[j >> 6] >> (j & 63)) & 1ull ? 1.0 : -1.0;
                    js = __dadd_rn(js, __dmul_rn(w[static_cast<long long>(eidx[e]) * K + k], sj));
                }
                const double si = (cw[i >> 6] >> (i & 63)) & 1ull ? 1.0 : -1.0;
                dot = __dadd_rn(dot, __dmul_rn(si, js));
            }
            out[u * K + k] = __dmul_rn(0.5, __dsub_rn(W[k], __dmul_rn(0.5, dot)));
        }
    }
}

// ---- K6: collapse equal vectors onto the lex-smallest config (pareto.hpp:383-387)
// vals: U x K; cfg: per-row config pointer index (into words); table slots hold a row index.
__global__ void k_collapse(const double* __restrict__ vals, long long U, int K, const uint64_t* __restrict__ words,
                           const uint32_t* __restrict__ cfg_of_row, int wpc, uint32_t* table, uint32_t* owner,
                           uint64_t tmask, uint32_t* reps, unsigned long long* vcount)
{
    __shared__ uint32_t pend[8][kWBuf];  // 256 threads
    WarpBuffer<kWBuf> wb{pend[threadIdx.x >> 5], 0};
    for (long long u0 = blockIdx.x * static_cast<long long>(blockDim.x); u0 < U;
         u0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long u = u0 + threadIdx.x;
        bool fresh = false;
        uint32_t slot_of = 0;
        if (u < U) {
            const double* v = vals + u * K;
            uint64_t h = hash_vals(v, K) & tmask;
            for (;;) {
                uint32_t s = atomicAdd(&table[h], 0u);
                if (s == kEmpty) {
                    s = atomicCAS(&table[h], kEmpty, static_cast<uint32_t>(u));
                    if (s == kEmpty) {
                        fresh = true;
                        break;
                    }
                }
                if (vals_equal(vals + static_cast<long long>(s) * K, v, K)) break;
                h = (h + 1) & tmask;
            }
            slot_of = static_cast<uint32_t>(h);
            if (words) {  // keep the lexicographically smallest configuration per vector
                const uint32_t me = static_cast<uint32_t>(u);
                uint32_t cur = atomicAdd(&owner[h], 0u);
                for (;;) {
                    if (cur != kEmpty) {
                        const uint64_t* a = words + static_cast<long long>(cfg_of_row ? cfg_of_row[me] : me) * wpc;
                        const uint64_t* b = words + static_cast<long long>(cfg_of_row ? cfg_of_row[cur] : cur) * wpc;
                        if (!config_less(a, b, wpc)) break;
                    }
                    const uint32_t prev = atomicCAS(&owner[h], cur, me);
                    if (prev == cur) break;
                    cur = prev;
                }
            }
        }
        wb.push(fresh, slot_of, reps, vcount, ~0ull, vcount);
    }
    wb.flush(reps, vcount, ~0ull, vcount);
}

// ---- distinct values of every axis (blockIdx.y = axis; hash set of keys per axis), then
// ascending order by rank count. The row count is *dV when given. Each block first keeps the
// keys it has seen in a shared-memory set, so only its first sighting of a value reaches the
// global set (a handful of values repeat across ~10^6 rows; their global slots are otherwise
// the hottest lines of the stage). A full global table (more distinct values than it holds)
// stops probing and reports count > cap (no grid).
__device__ __forceinline__ void distinct_insert_global(unsigned long long key, double v, unsigned long long* table,
                                                       uint64_t tmask, double* out, unsigned long long* count,
                                                       long long cap)
{
    uint64_t h = mix64(key) & tmask;
    for (uint64_t probe = 0;; ++probe) {
        if (probe > 1024) {  // the table (>= 4 x cap slots) is crowded: too many values
            atomicMax(count, static_cast<unsigned long long>(cap) + 1);
            return;
        }
        unsigned long long s = __ldcg(&table[h]);
        if (s == key) return;
        if (s == 0ull) s = atomicCAS(&table[h], 0ull, key);
        if (s == 0ull) {
            const unsigned long long at = atomicAdd(count, 1ull);
            if (static_cast<long long>(at) < cap) out[at] = v + 0.0;
            return;
        }
        if (s == key) return;
        h = (h + 1) & tmask;
    }
}

__global__ void k_distinct(const double* __restrict__ vals, long long V, const unsigned long long* __restrict__ dV,
                           int K, unsigned long long* tables, uint64_t tsize, double* outs, unsigned long long* counts,
                           long long cap)
{
    constexpr int kSet = 1024;
    __shared__ unsigned long long sset[kSet];
    const int axis = blockIdx.y;
    if (dV) V = static_cast<long long>(*dV);
    unsigned long long* table = tables + tsize * axis;
    double* out = outs + cap * axis;
    unsigned long long* count = counts + axis;
    const uint64_t tmask = tsize - 1;
    for (int q = threadIdx.x; q < kSet; q += blockDim.x) sset[q] = 0ull;
    __syncthreads();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double v = vals[i * K + axis];
        const unsigned long long key = dkey(v);
        uint32_t h = static_cast<uint32_t>(mix64(key)) & (kSet - 1);
        bool fresh = true, seen = false;
        for (int probe = 0; probe < 32; ++probe) {  // a full set passes the value through
            const unsigned long long s = atomicCAS(&sset[h], 0ull, key);
            if (s == 0ull) break;
            if (s == key) {
                seen = true;
                break;
            }
            h = (h + 1) & (kSet - 1);
        }
        fresh = !seen;
        if (fresh) {
            // more distinct values than a grid takes: this axis is done (no grid)
            if (static_cast<long long>(__ldcg(count)) > cap) break;
            distinct_insert_global(key, v, table, tmask, out, count, cap);
        }
    }
}

struct AxisCounts {
    int d[kMaxK];
};

// axes with at most this many distinct values are ordered by k_rank_sort_asc (every value
// counts the smaller ones: D^2 compares, ~5 us at the C2 front's ~900); larger ones by a radix sort
constexpr int kRankSortMax = 2048;

__global__ void k_rank_sort_asc(const double* __restrict__ ins, AxisCounts Ds, long long cap, double* outs)
{  // distinct values: rank = #smaller (blockIdx.y = axis)
    extern __shared__ double tile[];
    const int D = Ds.d[blockIdx.y];
    if (D > kRankSortMax) return;  // (radix-sorted by the host)
    const double* in = ins + cap * blockIdx.y;
    double* out = outs + cap * blockIdx.y;
    for (int base = blockIdx.x * blockDim.x; base < D; base += gridDim.x * blockDim.x) {
        const int i = base + threadIdx.x;
        const double v = i < D ? in[i] : 0.0;
        int rank = 0;
        for (int t0 = 0; t0 < D; t0 += blockDim.x) {
            __syncthreads();
            if (t0 + threadIdx.x < D) tile[threadIdx.x] = in[t0 + threadIdx.x];
            __syncthreads();
            const int lim = min(static_cast<int>(blockDim.x), D - t0);
            if (i < D)
                for (int q = 0; q < lim; ++q) rank += tile[q] < v;
        }
        if (i < D) out[rank] = v;
    }
}

__device__ __forceinline__ int lower_rank(const double* sorted, int D, double v)
{
    int lo = 0, hi = D;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sorted[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct GridGeo {
    int dims;                 // K - 1
    long long stride[kMaxK];  // row-major strides over the first K-1 axes
    int D[kMaxK];             // distinct values per axis (all K axes)
    const double* axis[kMaxK];  // sorted distinct values per axis
};

// cell index and last-axis rank+1 of vector i
__device__ __forceinline__ long long cell_of(const GridGeo& g, const double* v, int* r)
{
    long long c = 0;
    for (int a = 0; a < g.dims; ++a) {
        r[a] = lower_rank(g.axis[a], g.D[a], v[a]);
        c += r[a] * g.stride[a];
    }
    return c;
}

__global__ void k_grid_scatter(const double* __restrict__ vals, long long V, int K, GridGeo g, uint32_t* T)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double* v = vals + i * K;
        int r[kMaxK];
        const long long c = cell_of(g, v, r);
        const uint32_t last = static_cast<uint32_t>(lower_rank(g.axis[g.dims], g.D[g.dims], v[g.dims])) + 1;
        atomicMax(&T[c], last);
    }
}

// suffix max along one axis: S[.., a, ..] = max(S[.., a, ..], S[.., a+1, ..])
// (consecutive threads take consecutive lines: coalesced; each thread loads 8 cells of its
// line before it stores any, so 8 loads are in flight instead of one dependent chain)
__global__ void k_suffix_max(uint32_t* S, long long cells, long long stride, int D)
{
    const long long lines = cells / D;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < lines;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long inner = t % stride, outer = t / stride;
        uint32_t* line = S + outer * stride * D + inner;
        uint32_t run = 0;
        for (int a = D - 1; a >= 0; a -= 8) {
            uint32_t v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = a - j >= 0 ? line[static_cast<long long>(a - j) * stride] : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                run = max(run, v[j]);
                if (a - j >= 0) line[static_cast<long long>(a - j) * stride] = run;
            }
        }
    }
}

// the same along the contiguous axis (stride 1): one warp per row, 32 cells per step
// from the end, an in-warp suffix max (shuffles) carried into the next chunk, so every load
// is coalesced
__global__ void k_suffix_max_rows(uint32_t* S, long long rows, int D)
{
    const int lane = threadIdx.x & 31;
    const long long warps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long row = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; row < rows;
         row += warps) {
        uint32_t* r = S + row * D;
        uint32_t carry = 0;
        for (int base = D - 32; base > -32; base -= 32) {
            const int a = base + lane;
            uint32_t v = a >= 0 ? r[a] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_down_sync(0xffffffffu, v, o);
                if (lane + o < 32) v = max(v, u);
            }
            v = max(v, carry);
            if (a >= 0) r[a] = v;
            carry = __shfl_sync(0xffffffffu, v, 0);
        }
    }
}

// weak dominance test of every vector (pareto.hpp:49-57): dominated iff a vector in the
// same cell has a larger last coordinate, or a vector at least as large in all axes and
// strictly larger in one of the first K-1 has a last coordinate >= this one
__global__ void k_grid_test(const double* __restrict__ vals, long long V, int K, GridGeo g, const uint32_t* T,
                            const uint32_t* S, unsigned char* keep)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double* v = vals + i * K;
        int r[kMaxK];
        const long long c = cell_of(g, v, r);
        const uint32_t last = static_cast<uint32_t>(lower_rank(g.axis[g.dims], g.D[g.dims], v[g.dims])) + 1;
        bool dom = T[c] > last;
        for (int a = 0; a < g.dims && !dom; ++a)
            if (r[a] + 1 < g.D[a]) dom = S[c + g.stride[a]] >= last;
        keep[i] = !dom;
    }
}

// all-pairs fallback: dominates_max over every other vector (distinct vectors)
__global__ void k_pairwise(const double* __restrict__ vals, long long V, int K, unsigned char* keep)
{
    extern __shared__ double tile[];  // blockDim.x x K
    for (long long base = blockIdx.x * static_cast<long long>(blockDim.x); base < V;
         base += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = base + threadIdx.x;
        double mine[kMaxK];
        for (int k = 0; k < K; ++k) mine[k] = i < V ? vals[i * K + k] : 0.0;
        bool dom = i >= V;
        for (long long t0 = 0; t0 < V; t0 += blockDim.x) {
            if (__syncthreads_and(dom)) break;
            for (int q = threadIdx.x; q < static_cast<int>(blockDim.x) * K; q += blockDim.x) {
                const long long row = t0 + q / K;
                tile[q] = row < V ? vals[row * K + q % K] : -INFINITY;
            }
            __syncthreads();
            const int lim = static_cast<int>(min(static_cast<long long>(blockDim.x), V - t0));
            for (int q = 0; q < lim && !dom; ++q) {
                bool ge = true, gt = false;
                for (int k = 0; k < K; ++k) {
                    const double a = tile[q * K + k];
                    ge &= a >= mine[k];
                    gt |= a > mine[k];
                }
                dom = ge && gt;
            }
        }
        if (i < V) keep[i] = !dom;
    }
}

// ---- archive order (pareto.hpp:405-406, lexicographically descending) by LSD radix passes:
// the last objective first, each pass a stable
// descending sort of the rows' current order by one objective (orderable u64 keys; -0 == +0)
__device__ __forceinline__ unsigned long long ord_key(double v)
{
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v == 0.0 ? 0.0 : v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_column_keys(const double* __restrict__ vals, const uint32_t* __restrict__ idx, long long F, int K,
                              int k, unsigned long long* keys)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < F;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        keys[i] = ord_key(vals[static_cast<long long>(idx[i]) * K + k]);
}

__global__ void k_iota_u32(uint32_t* a, long long n)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        a[i] = static_cast<uint32_t>(i);
}

__global__ void k_rank_of(const uint32_t* __restrict__ order, long long F, long long* rank)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < F;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        rank[order[i]] = i;
}

__global__ void k_gather_rows(const double* __restrict__ src_vals, const uint32_t* __restrict__ rows, long long F, int K,
                              const uint64_t* __restrict__ src_words, const uint32_t* __restrict__ cfg_rows, int wpc,
                              const long long* __restrict__ rank, double* dst_vals, uint64_t* dst_words)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < F;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long dst = rank ? rank[i] : i;
        const long long sr = rows ? rows[i] : i;
        for (int k = 0; k < K; ++k) dst_vals[dst * K + k] = src_vals[sr * K + k];
        if (dst_words) {
            const long long cr = cfg_rows ? cfg_rows[i] : sr;
            for (int q = 0; q < wpc; ++q) dst_words[dst * wpc + q] = src_words[cr * wpc + q];
        }
    }
}

// ---- reference_point_sampled (pareto.hpp:620-642): cut_values (instance.hpp:183-194, edge
// order) of `count` configs drawn 64 spins per next_u64 from
// Stream(derive_key(seed, 0x70617265), c, 0, tag_word(reference_sample)); per-objective min.
__global__ void k_ref_sample(int count, uint64_t key, int n, int m, int K, const int* __restrict__ ei,
                             const int* __restrict__ ej, const double* __restrict__ w, unsigned long long* rmin,
                             bool staged)
{
    const int wpc = (n + 63) / 64;
    if (staged) {  // (n <= 64)  // one word per config: register-resident, edges and weights in shared memory
        extern __shared__ __align__(16) unsigned char sraw[];
        double* sw = reinterpret_cast<double*>(sraw);                 // m x K
        int* spair = reinterpret_cast<int*>(sw + static_cast<long long>(m) * K);  // (ei | ej << 16) x m
        for (int e = threadIdx.x; e < m; e += blockDim.x) spair[e] = ei[e] | (ej[e] << 16);
        for (int q = threadIdx.x; q < m * K; q += blockDim.x) sw[q] = w[q];
        __syncthreads();
        for (int c0 = blockIdx.x * blockDim.x; c0 < count; c0 += gridDim.x * blockDim.x) {
            const int c = c0 + threadIdx.x;
            uint64_t w0 = 0;
            if (c < count) {
                DevStream s;
                s.init(key, static_cast<uint32_t>(c), 0u, tag_word(kTagReferenceSample, 0));
                w0 = s.next_u64();
            }
            for (int k = 0; k < K; ++k) {
                double acc = 0.0;
                for (int e = 0; e < m; ++e) {
                    const int pr = spair[e];
                    if (((w0 >> (pr & 0xFFFF)) ^ (w0 >> (pr >> 16))) & 1ull) acc = __dadd_rn(acc, sw[e * K + k]);
                }
                unsigned long long mk = c < count ? dkey(acc) : ~0ull;
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long u = __shfl_xor_sync(0xffffffffu, mk, o);
                    mk = u < mk ? u : mk;
                }
                if ((threadIdx.x & 31) == 0 && mk != ~0ull) atomicMin(&rmin[k], mk);
            }
        }
        return;
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < count; c += gridDim.x * blockDim.x) {
        DevStream s;
        s.init(key, static_cast<uint32_t>(c), 0u, tag_word(kTagReferenceSample, 0));
        uint64_t wd[64];
        for (int q = 0; q < wpc && q < 64; ++q) wd[q] = s.next_u64();
        for (int k = 0; k < K; ++k) {
            double acc = 0.0;
            for (int e = 0; e < m; ++e) {
                const int a = ei[e], b = ej[e];
                if (((wd[a >> 6] >> (a & 63)) ^ (wd[b >> 6] >> (b & 63))) & 1ull)
                    acc = __dadd_rn(acc, w[static_cast<long long>(e) * K + k]);
            }
            atomicMin(&rmin[k], dkey(acc));
        }
    }
}

// reference-sample configurations only (the cut values then come from the GEMM evaluator)
__global__ void k_ref_words(int count, uint64_t key, int n, uint64_t* words)
{
    const int wpc = (n + 63) / 64;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < count; c += gridDim.x * blockDim.x) {
        DevStream s;
        s.init(key, static_cast<uint32_t>(c), 0u, tag_word(kTagReferenceSample, 0));
        for (int q = 0; q < wpc; ++q) {
            uint64_t v = s.next_u64();
            if (q == wpc - 1 && (n & 63)) v &= (1ull << (n & 63)) - 1;
            words[static_cast<long long>(c) * wpc + q] = v;
        }
    }
}

// per-objective minimum (ordered keys): one thread per row, a warp minimum per objective,
// then one atomic per warp and objective (the K counters are contended otherwise)
__global__ void k_col_min(const double* __restrict__ vals, long long rows, int K, unsigned long long* rmin)
{
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long base0 = blockIdx.x * static_cast<long long>(blockDim.x);
    for (long long b = base0; b < rows; b += stride) {
        const long long i = b + threadIdx.x;
        for (int k = 0; k < K; ++k) {
            unsigned long long m = i < rows ? dkey(vals[i * K + k]) : ~0ull;
            for (int o = 16; o; o >>= 1) {
                const unsigned long long u = __shfl_xor_sync(0xffffffffu, m, o);
                m = u < m ? u : m;
            }
            if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(&rmin[k], m);
        }
    }
}

// ---- K8: hypervolume over a compressed grid (gains g = v - r). One warp per line of the
// innermost grid axis: the other axes' widths are a per-line product, the lanes stride the
// line's cells (coalesced S loads). Widths are clamped at r, so a grid built over more vectors
// than the archive (the front's grid over every distinct vector, whose dominated region is the
// archive's) gives the same exact value; over the archive's own grid (values >= r) the clamp is
// the identity. The mode comes from k_hv_stats on the device (stats[0]: every value integral,
// stats[1]: the largest gain's key): integral data and r give the exact __int128 sum (64-bit
// cell products when gain^K < 2^62), anything else the Kahan FP64 sum; the host reads the
// matching partials.
__global__ void k_hv_cells(const uint32_t* __restrict__ S, long long cells, GridGeo g, const double* __restrict__ r,
                           const unsigned long long* __restrict__ stats, __int128* ipart, double* dpart)
{
    const int lane = threadIdx.x & 31;
    const int da = g.dims - 1;  // the innermost grid axis (stride 1)
    const long long len = g.D[da];
    const long long lines = cells / len;
    const long long warps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    __int128 iacc = 0;
    double dacc = 0.0, dc = 0.0;
    const double rl = r[g.dims];
    bool integral = stats[0] != 0;
    for (int a = 0; a <= g.dims; ++a) integral &= floor(r[a]) == r[a];
    bool fit64 = false;
    if (integral) {  // the host's rule (hypervolume_device): exact while K e <= 120, maxg < 2^e
        const uint64_t key = stats[1];
        const uint64_t b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
        int e = 0;
        frexp(fmax(__longlong_as_double(static_cast<long long>(b)), 1.0), &e);
        integral = (g.dims + 1) * e <= 120;
        fit64 = (g.dims + 1) * e <= 62;
    }
    for (long long line = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; line < lines;
         line += warps) {
        // widths of the outer axes of this line (cells < 2^27: 32-bit index arithmetic)
        uint32_t rem = static_cast<uint32_t>(line * len);
        double pw = 1.0;
        long long pwi = 1;
        bool empty = false;
        for (int a = 0; a < da; ++a) {
            const uint32_t sa = static_cast<uint32_t>(g.stride[a]);
            const uint32_t ra = rem / sa;
            rem -= ra * sa;
            const double lo = fmax(ra ? g.axis[a][ra - 1] : r[a], r[a]);
            const double w = g.axis[a][ra] - lo;
            if (!(w > 0.0)) empty = true;
            pw *= w;
            pwi *= static_cast<long long>(w);
        }
        if (empty) continue;
        const double* ax = g.axis[da];
        const double rd = r[da];
        const uint32_t* Sl = S + line * len;
        for (long long q = lane; q < len; q += 32) {
            const uint32_t top = Sl[q];
            if (!top) continue;
            const double hgain = g.axis[g.dims][top - 1] - rl;
            if (!(hgain > 0.0)) continue;
            const double w = ax[q] - fmax(q ? ax[q - 1] : rd, rd);
            if (!(w > 0.0)) continue;
            if (integral) {
                if (fit64) {
                    iacc += pwi * static_cast<long long>(w) * static_cast<long long>(hgain);
                } else {
                    __int128 ivol = pwi;
                    ivol *= static_cast<long long>(w);
                    ivol *= static_cast<long long>(hgain);
                    iacc += ivol;
                }
            } else {
                const double vol = hgain * pw * w;
                const double y = vol - dc;  // Kahan
                const double t = dacc + y;
                dc = (t - dacc) - y;
                dacc = t;
            }
        }
    }
    // block partials: shuffle sums within each warp (the __int128 as two 64-bit halves with the
    // carry), then the 8 warp sums by thread 0
    double dsum = dacc - dc;
    for (int o = 16; o; o >>= 1) {
        const unsigned long long lo = static_cast<unsigned long long>(iacc);
        const long long hi = static_cast<long long>(iacc >> 64);
        const unsigned long long olo = __shfl_down_sync(0xffffffffu, lo, o);
        const long long ohi = __shfl_down_sync(0xffffffffu, hi, o);
        iacc += (static_cast<__int128>(ohi) << 64) | static_cast<__int128>(olo);
        dsum += __shfl_down_sync(0xffffffffu, dsum, o);
    }
    __shared__ __int128 si[8];
    __shared__ double sd[8];
    if (lane == 0) {
        si[threadIdx.x >> 5] = iacc;
        sd[threadIdx.x >> 5] = dsum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __int128 a = 0;
        double b = 0.0;
        for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
            a += si[q];
            b += sd[q];
        }
        ipart[blockIdx.x] = a;
        dpart[blockIdx.x] = b;
    }
}


// integrality of the archive values and the largest gain v - r (decides the exact __int128 HV
// sum): flags[0] &= every value is an integer below 9e15, flags[1] = max dkey(gain); and
// validate_reference (pareto.hpp:103-118): *first = the first (entry K + objective) with
// r > v. With rkeys the reference comes as ordered keys (reference_keys_device): it is decoded
// here and written to r for the kernels that follow.
__global__ void k_hv_stats(const double* __restrict__ vals, long long F, int K, double* r,
                           const unsigned long long* __restrict__ rkeys, unsigned long long* flags,
                           unsigned long long* first)
{
    double rr[kMaxK];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) {
        if (k < K) {
            if (rkeys) {
                const unsigned long long key = rkeys[k];
                const unsigned long long b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
                rr[k] = __longlong_as_double(static_cast<long long>(b));
            } else {
                rr[k] = r[k];
            }
        }
    }
    if (rkeys && blockIdx.x == 0 && threadIdx.x < K) r[threadIdx.x] = rr[threadIdx.x];
    bool integral = true;
    unsigned long long gmax = dkey(0.0);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < F * K;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double v = vals[i];
        const int k = static_cast<int>(i % K);
        double rk = rr[0];
#pragma unroll
        for (int q = 1; q < kMaxK; ++q)
            if (q == k) rk = rr[q];
        integral &= floor(v) == v && fabs(v) < 9.0e15;
        if (rk > v) atomicMin(first, static_cast<unsigned long long>(i));
        const unsigned long long g = dkey(v - rk);
        gmax = g > gmax ? g : gmax;
    }
    if (!__all_sync(0xffffffffu, integral) && (threadIdx.x & 31) == 0) atomicAnd(&flags[0], 0ull);
    for (int o = 16; o; o >>= 1) {
        const unsigned long long u = __shfl_xor_sync(0xffffffffu, gmax, o);
        gmax = u > gmax ? u : gmax;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(&flags[1], gmax);
}

// MOMC_TRACE=1: host timestamps of the Pareto stage on stderr (diagnostics)
void trace(const char* what)
{
    static const bool on = std::getenv("MOMC_TRACE") != nullptr;
    if (!on) return;
    static auto t0 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[momc %9.3f ms] %s\n", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), what);
}

uint64_t pow2_at_least(uint64_t x)
{
    uint64_t p = 1024;
    while (p < x) p <<= 1;
    return p;
}

int grid_blocks(long long n, int threads = 256)
{
    long long b = (n + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    if (b < 1) b = 1;
    return static_cast<int>(b);
}

void launch_eval_int(Ctx& c, const uint64_t* words, const uint32_t* idx, long long U, int wpc, double* out)
{
    const int K = c.k;
    const int sm = c.m * (2 + K) <= 12000 ? c.m * (2 + K) * 4 : 0;
    auto kern = K <= 2 ? k_eval_int<2> : K <= 4 ? k_eval_int<4> : K <= 8 ? k_eval_int<8> : k_eval_int<16>;
    kern<<<grid_blocks(U), 256, sm, c.stream>>>(words, idx, U, wpc, c.m, K, c.d_ei.p, c.d_ej.p, c.d_wi.p, out);
}

double seconds_between(cudaEvent_t a, cudaEvent_t b)
{
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
}

// scratch reused across calls
struct Scratch {
    DevBuf<uint32_t> table, uniq, table2, owner, reps, rows, cfgrows;
    DevBuf<unsigned long long> counters, dtable, dtab64;
    DevBuf<double> vals, axisbuf, axis_sorted, rdev;
    DevBuf<uint32_t> T, S;
    DevBuf<unsigned char> keep;
    DevBuf<long long> rank;
    DevBuf<__int128> ipart;
    DevBuf<double> front_vals;  // unordered front rows kept for an async order (finish_archive)
    DevBuf<uint32_t> front_own;
    DevBuf<uint64_t> front_words;
    DevBuf<double> dpart;
    GridGeo front_geo{};        // the grid of the last filter's front (see Ctx::grid_gen)
    long long front_cells = 0;
};
Scratch& scratch(Ctx& c)
{
    if (!c.pareto_scratch) c.pareto_scratch = std::shared_ptr<void>(new Scratch(), [](void* p) {
        auto* s = static_cast<Scratch*>(p);
        s->table.release(); s->uniq.release(); s->table2.release(); s->owner.release(); s->reps.release();
        s->rows.release(); s->cfgrows.release(); s->counters.release(); s->dtable.release(); s->vals.release();
        s->axisbuf.release(); s->axis_sorted.release(); s->rdev.release(); s->T.release(); s->S.release();
        s->dtab64.release();
        s->keep.release(); s->rank.release(); s->ipart.release(); s->dpart.release();
        s->front_vals.release(); s->front_own.release(); s->front_words.release();
        delete s;
    });
    return *static_cast<Scratch*>(c.pareto_scratch.get());
}

unsigned long long read_counter(Ctx& c, unsigned long long* d)
{
    auto* h = static_cast<unsigned long long*>(pinned_buf(c, sizeof(unsigned long long)));
    ck(cudaMemcpyAsync(h, d, sizeof *h, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "sync");
    return *h;
}

// Compressed grid over V vectors (K >= 2), in two phases around the one read-back of the
// per-axis distinct counts. grid_distinct: the distinct values of every axis (V rows, or *dV
// rows when dV is given; Vcap bounds them), counts at counters[8 .. 8+K).
void grid_distinct(Ctx& c, Scratch& s, const double* d_vals, long long Vcap, const unsigned long long* dV, int K)
{
    ++c.grid_gen;
    const uint64_t tsize =
        pow2_at_least(4ull * static_cast<uint64_t>(std::min<long long>(Vcap, kDistinctCap)) + 16);
    s.dtable.reserve(tsize * K);
    s.axisbuf.reserve(static_cast<size_t>(kDistinctCap) * K);
    s.axis_sorted.reserve(static_cast<size_t>(kDistinctCap) * K);
    s.counters.reserve(8 + kMaxK);
    ck(cudaMemsetAsync(s.dtable.p, 0, sizeof(unsigned long long) * tsize * K, c.stream), "memset");
    ck(cudaMemsetAsync(s.counters.p + 8, 0, sizeof(unsigned long long) * K, c.stream), "memset");
    const int gx = std::min(grid_blocks(Vcap), 256);  // long block loops: few first sightings per block
    k_distinct<<<dim3(gx, K), 256, 0, c.stream>>>(d_vals, Vcap, dV, K, s.dtable.p, tsize, s.axisbuf.p,
                                                   s.counters.p + 8, kDistinctCap);
    c.launches++;
}

// grid_finish: with the distinct counts on the host, sort the axes and build the cell table
// T (max last-axis rank + 1 per cell) and its suffix max S. Returns false when it would not fit.
bool grid_finish(Ctx& c, Scratch& s, const double* d_vals, long long V, int K, const unsigned long long* dcount,
                 GridGeo& g, long long& cells, std::vector<std::vector<double>>* host_axes = nullptr)
{
    g.dims = K - 1;
    long long prod = 1;
    AxisCounts dc{};
    int maxD = 1;
    for (int a = 0; a < K; ++a) {
        const long long D = static_cast<long long>(dcount[a]);
        if (D > kDistinctCap) return false;
        g.D[a] = static_cast<int>(D);
        dc.d[a] = static_cast<int>(D);
        maxD = std::max(maxD, static_cast<int>(D));
        g.axis[a] = s.axis_sorted.p + static_cast<size_t>(a) * kDistinctCap;
        if (a < K - 1) {
            prod *= D;
            if (prod > kGridCap) return false;
        }
    }
    k_rank_sort_asc<<<dim3(grid_blocks(std::min(maxD, kRankSortMax), 256), K), 256, 256 * sizeof(double),
                      c.stream>>>(s.axisbuf.p, dc, kDistinctCap, s.axis_sorted.p);
    c.launches++;
    if (maxD > kRankSortMax) {  // O(D) per large axis instead of D^2 compares
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, s.axisbuf.p, s.axis_sorted.p, maxD, 0, 64, c.stream);
        DevBuf<unsigned char> tmp;
        tmp.reserve(tb + 1);
        for (int a = 0; a < K; ++a)
            if (g.D[a] > kRankSortMax) {
                const size_t off = static_cast<size_t>(a) * kDistinctCap;
                ck(cub::DeviceRadixSort::SortKeys(tmp.p, tb, s.axisbuf.p + off, s.axis_sorted.p + off, g.D[a], 0, 64,
                                                  c.stream),
                   "axis sort");
                c.launches += 4;
            }
        tmp.release();
    }
    if (host_axes) {
        for (int a = 0; a < K; ++a) {
            std::vector<double> hv(static_cast<size_t>(g.D[a]));
            ck(cudaMemcpyAsync(hv.data(), g.axis[a], sizeof(double) * g.D[a], cudaMemcpyDeviceToHost, c.stream),
               "D2H");
            ck(cudaStreamSynchronize(c.stream), "sync");
            host_axes->push_back(std::move(hv));
        }
    }
    cells = prod;
    long long st = 1;
    for (int a = K - 2; a >= 0; --a) {
        g.stride[a] = st;
        st *= g.D[a];
    }
    s.T.reserve(static_cast<size_t>(cells));
    s.S.reserve(static_cast<size_t>(cells));
    ck(cudaMemsetAsync(s.T.p, 0, sizeof(uint32_t) * cells, c.stream), "memset");
    k_grid_scatter<<<grid_blocks(V), 256, 0, c.stream>>>(d_vals, V, K, g, s.T.p);
    c.launches++;
    ck(cudaMemcpyAsync(s.S.p, s.T.p, sizeof(uint32_t) * cells, cudaMemcpyDeviceToDevice, c.stream), "D2D");
    for (int a = 0; a < K - 1; ++a) {
        if (g.D[a] < 2) continue;
        if (g.stride[a] == 1)
            k_suffix_max_rows<<<grid_blocks(cells / g.D[a] * 32), 256, 0, c.stream>>>(s.S.p, cells / g.D[a], g.D[a]);
        else
            k_suffix_max<<<grid_blocks(cells / g.D[a]), 256, 0, c.stream>>>(s.S.p, cells, g.stride[a], g.D[a]);
        c.launches++;
    }
    return true;
}

bool build_grid(Ctx& c, Scratch& s, const double* d_vals, long long V, int K, GridGeo& g, long long& cells,
                std::vector<std::vector<double>>* host_axes = nullptr)
{
    grid_distinct(c, s, d_vals, V, nullptr, K);
    auto* pc = static_cast<unsigned long long*>(pinned_buf(c, sizeof(unsigned long long) * K));
    ck(cudaMemcpyAsync(pc, s.counters.p + 8, sizeof(unsigned long long) * K, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "sync");
    const std::vector<unsigned long long> dcount(pc, pc + K);
    return grid_finish(c, s, d_vals, V, K, dcount.data(), g, cells, host_axes);
}

// ---- sieve front for large value sets the compressed grid cannot hold: a front F0 of a
// good sample (the rows with the largest objective sums) kills most rows; the front of the
// survivors is the front. Exact whatever the sample: a dominated row is dominated by a
// front row, which either lies in F0 (the row is killed) or survives (pairwise removes it).
__global__ void k_sum_keys(const double* __restrict__ vals, long long V, int K, unsigned long long* keys, uint32_t* idx)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double sum = 0.0;
        for (int k = 0; k < K; ++k) sum += vals[i * K + k];
        const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(sum == 0.0 ? 0.0 : sum));
        keys[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
        idx[i] = static_cast<uint32_t>(i);
    }
}

__global__ void k_gather_vals_idx(const double* __restrict__ vals, const uint32_t* __restrict__ idx, long long n, int K,
                                  double* out)
{
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n * K;
         q += static_cast<long long>(gridDim.x) * blockDim.x)
        out[q] = vals[static_cast<long long>(idx[q / K]) * K + q % K];
}

// alive[i] = no row of F (nF x K, staged in shared memory) dominates row i
__global__ void k_kill(const double* __restrict__ vals, long long V, int K, const double* __restrict__ F, int nF,
                       unsigned char* alive)
{
    extern __shared__ double fs[];
    for (int q = threadIdx.x; q < nF * K; q += blockDim.x) fs[q] = F[q];
    __syncthreads();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double mine[kMaxK];
        for (int k = 0; k < K; ++k) mine[k] = vals[i * K + k];
        bool dom = false;
        for (int f = 0; f < nF && !dom; ++f) {
            bool ge = true, gt = false;
            for (int k = 0; k < K; ++k) {
                ge &= fs[f * K + k] >= mine[k];
                gt |= fs[f * K + k] > mine[k];
            }
            dom = ge && gt;
        }
        alive[i] = !dom;
    }
}

__global__ void k_scatter_keep(const uint32_t* __restrict__ idx, const unsigned char* __restrict__ sub_keep, long long n,
                               unsigned char* keep)
{
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<long long>(gridDim.x) * blockDim.x)
        keep[idx[q]] = sub_keep[q];
}

__global__ void k_map_u32(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ map, long long n, uint32_t* out);

__global__ void k_compact_flags(const unsigned char* __restrict__ f, long long V, uint32_t* out, unsigned long long* count)
{
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < V;
         i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        const bool on = i < V && f[i];
        const unsigned b = __ballot_sync(0xffffffffu, on);
        unsigned long long base = 0;
        if ((threadIdx.x & 31) == 0 && b) base = atomicAdd(count, static_cast<unsigned long long>(__popc(b)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (on) out[base + __popc(b & ((1u << (threadIdx.x & 31)) - 1))] = static_cast<uint32_t>(i);
    }
}

// rows `idx` (n of them) -> keep flags of their pairwise front (sub_keep, n)
void pairwise_subset(Ctx& c, const double* d_vals, const uint32_t* idx, long long n, int K, unsigned char* sub_keep)
{
    DevBuf<double> sub;
    sub.reserve(static_cast<size_t>(n) * K + 1);
    k_gather_vals_idx<<<grid_blocks(n * K), 256, 0, c.stream>>>(d_vals, idx, n, K, sub.p);
    k_pairwise<<<grid_blocks(n), 256, 256 * K * sizeof(double), c.stream>>>(sub.p, n, K, sub_keep);
    c.launches += 2;
    ck(cudaStreamSynchronize(c.stream), "pairwise subset");
    sub.release();
}

void sieve_front(Ctx& c, Scratch& s, const double* d_vals, long long V, int K)
{
    const long long B = std::min<long long>(V, 8192);
    DevBuf<unsigned long long> ka, kb;
    DevBuf<uint32_t> ia, ib, fidx, sidx;
    DevBuf<unsigned char> fkeep, alive, skeep, tmp;
    ka.reserve(static_cast<size_t>(V));
    kb.reserve(static_cast<size_t>(V));
    ia.reserve(static_cast<size_t>(V));
    ib.reserve(static_cast<size_t>(V));
    k_sum_keys<<<grid_blocks(V), 256, 0, c.stream>>>(d_vals, V, K, ka.p, ia.p);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, ka.p, kb.p, ia.p, ib.p, static_cast<int>(V), 0, 64, c.stream);
    tmp.reserve(tb + 1);
    ck(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, ka.p, kb.p, ia.p, ib.p, static_cast<int>(V), 0, 64,
                                                 c.stream),
       "sort");
    c.launches += 2;
    // F0 = front of the B rows with the largest sums
    fkeep.reserve(static_cast<size_t>(B));
    pairwise_subset(c, d_vals, ib.p, B, K, fkeep.p);
    s.counters.reserve(8);
    ck(cudaMemsetAsync(s.counters.p + 3, 0, sizeof(unsigned long long), c.stream), "memset");
    fidx.reserve(static_cast<size_t>(B));
    k_compact_flags<<<grid_blocks(B), 256, 0, c.stream>>>(fkeep.p, B, fidx.p, s.counters.p + 3);
    c.launches++;
    const long long nF0 = static_cast<long long>(read_counter(c, s.counters.p + 3));
    // positions in the sorted order -> row ids, then the F0 rows themselves
    DevBuf<uint32_t> f0rows;
    f0rows.reserve(static_cast<size_t>(nF0) + 1);
    k_map_u32<<<grid_blocks(nF0), 256, 0, c.stream>>>(fidx.p, ib.p, nF0, f0rows.p);
    DevBuf<double> f0;
    f0.reserve(static_cast<size_t>(nF0) * K + 1);
    k_gather_vals_idx<<<grid_blocks(nF0 * K), 256, 0, c.stream>>>(d_vals, f0rows.p, nF0, K, f0.p);
    c.launches += 2;
    // kill every row dominated by F0 (F0 staged in shared memory when it fits)
    alive.reserve(static_cast<size_t>(V));
    const size_t fbytes = static_cast<size_t>(nF0) * K * sizeof(double);
    if (fbytes <= 160 * 1024) {
        if (fbytes > 48 * 1024)
            ck(cudaFuncSetAttribute(k_kill, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fbytes)),
               "smem");
        k_kill<<<grid_blocks(V), 256, fbytes, c.stream>>>(d_vals, V, K, f0.p, static_cast<int>(nF0), alive.p);
    } else {  // F0 too large to stage: plain pairwise over everything
        k_pairwise<<<grid_blocks(V), 256, 256 * K * sizeof(double), c.stream>>>(d_vals, V, K, s.keep.p);
        c.launches++;
        return;
    }
    c.launches++;
    ck(cudaMemsetAsync(s.counters.p + 3, 0, sizeof(unsigned long long), c.stream), "memset");
    sidx.reserve(static_cast<size_t>(V));
    k_compact_flags<<<grid_blocks(V), 256, 0, c.stream>>>(alive.p, V, sidx.p, s.counters.p + 3);
    c.launches++;
    const long long nS = static_cast<long long>(read_counter(c, s.counters.p + 3));
    skeep.reserve(static_cast<size_t>(nS) + 1);
    pairwise_subset(c, d_vals, sidx.p, nS, K, skeep.p);
    ck(cudaMemsetAsync(s.keep.p, 0, static_cast<size_t>(V), c.stream), "memset");
    k_scatter_keep<<<grid_blocks(nS), 256, 0, c.stream>>>(sidx.p, skeep.p, nS, s.keep.p);
    c.launches++;
    for (auto* b : {&ka, &kb}) b->release();
    for (auto* b : {&ia, &ib, &fidx, &sidx, &f0rows}) b->release();
    for (auto* b : {&fkeep, &alive, &skeep, &tmp}) b->release();
    f0.release();
}

// front of V distinct vectors (device rows); keep[i] set for non-dominated rows
int front_keep(Ctx& c, Scratch& s, const double* d_vals, long long V, int K,
               const unsigned long long* dcount = nullptr)
{
    s.keep.reserve(static_cast<size_t>(V) + 1);
    if (K >= 2) {
        GridGeo g{};
        long long cells = 0;
        if (dcount ? grid_finish(c, s, d_vals, V, K, dcount, g, cells) : build_grid(c, s, d_vals, V, K, g, cells)) {
            k_grid_test<<<grid_blocks(V), 256, 0, c.stream>>>(d_vals, V, K, g, s.T.p, s.S.p, s.keep.p);
            c.launches++;
            s.front_geo = g;
            s.front_cells = cells;
            return 1;
        }
    }
    if (V > 16384) {  // the sieve: a good sample's front kills most rows first
        sieve_front(c, s, d_vals, V, K);
        return 3;
    }
    k_pairwise<<<grid_blocks(V), 256, 256 * K * sizeof(double), c.stream>>>(d_vals, V, K, s.keep.p);
    c.launches++;
    return 2;
}

__global__ void k_compact_keep(const unsigned char* __restrict__ keep, long long V, const uint32_t* __restrict__ map,
                               uint32_t* out, unsigned long long* count)
{
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x); i0 < V;
         i0 += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        const bool f = i < V && keep[i];
        warp_append(f, f ? (map ? map[i] : static_cast<uint32_t>(i)) : 0u, out, count);
    }
}

__global__ void k_slots_to_rows(const uint32_t* __restrict__ slots, long long V, const uint32_t* __restrict__ table,
                                const uint32_t* __restrict__ owner, uint32_t* rows, uint32_t* own_rows)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        rows[i] = table[slots[i]];
        if (own_rows) own_rows[i] = owner[slots[i]];
    }
}

__global__ void k_gather_vals(const double* __restrict__ src, const uint32_t* __restrict__ rows, long long V, int K,
                              double* dst)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < V * K;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[i] = src[static_cast<long long>(rows[i / K]) * K + i % K];
}

__global__ void k_map_u32(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ map, long long n, uint32_t* out)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = map[idx[i]];
}


// packed lexicographic key: objective 0 in the most significant bits (exact: integer cut
// values within their ranges)
__global__ void k_packed_keys(const double* __restrict__ vals, long long F, int K, PackGeo g, unsigned long long* keys,
                              uint32_t* idx)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < F;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        unsigned long long key = 0;
        for (int k = 0; k < K; ++k)
            key |= static_cast<unsigned long long>(static_cast<long long>(vals[i * K + k]) - g.lo[k]) << g.shift[k];
        keys[i] = key;
        idx[i] = static_cast<uint32_t>(i);
    }
}

void lex_desc_rank(Ctx& c, const double* d_vals, long long F, int K, long long* rank)
{
    if (F <= 0) return;
    if (c.values_are_cuts && c.cut_pack && K == c.k) {  // one radix pass over packed keys
        PackGeo g{};
        int sh = 64;
        for (int k = 0; k < K; ++k) {
            sh -= c.cut_bits[static_cast<size_t>(k)];
            g.lo[k] = c.cut_lo[static_cast<size_t>(k)];
            g.shift[k] = sh;
        }
        DevBuf<uint32_t> ia, ib;
        DevBuf<unsigned long long> ka, kb;
        ia.reserve(static_cast<size_t>(F));
        ib.reserve(static_cast<size_t>(F));
        ka.reserve(static_cast<size_t>(F));
        kb.reserve(static_cast<size_t>(F));
        k_packed_keys<<<grid_blocks(F), 256, 0, c.stream>>>(d_vals, F, K, g, ka.p, ia.p);
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, ka.p, kb.p, ia.p, ib.p, static_cast<int>(F), sh, 64,
                                                  c.stream);
        DevBuf<unsigned char> tmp;
        tmp.reserve(tb + 1);
        ck(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, ka.p, kb.p, ia.p, ib.p, static_cast<int>(F), sh, 64,
                                                     c.stream),
           "sort");
        k_rank_of<<<grid_blocks(F), 256, 0, c.stream>>>(ib.p, F, rank);
        c.launches += 3;
        ia.release();
        ib.release();
        ka.release();
        kb.release();
        tmp.release();
        return;
    }
    DevBuf<uint32_t> ia, ib;
    DevBuf<unsigned long long> ka, kb;
    ia.reserve(static_cast<size_t>(F));
    ib.reserve(static_cast<size_t>(F));
    ka.reserve(static_cast<size_t>(F));
    kb.reserve(static_cast<size_t>(F));
    k_iota_u32<<<grid_blocks(F), 256, 0, c.stream>>>(ia.p, F);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, ka.p, kb.p, ia.p, ib.p, static_cast<int>(F), 0, 64,
                                              c.stream);
    DevBuf<unsigned char> tmp;
    tmp.reserve(tb + 1);
    uint32_t* cur = ia.p;
    uint32_t* nxt = ib.p;
    for (int k = K - 1; k >= 0; --k) {
        k_column_keys<<<grid_blocks(F), 256, 0, c.stream>>>(d_vals, cur, F, K, k, ka.p);
        ck(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, ka.p, kb.p, cur, nxt, static_cast<int>(F), 0, 64,
                                                     c.stream),
           "sort");
        std::swap(cur, nxt);
        c.launches += 2;
    }
    k_rank_of<<<grid_blocks(F), 256, 0, c.stream>>>(cur, F, rank);
    c.launches += 2;
    ia.release();
    ib.release();
    ka.release();
    kb.release();
    tmp.release();
}

__global__ void k_gather_words(const uint64_t* __restrict__ words, const uint32_t* __restrict__ idx, long long U, int wpc,
                               uint64_t* out)
{
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < U * wpc;
         q += static_cast<long long>(gridDim.x) * blockDim.x)
        out[q] = words[static_cast<long long>(idx[q / wpc]) * wpc + q % wpc];
}

// Shared tail of both filters: V distinct vectors (d_vv, V x K) with owner configs
// (row index into `words` via d_own, or none) -> front -> archive (lex-descending).
void finish_archive(Ctx& c, Scratch& s, const double* d_vv, long long V, int K, const uint64_t* words,
                    const uint32_t* d_own, int wpc, DevArchive& out, ParetoTimings* tm,
                    const unsigned long long* dcount = nullptr)
{
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    cudaEventRecord(e0, c.stream);
    const int method = front_keep(c, s, d_vv, V, K, dcount);
    trace("finish_archive: front launched");
    s.rows.reserve(static_cast<size_t>(V) + 1);
    ck(cudaMemsetAsync(s.counters.p + 1, 0, sizeof(unsigned long long), c.stream), "memset");
    k_compact_keep<<<grid_blocks(V), 256, 0, c.stream>>>(s.keep.p, V, nullptr, s.rows.p, s.counters.p + 1);
    c.launches++;
    const long long F = static_cast<long long>(read_counter(c, s.counters.p + 1));
    cudaEventRecord(e1, c.stream);
    // gather front rows, then order them lexicographically descending. With c.order_async the
    // front rows stay in scratch (the caller's HV reads them) and the order runs on
    // c.order_stream; the caller joins it (momc_b200_pipeline)
    const bool async = c.order_async && !c.skip_order;
    DevBuf<double> fv_local;
    DevBuf<uint32_t> fown_local;
    DevBuf<double>& fv = async ? s.front_vals : fv_local;
    DevBuf<uint32_t>& fown = async ? s.front_own : fown_local;
    fv.reserve(static_cast<size_t>(F) * K + 1);
    if (d_own) {
        fown.reserve(static_cast<size_t>(F) + 1);
        k_map_u32<<<grid_blocks(F), 256, 0, c.stream>>>(s.rows.p, d_own, F, fown.p);
        c.launches++;
    }
    k_gather_rows<<<grid_blocks(F), 256, 0, c.stream>>>(d_vv, s.rows.p, F, K, nullptr, nullptr, 0, nullptr, fv.p,
                                                         nullptr);
    c.launches++;
    s.rank.reserve(static_cast<size_t>(F) + 1);
    out.F = F;
    out.K = K;
    out.wpc = d_own ? wpc : 0;
    out.vals.reserve(static_cast<size_t>(F) * K + 1);
    if (d_own) out.words.reserve(static_cast<size_t>(F) * wpc + 1);
    const uint64_t* ow = words;  // the order's config source, rows fown (or the front's own rows)
    const uint32_t* orows = d_own ? fown.p : nullptr;
    if (async && d_own) {  // the caller's `words` may be freed on c.stream before the order runs
        s.front_words.reserve(static_cast<size_t>(F) * wpc + 1);
        k_gather_words<<<grid_blocks(F * wpc), 256, 0, c.stream>>>(words, fown.p, F, wpc, s.front_words.p);
        c.launches++;
        ow = s.front_words.p;
        orows = nullptr;
    }
    auto order = [&] {
        if (!c.skip_order) lex_desc_rank(c, fv.p, F, K, s.rank.p);
        k_gather_rows<<<grid_blocks(F), 256, 0, c.stream>>>(fv.p, nullptr, F, K, ow, orows, wpc,
                                                             c.skip_order ? nullptr : s.rank.p, out.vals.p,
                                                             d_own ? out.words.p : nullptr);
        c.launches++;
    };
    if (async) {
        if (!c.order_stream) {
            int least = 0, greatest = 0;
            ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "stream priorities");
            ck(cudaStreamCreateWithPriority(&c.order_stream, cudaStreamNonBlocking, greatest), "stream");
            ck(cudaEventCreate(&c.ev_order_fork), "event");
            ck(cudaEventCreate(&c.ev_order_done), "event");
        }
        ck(cudaEventRecord(c.ev_order_fork, c.stream), "event");
        ck(cudaStreamWaitEvent(c.order_stream, c.ev_order_fork, 0), "event wait");
        struct Swap {  // the order's launches, allocations and frees go to order_stream
            Ctx& c;
            cudaStream_t main;
            explicit Swap(Ctx& cc) : c(cc), main(cc.stream) { c.stream = c.order_stream; g_alloc_stream = c.order_stream; }
            ~Swap() { c.stream = main; g_alloc_stream = main; }
        };
        {
            Swap swap(c);
            order();
            ck(cudaEventRecord(c.ev_order_done, c.stream), "event");
        }
        c.order_pending = true;
        c.order_front = fv.p;
    } else {
        order();
    }
    cudaEventRecord(e2, c.stream);
    if (method == 1) {  // the front's grid covers this archive (hypervolume_device)
        c.front_grid_gen = c.grid_gen;
        c.grid_archive = async ? fv.p : out.vals.p;  // (the pipeline's join points it at out.vals)
        c.grid_rows = F;
    }
    if (tm) {
        ck(cudaStreamSynchronize(c.stream), "archive");
        tm->front_s = seconds_between(e0, e1);
        tm->order_s = async ? 0.0 : seconds_between(e1, e2);  // async: the pipeline times it
        tm->front_method = method;
        tm->unique_vectors = V;
    }
    fv_local.release();
    fown_local.release();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
}

}  // namespace

void evaluate_cuts_device(Ctx& c, const uint64_t* d_words, long long U, double* d_out)
{
    evaluate_cuts_rows(c, d_words, nullptr, U, d_out);
}

void evaluate_cuts_rows(Ctx& c, const uint64_t* d_words, const uint32_t* idx, long long U, double* d_out)
{
    const int wpc = (c.n + 63) / 64;
    if (c.k > kMaxK) usage("the GPU path supports at most 16 objectives");
    if (U == 0) return;
    if (eval_gemm_ok(c)) {
        evaluate_cuts_gemm(c, d_words, idx, U, d_out);
    } else if (c.integer_weights) {
        launch_eval_int(c, d_words, idx, U, wpc, d_out);
    } else {
        k_eval_dbl<<<grid_blocks(U, 128), 128, 0, c.stream>>>(d_words, idx, U, wpc, c.n, c.k, c.d_rowptr.p,
                                                               c.d_col.p, c.d_eidx.p, c.d_w.p, weight_totals(c), d_out);
    }
    c.launches++;
    ck(cudaGetLastError(), "evaluate_cuts");
}

// filter_pool_device for one-word configs with integer weights: dedup + evaluation + collapse
// in one kernel, the distinct values of the grid axes right after, and a single read-back of
// the counts before the front (three fewer host round trips than the staged path below)
// the fused dedup + evaluation + collapse pass applies: one-word configs, integer weights, the
// per-CTA edge tables fit shared memory, tables sized by rows <= 2^24
bool fused_filter_ok(Ctx& c, long long rows)
{
    return c.n <= 63 && c.k >= 2 && c.integer_weights && !eval_gemm_ok(c) && c.m * 17 <= 12000 && rows <= (1ll << 24);
}

// the K cut values of this instance pack into one 64-bit key below ~0
bool cuts_pack63(const Ctx& c)
{
    int pbits = 0;
    for (int k = 0; k < c.k; ++k) pbits += c.cut_bits[static_cast<size_t>(k)];
    return c.cut_pack && pbits <= 63;
}

// X > 0 (packed only): the X rows (xv: X x K values, xw: one config word each) of a running
// archive join the collapse, so out = filter(pool U archive) in one pass (stream_step)
void filter_pool_fused(Ctx& c, Scratch& s, const uint64_t* d_words, long long M, DevArchive& out, ParetoTimings* tm,
                       const double* xv = nullptr, const uint64_t* xw = nullptr, long long X = 0)
{
    const int K = c.k;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c.stream);
    const bool packed = cuts_pack63(c);  // ~0 is then no vector's key
    if (X > 0 && !packed) usage("internal: archive rows need packed keys");
    const long long MX = M + X;  // bound on the distinct vectors
    const uint64_t t1 = pow2_at_least(2ull * static_cast<uint64_t>(MX) + 16);
    s.dtab64.reserve(t1 * 2);  // dedup keys | collapse owners
    if (!packed) {
        s.table2.reserve(t1);  // collapse rows
        s.vals.reserve(static_cast<size_t>(M) * K + 1);
        ck(cudaMemsetAsync(s.table2.p, 0xFF, sizeof(uint32_t) * t1, c.stream), "memset");
    }
    s.reps.reserve(static_cast<size_t>(MX) + 1);
    s.counters.reserve(64);  // [0] unique configs, [2] distinct vectors, [8, 8+K) axis counts,
                             // [32, 64) spread unique-config counters (packed path)
    ck(cudaMemsetAsync(s.dtab64.p, 0xFF, sizeof(unsigned long long) * t1 * 2, c.stream), "memset");
    ck(cudaMemsetAsync(s.counters.p, 0, sizeof(unsigned long long) * 64, c.stream), "memset");
    const int KM = K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16;
    const int sm = c.m * (1 + KM) * 4;
    DevBuf<uint32_t> vrow, vown;
    DevBuf<uint64_t> vcfg;
    DevBuf<double> vv;
    vown.reserve(static_cast<size_t>(MX) + 1);
    vcfg.reserve(static_cast<size_t>(MX) + 1);
    vv.reserve(static_cast<size_t>(MX) * K + 1);
    const unsigned long long* dV = s.counters.p + 2;
    if (packed) {
        PackGeo g{};
        AxisBits b{};
        int sh = 64;
        for (int k = 0; k < K; ++k) {
            const int bits = c.cut_bits[static_cast<size_t>(k)];
            sh -= bits;
            g.lo[k] = c.cut_lo[static_cast<size_t>(k)];
            g.shift[k] = sh;
            b.mask[k] = bits >= 64 ? ~0ull : (1ull << bits) - 1;
        }
        DevBuf<unsigned long long> t2;
        t2.reserve(t1);
        ck(cudaMemsetAsync(t2.p, 0xFF, sizeof(unsigned long long) * t1, c.stream), "memset");
        auto kern = KM == 2 ? k_dedup_eval_collapse_packed<2> : KM == 4 ? k_dedup_eval_collapse_packed<4>
                    : KM == 8 ? k_dedup_eval_collapse_packed<8> : k_dedup_eval_collapse_packed<16>;
        kern<<<grid_blocks(M), 256, sm, c.stream>>>(d_words, M, c.m, K, c.d_ei.p, c.d_ej.p, c.d_wi.p, s.dtab64.p,
                                                     t1 - 1, t2.p, s.dtab64.p + t1, t1 - 1, g, s.reps.p,
                                                     s.counters.p);
        ck(cudaGetLastError(), "dedup+eval+collapse");
        if (X > 0) {
            auto ki = KM == 2 ? k_insert_rows_packed<2> : KM == 4 ? k_insert_rows_packed<4>
                      : KM == 8 ? k_insert_rows_packed<8> : k_insert_rows_packed<16>;
            ki<<<grid_blocks(X), 256, 0, c.stream>>>(xv, xw, X, K, g, t2.p, s.dtab64.p + t1, t1 - 1, s.reps.p,
                                                     s.counters.p);
            c.launches++;
        }
        auto ks = KM == 2 ? k_slots_packed<2> : KM == 4 ? k_slots_packed<4>
                  : KM == 8 ? k_slots_packed<8> : k_slots_packed<16>;
        ks<<<grid_blocks(MX), 256, 0, c.stream>>>(s.reps.p, dV, t2.p, s.dtab64.p + t1, K, g, b, vv.p, vcfg.p, vown.p);
        t2.release();
        c.launches += 2;
    } else {
        auto kern = KM == 2 ? k_dedup_eval_collapse<2> : KM == 4 ? k_dedup_eval_collapse<4>
                    : KM == 8 ? k_dedup_eval_collapse<8> : k_dedup_eval_collapse<16>;
        kern<<<grid_blocks(M), 256, sm, c.stream>>>(d_words, M, c.m, K, c.d_ei.p, c.d_ej.p, c.d_wi.p, s.dtab64.p,
                                                     t1 - 1, s.table2.p, s.dtab64.p + t1, t1 - 1, s.vals.p, s.reps.p,
                                                     s.counters.p);
        c.launches++;
        ck(cudaGetLastError(), "dedup+eval+collapse");
        vrow.reserve(static_cast<size_t>(M) + 1);
        k_slots_fused<<<grid_blocks(M), 256, 0, c.stream>>>(s.reps.p, dV, s.table2.p, s.dtab64.p + t1, vrow.p,
                                                              vcfg.p, vown.p);
        k_gather_vals_dev<<<grid_blocks(M * K), 256, 0, c.stream>>>(s.vals.p, vrow.p, dV, K, vv.p);
        c.launches += 2;
    }
    grid_distinct(c, s, vv.p, MX, dV, K);
    cudaEventRecord(e1, c.stream);
    auto* ph = static_cast<unsigned long long*>(pinned_buf(c, sizeof(unsigned long long) * 64));
    ck(cudaMemcpyAsync(ph, s.counters.p, sizeof(unsigned long long) * 64, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "counts");
    unsigned long long h[64];
    std::memcpy(h, ph, sizeof h);
    long long U = static_cast<long long>(h[0]);
    if (packed)
        for (int q = 32; q < 64; ++q) U += static_cast<long long>(h[q]);
    const long long V = static_cast<long long>(h[2]);
    if (tm) {
        tm->unique_configs = U;
        tm->dedup_s = seconds_between(e0, e1);  // dedup + evaluation + collapse + axis values
        tm->eval_s = 0;
        tm->collapse_s = 0;
    }
    c.values_are_cuts = true;
    try {
        finish_archive(c, s, vv.p, V, K, vcfg.p, vown.p, 1, out, tm, h + 8);
    } catch (...) {
        c.values_are_cuts = false;
        throw;
    }
    c.values_are_cuts = false;
    vrow.release();
    vown.release();
    vcfg.release();
    vv.release();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

void filter_pool_device(Ctx& c, const uint64_t* d_words, long long M, DevArchive& out, ParetoTimings* tm)
{
    if (M <= 0) usage("non-dominated filter needs a non-empty pool");
    if (c.n == 0) usage("pool does not match instance");
    if (c.k > kMaxK) usage("the GPU path supports at most 16 objectives");
    if (M >= 0xFFFFFFFFll) usage("pool too large for one device pass (shard it)");
    trace("filter_pool: enter");
    Scratch& s = scratch(c);
    const int wpc = (c.n + 63) / 64;
    const int K = c.k;
    // (tables sized by M: pools beyond 2^24 configs take the staged path, sized by the counts)
    if (fused_filter_ok(c, M)) {
        filter_pool_fused(c, s, d_words, M, out, tm);
        return;
    }
    cudaEvent_t e0, e1, e2, e3;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    cudaEventCreate(&e3);
    cudaEventRecord(e0, c.stream);
    // K5 dedup
    const uint64_t tsize = pow2_at_least(2ull * static_cast<uint64_t>(M));
    s.uniq.reserve(static_cast<size_t>(M));
    s.counters.reserve(8);
    ck(cudaMemsetAsync(s.counters.p, 0, sizeof(unsigned long long) * 8, c.stream), "memset");
    if (c.n <= 63) {
        // an L2-sized table first (2^24 keys, 128 MB; a pool of 1e8 configs has ~7e6 distinct
        // ones), the full 2M-slot table only if it fills to 3/4
        uint64_t small = std::min<uint64_t>(tsize, 1ull << 24);
        // test hook: MOMC_TEST_DEDUP_SLOTS=s starts with an s-slot table (forces the redo)
        if (const char* f = std::getenv("MOMC_TEST_DEDUP_SLOTS")) small = std::min<uint64_t>(small, pow2_at_least(std::atoll(f)));
        for (uint64_t ts : {small, tsize}) {
            s.dtab64.reserve(ts);
            ck(cudaMemsetAsync(s.dtab64.p, 0xFF, sizeof(unsigned long long) * ts, c.stream), "memset");
            ck(cudaMemsetAsync(s.counters.p, 0, sizeof(unsigned long long) * 2, c.stream), "memset");
            k_dedup64<<<grid_blocks(M), 256, 0, c.stream>>>(d_words, M, s.dtab64.p, ts - 1, s.uniq.p, s.counters.p,
                                                             ts / 4 * 3);
            if (ts == tsize) break;
            auto* pf = static_cast<unsigned long long*>(pinned_buf(c, 2 * sizeof(unsigned long long)));
            ck(cudaMemcpyAsync(pf, s.counters.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream),
               "D2H");
            ck(cudaStreamSynchronize(c.stream), "sync");
            if (!pf[1]) break;
            c.launches++;
        }
    } else {
        s.table.reserve(tsize);
        ck(cudaMemsetAsync(s.table.p, 0xFF, sizeof(uint32_t) * tsize, c.stream), "memset");
        k_dedup<<<grid_blocks(M), 256, 0, c.stream>>>(d_words, M, wpc, s.table.p, tsize - 1, s.uniq.p, s.counters.p);
    }
    c.launches++;
    const long long U = static_cast<long long>(read_counter(c, s.counters.p));
    trace("filter_pool: dedup done");
    cudaEventRecord(e1, c.stream);
    // K4 eval of the unique configs
    s.vals.reserve(static_cast<size_t>(U) * K + 1);
    if (eval_gemm_ok(c)) {  // large dense instances: exact int8 tensor-core form
        evaluate_cuts_gemm(c, d_words, s.uniq.p, U, s.vals.p);
    } else if (c.integer_weights) {
        launch_eval_int(c, d_words, s.uniq.p, U, wpc, s.vals.p);
        c.launches++;
    } else {
        k_eval_dbl<<<grid_blocks(U, 128), 128, 0, c.stream>>>(d_words, s.uniq.p, U, wpc, c.n, K, c.d_rowptr.p,
                                                               c.d_col.p, c.d_eidx.p, c.d_w.p, weight_totals(c),
                                                               s.vals.p);
        c.launches++;
    }
    ck(cudaGetLastError(), "eval");
    cudaEventRecord(e2, c.stream);
    // K6 collapse onto the lex-smallest config
    const uint64_t t2 = pow2_at_least(2ull * static_cast<uint64_t>(U) + 16);
    s.table2.reserve(t2);
    s.owner.reserve(t2);
    s.reps.reserve(static_cast<size_t>(U) + 1);
    ck(cudaMemsetAsync(s.table2.p, 0xFF, sizeof(uint32_t) * t2, c.stream), "memset");
    ck(cudaMemsetAsync(s.owner.p, 0xFF, sizeof(uint32_t) * t2, c.stream), "memset");
    k_collapse<<<grid_blocks(U), 256, 0, c.stream>>>(s.vals.p, U, K, d_words, s.uniq.p, wpc, s.table2.p, s.owner.p,
                                                      t2 - 1, s.reps.p, s.counters.p + 2);
    c.launches++;
    const long long V = static_cast<long long>(read_counter(c, s.counters.p + 2));
    trace("filter_pool: eval+collapse done");
    // distinct vectors (row of the first inserter) + owner rows -> dense arrays
    DevBuf<uint32_t> vrow, vown;
    vrow.reserve(static_cast<size_t>(V) + 1);
    vown.reserve(static_cast<size_t>(V) + 1);
    k_slots_to_rows<<<grid_blocks(V), 256, 0, c.stream>>>(s.reps.p, V, s.table2.p, s.owner.p, vrow.p, vown.p);
    c.launches++;
    DevBuf<double> vv;
    vv.reserve(static_cast<size_t>(V) * K + 1);
    k_gather_vals<<<grid_blocks(V * K), 256, 0, c.stream>>>(s.vals.p, vrow.p, V, K, vv.p);
    c.launches++;
    // owner rows index the unique list; map them to pool rows
    DevBuf<uint32_t> vcfg;
    vcfg.reserve(static_cast<size_t>(V) + 1);
    k_map_u32<<<grid_blocks(V), 256, 0, c.stream>>>(vown.p, s.uniq.p, V, vcfg.p);
    c.launches++;
    cudaEventRecord(e3, c.stream);
    if (tm) tm->unique_configs = U;
    trace("filter_pool: finish_archive");
    c.values_are_cuts = true;
    try {
        finish_archive(c, s, vv.p, V, K, d_words, vcfg.p, wpc, out, tm);
    } catch (...) {
        c.values_are_cuts = false;
        throw;
    }
    c.values_are_cuts = false;
    if (tm) {  // the events completed: finish_archive read results back after them
        ck(cudaEventSynchronize(e3), "events");
        tm->dedup_s = seconds_between(e0, e1);
        tm->eval_s = seconds_between(e1, e2);
        tm->collapse_s = seconds_between(e2, e3);
    }
    trace("filter_pool: archive done");
    vrow.release();
    vown.release();
    vv.release();
    vcfg.release();
    for (auto ev : {e0, e1, e2, e3}) cudaEventDestroy(ev);
}


// front of (the M pool configs U the X rows xv / xw) into `out` in one collapse + front pass:
// the streaming step's "run front merged into the running archive" without a separate run
// front. xv / xw may alias `out` (they are copied first).
bool filter_pool_merge_device(Ctx& c, const uint64_t* d_words, long long M, const double* xv, const uint64_t* xw,
                              long long X, DevArchive& out, DevBuf<double>& all_vals)
{
    if (M <= 0) usage("non-dominated filter needs a non-empty pool");
    if (c.k > kMaxK) usage("the GPU path supports at most 16 objectives");
    if (M >= 0xFFFFFFFFll) usage("pool too large for one device pass (shard it)");
    Scratch& s = scratch(c);
    const int wpc = (c.n + 63) / 64;
    const int K = c.k;
    if (fused_filter_ok(c, M + X) && cuts_pack63(c)) {
        // the fused pool pass with the archive rows inserted into its collapse table; the old
        // rows go to all_vals first (the caller compares them with the result)
        all_vals.reserve(static_cast<size_t>(X) * K + 1);
        if (X) ck(cudaMemcpyAsync(all_vals.p, xv, sizeof(double) * X * K, cudaMemcpyDeviceToDevice, c.stream), "D2D");
        filter_pool_fused(c, s, d_words, M, out, nullptr, all_vals.p, xw, X);
        return true;
    }
    const uint64_t tsize = pow2_at_least(2ull * static_cast<uint64_t>(M));
    s.table.reserve(tsize);
    s.uniq.reserve(static_cast<size_t>(M));
    s.counters.reserve(8);
    ck(cudaMemsetAsync(s.table.p, 0xFF, sizeof(uint32_t) * tsize, c.stream), "memset");
    ck(cudaMemsetAsync(s.counters.p, 0, sizeof(unsigned long long) * 8, c.stream), "memset");
    k_dedup<<<grid_blocks(M), 256, 0, c.stream>>>(d_words, M, wpc, s.table.p, tsize - 1, s.uniq.p, s.counters.p);
    c.launches++;
    const long long U = static_cast<long long>(read_counter(c, s.counters.p));
    const long long T = U + X;
    all_vals.reserve(static_cast<size_t>(T) * K + 1);
    DevBuf<uint64_t> aw;
    aw.reserve(static_cast<size_t>(T) * wpc + 1);
    // the X rows first (rows [0, X): the caller compares them with the result), then the pool
    if (X) {
        ck(cudaMemcpyAsync(all_vals.p, xv, sizeof(double) * X * K, cudaMemcpyDeviceToDevice, c.stream), "D2D");
        ck(cudaMemcpyAsync(aw.p, xw, sizeof(uint64_t) * X * wpc, cudaMemcpyDeviceToDevice, c.stream), "D2D");
    }
    evaluate_cuts_rows(c, d_words, s.uniq.p, U, all_vals.p + X * K);
    k_gather_words<<<grid_blocks(U * wpc), 256, 0, c.stream>>>(d_words, s.uniq.p, U, wpc, aw.p + X * wpc);
    c.launches++;
    filter_values_device(c, all_vals.p, aw.p, wpc, c.n, T, K, out, nullptr);
    aw.release();
    return false;
}

void filter_values_device(Ctx& c, const double* d_vals, const uint64_t* d_words, int wpc, int n_spins, long long M,
                          int K, DevArchive& out, ParetoTimings* tm)
{
    (void)n_spins;
    if (M <= 0) usage("non-dominated filter needs a non-empty pool");
    if (K > kMaxK) usage("the GPU path supports at most 16 objectives");
    Scratch& s = scratch(c);
    s.counters.reserve(8);
    ck(cudaMemsetAsync(s.counters.p, 0, sizeof(unsigned long long) * 8, c.stream), "memset");
    const uint64_t t2 = pow2_at_least(2ull * static_cast<uint64_t>(M) + 16);
    s.table2.reserve(t2);
    s.owner.reserve(t2);
    s.reps.reserve(static_cast<size_t>(M) + 1);
    ck(cudaMemsetAsync(s.table2.p, 0xFF, sizeof(uint32_t) * t2, c.stream), "memset");
    ck(cudaMemsetAsync(s.owner.p, 0xFF, sizeof(uint32_t) * t2, c.stream), "memset");
    k_collapse<<<grid_blocks(M), 256, 0, c.stream>>>(d_vals, M, K, d_words, nullptr, wpc, s.table2.p, s.owner.p,
                                                      t2 - 1, s.reps.p, s.counters.p + 2);
    c.launches++;
    const long long V = static_cast<long long>(read_counter(c, s.counters.p + 2));
    DevBuf<uint32_t> vrow, vown;
    vrow.reserve(static_cast<size_t>(V) + 1);
    vown.reserve(static_cast<size_t>(V) + 1);
    k_slots_to_rows<<<grid_blocks(V), 256, 0, c.stream>>>(s.reps.p, V, s.table2.p, s.owner.p, vrow.p,
                                                           d_words ? vown.p : nullptr);
    c.launches++;
    DevBuf<double> vv;
    vv.reserve(static_cast<size_t>(V) * K + 1);
    k_gather_vals<<<grid_blocks(V * K), 256, 0, c.stream>>>(d_vals, vrow.p, V, K, vv.p);
    c.launches++;
    if (tm) {
        tm->unique_configs = M;
    }
    finish_archive(c, s, vv.p, V, K, d_words, d_words ? vown.p : nullptr, wpc, out, tm);
    vrow.release();
    vown.release();
    vv.release();
}

namespace {

// reference_point_sampled (pareto.hpp:620-642) [+ clamp_reference :647-655] as K ordered keys
// in d_keys (dkey of each objective's minimum), launches only
void reference_keys_device(Ctx& c, int count, uint64_t seed, const double* clamp_vals, long long clamp_rows,
                           unsigned long long* d_keys)
{
    if (count < 1) usage("sampled reference needs count >= 1");
    if (c.n > 4096) usage("reference sampling on the GPU path supports n <= 4096");
    ck(cudaMemsetAsync(d_keys, 0xFF, sizeof(unsigned long long) * c.k, c.stream), "memset");
    if (eval_gemm_ok(c)) {  // cut_values == evaluate_cuts exactly for integer weights
        const int wpc = (c.n + 63) / 64;
        DevBuf<uint64_t> wd;
        DevBuf<double> cv;
        wd.reserve(static_cast<size_t>(count) * wpc);
        cv.reserve(static_cast<size_t>(count) * c.k);
        k_ref_words<<<grid_blocks(count, 128), 128, 0, c.stream>>>(count, derive_key(seed, 0x70617265u), c.n, wd.p);
        c.launches++;
        evaluate_cuts_gemm(c, wd.p, nullptr, count, cv.p);
        k_col_min<<<grid_blocks(count), 256, 0, c.stream>>>(cv.p, count, c.k, d_keys);
        c.launches++;
        wd.release();  // stream-ordered: no host sync needed
        cv.release();
    } else {
        const size_t sm = static_cast<size_t>(c.m) * (c.k * 8 + 4);
        const bool staged = c.n <= 64 && sm <= 48 * 1024;
        k_ref_sample<<<grid_blocks(count, 128), 128, staged ? sm : 0, c.stream>>>(
            count, derive_key(seed, 0x70617265u), c.n, c.m, c.k, c.d_ei.p, c.d_ej.p, c.d_w.p, d_keys, staged);
        c.launches++;
    }
    if (clamp_vals && clamp_rows > 0) {  // clamp_reference (pareto.hpp:647-655): min with every archive row
        k_col_min<<<grid_blocks(clamp_rows), 256, 0, c.stream>>>(clamp_vals, clamp_rows, c.k, d_keys);
        c.launches++;
    }
}

std::vector<double> decode_keys(const unsigned long long* h, int K)
{
    std::vector<double> r(static_cast<size_t>(K));
    for (int k = 0; k < K; ++k) {
        const uint64_t key = h[k];
        const uint64_t b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
        std::memcpy(&r[static_cast<size_t>(k)], &b, 8);
    }
    return r;
}

}  // namespace

std::vector<double> reference_point_sampled_device(Ctx& c, int count, uint64_t seed, const double* clamp_vals,
                                                   long long clamp_rows)
{
    DevBuf<unsigned long long> rmin;
    rmin.reserve(static_cast<size_t>(c.k));
    reference_keys_device(c, count, seed, clamp_vals, clamp_rows, rmin.p);
    auto* ph = static_cast<unsigned long long*>(pinned_buf(c, sizeof(unsigned long long) * c.k));
    ck(cudaMemcpyAsync(ph, rmin.p, sizeof(unsigned long long) * c.k, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "reference point");
    const std::vector<double> r = decode_keys(ph, c.k);
    rmin.release();
    return r;
}

namespace {

// Hypervolume of the archive (d_vals, F x K) at the reference point in device memory (d_r).
// With rkeys (the K ordered keys d_r was decoded from) r is read back with the sums and
// returned in r; otherwise r holds it already. One read-back: [r keys] | checks | partials.
double hv_core(Ctx& c, Scratch& s, const double* d_vals, long long F, int K, const double* d_r,
               std::vector<double>& r, const unsigned long long* rkeys, bool reuse_front_grid)
{
    if (F <= 0) usage("hypervolume of an empty archive");
    if (K > kMaxK) usage("the GPU path supports at most 16 objectives");
    const unsigned long long none = ~0ull;
    // counters[3] first bad entry (none), [4] integral flag (all ones), [5] max dkey(gain)
    // (0: below every gain's key; the host floors it at 1 anyway)
    ck(cudaMemsetAsync(s.counters.p + 3, 0xFF, sizeof(unsigned long long) * 2, c.stream), "memset");
    ck(cudaMemsetAsync(s.counters.p + 5, 0, sizeof(unsigned long long), c.stream), "memset");
    // gains are exact integers when every value and r is integral (n=42 configs): then the
    // __int128 cell sum is the exact hypervolume, i.e. the reference's exact double result
    k_hv_stats<<<grid_blocks(F * K), 256, 0, c.stream>>>(d_vals, F, K, const_cast<double*>(d_r), rkeys,
                                                          s.counters.p + 4, s.counters.p + 3);
    c.launches++;
    auto finish_checks = [&](const unsigned long long* st, bool& integral) {
        if (st[0] != none)
            usage("reference point not dominated by archive entry " + std::to_string(st[0] / K) + " (objective " +
                  std::to_string(st[0] % K) + ")");
        integral = st[1] != 0;
        double maxg;
        const uint64_t key = st[2];
        const uint64_t b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
        std::memcpy(&maxg, &b, 8);
        for (int k = 0; k < K; ++k) integral &= std::floor(r[static_cast<size_t>(k)]) == r[static_cast<size_t>(k)];
        int e = 0;  // keep __int128 exact: maxg < 2^e, K e <= 120 (the same rule as k_hv_cells)
        std::frexp(std::max(maxg, 1.0), &e);
        if (integral && K * e > 120) integral = false;
    };
    const size_t kb = rkeys ? 16 * sizeof(unsigned long long) : 0;  // r keys lead the read-back
    if (K == 1) {
        unsigned long long st[3];
        unsigned char* pb = static_cast<unsigned char*>(pinned_buf(c, kb + sizeof st));
        if (rkeys) ck(cudaMemcpyAsync(pb, rkeys, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaMemcpyAsync(pb + kb, s.counters.p + 3, sizeof st, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "sync");
        if (rkeys) r = decode_keys(reinterpret_cast<const unsigned long long*>(pb), 1);
        std::memcpy(st, pb + kb, sizeof st);
        bool integral;
        finish_checks(st, integral);
        double best = 0;  // pareto.hpp:544-548
        std::vector<double> hv(static_cast<size_t>(F));
        ck(cudaMemcpyAsync(hv.data(), d_vals, sizeof(double) * F, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "sync");
        for (long long i = 0; i < F; ++i) best = std::max(best, hv[static_cast<size_t>(i)] - r[0]);
        return best;
    }
    GridGeo g{};
    long long cells = 0;
    if (reuse_front_grid && c.front_grid_gen == c.grid_gen && c.grid_archive == d_vals && c.grid_rows == F) {
        g = s.front_geo;  // built over every distinct vector of the pool: the same dominated region
        cells = s.front_cells;
    } else if (!build_grid(c, s, d_vals, F, K, g, cells)) {
        runtime("hypervolume: front too large for the compressed-grid method (" + std::to_string(F) + " points)");
    }
    const long long lines = cells / g.D[g.dims - 1];
    const int blocks = grid_blocks(lines * 32);
    s.ipart.reserve(static_cast<size_t>(blocks));
    s.dpart.reserve(static_cast<size_t>(blocks));
    k_hv_cells<<<blocks, 256, 0, c.stream>>>(s.S.p, cells, g, d_r, s.counters.p + 4, s.ipart.p, s.dpart.p);
    c.launches++;
    ck(cudaGetLastError(), "hv");
    unsigned long long st[3];
    const size_t nb = static_cast<size_t>(blocks);
    unsigned char* pb =
        static_cast<unsigned char*>(pinned_buf(c, kb + 32 + nb * (sizeof(__int128) + sizeof(double))));
    if (rkeys) ck(cudaMemcpyAsync(pb, rkeys, sizeof(unsigned long long) * K, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(pb + kb, s.counters.p + 3, sizeof st, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(pb + kb + 32, s.ipart.p, sizeof(__int128) * nb, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(pb + kb + 32 + sizeof(__int128) * nb, s.dpart.p, sizeof(double) * nb, cudaMemcpyDeviceToHost,
                       c.stream),
       "D2H");
    ck(cudaStreamSynchronize(c.stream), "hv");
    if (rkeys) r = decode_keys(reinterpret_cast<const unsigned long long*>(pb), K);
    std::memcpy(st, pb + kb, sizeof st);
    std::vector<__int128> ip(nb);
    std::vector<double> dp(nb);
    std::memcpy(ip.data(), pb + kb + 32, sizeof(__int128) * nb);
    std::memcpy(dp.data(), pb + kb + 32 + sizeof(__int128) * nb, sizeof(double) * nb);
    bool integral;
    finish_checks(st, integral);
    if (integral) {
        __int128 tot = 0;
        for (auto v : ip) tot += v;
        return static_cast<double>(tot);
    }
    double tot = 0, comp = 0;
    for (double v : dp) {
        const double y = v - comp;
        const double t = tot + y;
        comp = (t - tot) - y;
        tot = t;
    }
    return tot;
}

}  // namespace

double hypervolume_device(Ctx& c, const double* d_vals, long long F, int K, const std::vector<double>& r,
                          bool reuse_front_grid)
{
    if (F <= 0) usage("hypervolume of an empty archive");
    if (static_cast<int>(r.size()) != K) usage("reference point length does not match archive");
    if (K > kMaxK) usage("the GPU path supports at most 16 objectives");
    Scratch& s = scratch(c);
    s.counters.reserve(8);
    s.rdev.reserve(static_cast<size_t>(kMaxK));
    auto* pr = static_cast<double*>(pinned_buf(c, sizeof(double) * K));
    std::memcpy(pr, r.data(), sizeof(double) * K);
    ck(cudaMemcpyAsync(s.rdev.p, pr, sizeof(double) * K, cudaMemcpyHostToDevice, c.stream), "H2D");
    std::vector<double> rr = r;
    return hv_core(c, s, d_vals, F, K, s.rdev.p, rr, nullptr, reuse_front_grid);
}

double hv_sampled_reference_device(Ctx& c, const double* d_vals, long long F, int K, int count, uint64_t seed,
                                   std::vector<double>& r_out, bool reuse_front_grid)
{
    if (F <= 0) usage("hypervolume of an empty archive");
    Scratch& s = scratch(c);
    s.counters.reserve(8);
    s.rdev.reserve(static_cast<size_t>(kMaxK));
    DevBuf<unsigned long long> keys;
    keys.reserve(static_cast<size_t>(kMaxK));
    reference_keys_device(c, count, seed, d_vals, F, keys.p);
    // (k_hv_stats decodes the keys into s.rdev for k_hv_cells)
    const double hv = hv_core(c, s, d_vals, F, K, s.rdev.p, r_out, keys.p, reuse_front_grid);
    keys.release();
    return hv;
}

namespace {

__device__ __forceinline__ uint64_t row_hash(const double* v, int K)
{
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (int k = 0; k < K; ++k) {
        const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v[k] == 0.0 ? 0.0 : v[k]));
        h ^= b + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xBF58476D1CE4E5B9ull;
    }
    return h ^ (h >> 31);
}

__global__ void k_set_insert(const double* __restrict__ v, long long F, int K, uint32_t* table, uint64_t mask)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < F;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        uint64_t q = row_hash(v + i * K, K) & mask;
        while (atomicCAS(&table[q], 0xFFFFFFFFu, static_cast<uint32_t>(i)) != 0xFFFFFFFFu) q = (q + 1) & mask;
    }
}

__global__ void k_set_missing(const double* __restrict__ a, const uint32_t* __restrict__ table, uint64_t mask,
                              const double* __restrict__ b, long long F, int K, unsigned long long* missing)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < F;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double* v = b + i * K;
        uint64_t q = row_hash(v, K) & mask;
        bool found = false;
        for (;;) {
            const uint32_t r = table[q];
            if (r == 0xFFFFFFFFu) break;
            bool eq = true;
            for (int k = 0; k < K; ++k) eq &= a[static_cast<long long>(r) * K + k] == v[k];
            if (eq) {
                found = true;
                break;
            }
            q = (q + 1) & mask;
        }
        if (!found) atomicAdd(missing, 1ull);
    }
}

}  // namespace

// true when the distinct vector sets a (Fa x K) and b (Fb x K) are equal (exact compare)
bool same_value_set(Ctx& c, const double* a, long long Fa, const double* b, long long Fb, int K)
{
    if (Fa != Fb) return false;
    if (Fa == 0) return true;
    uint64_t size = 1;
    while (size < 2ull * static_cast<uint64_t>(Fa) + 16) size <<= 1;
    DevBuf<uint32_t> table;
    DevBuf<unsigned long long> miss;
    table.reserve(size);
    miss.reserve(1);
    ck(cudaMemsetAsync(table.p, 0xFF, sizeof(uint32_t) * size, c.stream), "memset");
    ck(cudaMemsetAsync(miss.p, 0, sizeof(unsigned long long), c.stream), "memset");
    k_set_insert<<<grid_blocks(Fa), 256, 0, c.stream>>>(a, Fa, K, table.p, size - 1);
    k_set_missing<<<grid_blocks(Fb), 256, 0, c.stream>>>(a, table.p, size - 1, b, Fb, K, miss.p);
    c.launches += 2;
    const unsigned long long m = read_counter(c, miss.p);
    table.release();
    miss.release();
    return m == 0;
}

}  // namespace momc_b200
