// Exact Pareto front by exhaustive enumeration on the device: brute_force_pareto
// (oracle.hpp:25-77) and reference_point_exact (pareto.hpp:603-617), without the reference's
// n <= 22 cap (enumerate.hpp:17) for integer-weight instances with n <= 64.
//
// The reference walks all 2^(n-1) configurations with s_0 = +1 in Gray-code order. Here the
// graph is split by a vertex separator S into parts A and B with no A-B edge, so for every
// assignment sigma of S the cut vector is C = C_A(s_A; sigma) + C_B(s_B; sigma), where C_A
// counts the edges inside A and between A and S (and S-S), C_B those touching B. Then:
//   * a part configuration whose part vector is dominated (>= everywhere, > somewhere) inside
//     its own class cannot be part of a front point, and among equal part vectors only the
//     lex-smallest part configuration can own a front point (the other bits are equal), so
//     each part reduces to its own front (with lex-min owners) per class;
//   * the front is the front of { a + b : a in front_A(sigma), b in front_B(sigma) } over all
//     sigma, with equal vectors collapsed onto the lex-smallest full configuration — the
//     reference's tie rule (oracle.hpp:43-58).
// Every piece runs through the device filter (filter_values_device), so the front, the
// owners and the lex-descending order are the same code as the sampled archive's. Exact for
// integer weights (all sums are integers < 2^31). reference_point_exact is the per-objective
// minimum, min over sigma of (min_A + min_B).
// Heavy-hex 42 (S = 3..4 spins, parts of ~20 spins) enumerates 2^41 configurations in
// ~10^7 part evaluations.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "pareto.cuh"

namespace momc_b200 {

DevArchive& resident_archive(Ctx& c);

namespace {

constexpr int kMaxK = 16;               // objectives (as pareto.cu)
constexpr int kMaxPartSpins = 34;             // 2^34 configurations per part and class
constexpr long long kChunk = 1ll << 24;        // configurations per enumeration launch
constexpr long long kPairChunk = 1ll << 25;    // candidate sums per launch

unsigned grid_for(long long n, int t = 256)
{
    long long b = (n + t - 1) / t;
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>(b, 148ll * 16)));
}

// part configurations t in [t0, t0 + cnt): spins U[q] take bit q of t (bit set = +1), the
// fixed bits are the class; cut values over the part's edges (int32, exact)
__global__ void k_enum_part(const int* __restrict__ U, int nu, uint64_t fixed, long long t0, long long cnt,
                            const int* __restrict__ ei, const int* __restrict__ ej, const int* __restrict__ wi,
                            int me, int K, double* vals, uint64_t* words, int* vmin)
{
    extern __shared__ int sh[];
    int* sei = sh;
    int* sej = sei + me;
    int* sw = sej + me;
    int* su = sw + me * K;
    for (int q = threadIdx.x; q < me; q += blockDim.x) {
        sei[q] = ei[q];
        sej[q] = ej[q];
    }
    for (int q = threadIdx.x; q < me * K; q += blockDim.x) sw[q] = wi[q];
    for (int q = threadIdx.x; q < nu; q += blockDim.x) su[q] = U[q];
    __syncthreads();
    int lmin[kMaxK];
    for (int l = 0; l < K; ++l) lmin[l] = INT_MAX;
    for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < cnt;
         r += static_cast<long long>(gridDim.x) * blockDim.x) {
        const unsigned long long t = static_cast<unsigned long long>(t0 + r);
        uint64_t w = fixed;
        for (int q = 0; q < nu; ++q) w |= ((t >> q) & 1ull) << su[q];
        int v[kMaxK];
        for (int l = 0; l < K; ++l) v[l] = 0;
        for (int e = 0; e < me; ++e) {
            const int cut = static_cast<int>(((w >> sei[e]) ^ (w >> sej[e])) & 1ull);
            for (int l = 0; l < K; ++l) v[l] += cut * sw[e * K + l];
        }
        for (int l = 0; l < K; ++l) {
            vals[r * K + l] = static_cast<double>(v[l]);
            lmin[l] = min(lmin[l], v[l]);
        }
        words[r] = w;
    }
    for (int l = 0; l < K; ++l) {
        int m = lmin[l];
        for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0 && m != INT_MAX) atomicMin(&vmin[l], m);
    }
}

// candidate sums: rows a in [a0, a0 + na) of A times all nb rows of B
__global__ void k_pair_sums(const double* __restrict__ av, const uint64_t* __restrict__ aw, long long a0, long long na,
                            const double* __restrict__ bv, const uint64_t* __restrict__ bw, long long nb, int K,
                            double* vals, uint64_t* words)
{
    const long long tot = na * nb;
    for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < tot;
         r += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long a = a0 + r / nb, b = r % nb;
        for (int l = 0; l < K; ++l) vals[r * K + l] = av[a * K + l] + bv[b * K + l];
        words[r] = aw[a] | bw[b];
    }
}

struct Part {
    std::vector<int> free_spins;  // enumerated spins (bit q of t -> spin free_spins[q])
    std::vector<int> ei, ej, w;   // the part's edges (w: me x K integers)
};

// A front with owners held in plain device buffers (so several can coexist).
struct Front {
    long long F = 0;
    DevBuf<double> vals;
    DevBuf<uint64_t> words;
    void release()
    {
        vals.release();
        words.release();
        F = 0;
    }
};

void take(Ctx& c, DevArchive& a, Front& f, int K)
{
    f.F = a.F;
    f.vals.reserve(static_cast<size_t>(a.F) * K + 1);
    f.words.reserve(static_cast<size_t>(a.F) + 1);
    if (a.F) {
        ck(cudaMemcpyAsync(f.vals.p, a.vals.p, sizeof(double) * a.F * K, cudaMemcpyDeviceToDevice, c.stream), "D2D");
        ck(cudaMemcpyAsync(f.words.p, a.words.p, sizeof(uint64_t) * a.F, cudaMemcpyDeviceToDevice, c.stream), "D2D");
    }
}

// running = front(running U (vals, words)); tmp is scratch
void merge_into(Ctx& c, Front& running, const double* vals, const uint64_t* words, long long M, int K, DevArchive& tmp)
{
    if (M == 0) return;
    DevBuf<double> cv;
    DevBuf<uint64_t> cw;
    const long long tot = running.F + M;
    cv.reserve(static_cast<size_t>(tot) * K);
    cw.reserve(static_cast<size_t>(tot));
    if (running.F) {
        ck(cudaMemcpyAsync(cv.p, running.vals.p, sizeof(double) * running.F * K, cudaMemcpyDeviceToDevice, c.stream),
           "D2D");
        ck(cudaMemcpyAsync(cw.p, running.words.p, sizeof(uint64_t) * running.F, cudaMemcpyDeviceToDevice, c.stream),
           "D2D");
    }
    ck(cudaMemcpyAsync(cv.p + running.F * K, vals, sizeof(double) * M * K, cudaMemcpyDeviceToDevice, c.stream), "D2D");
    ck(cudaMemcpyAsync(cw.p + running.F, words, sizeof(uint64_t) * M, cudaMemcpyDeviceToDevice, c.stream), "D2D");
    filter_values_device(c, cv.p, cw.p, 1, c.n, tot, K, tmp, nullptr);
    take(c, tmp, running, K);
    cv.release();
    cw.release();
}

// front (with lex-min owners) of one part in one class; part minima added into vmin
void part_front(Ctx& c, const Part& p, uint64_t fixed, int K, Front& out, DevArchive& tmp, int* vmin, bool front)
{
    out.release();
    const int me = static_cast<int>(p.ei.size());
    const int nu = static_cast<int>(p.free_spins.size());
    if (me == 0) {  // no edges: the single zero vector, owned by the all -1 part assignment
        std::vector<double> z(static_cast<size_t>(K), 0.0);
        out.F = 1;
        out.vals.reserve(static_cast<size_t>(K));
        out.words.reserve(1);
        ck(cudaMemcpyAsync(out.vals.p, z.data(), sizeof(double) * K, cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cudaMemcpyAsync(out.words.p, &fixed, sizeof(uint64_t), cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cudaStreamSynchronize(c.stream), "sync");
        return;  // minima stay INT_MAX: read as 0 by the caller
    }
    DevBuf<int> dU, dei, dej, dw;
    dU.reserve(static_cast<size_t>(std::max(nu, 1)));
    dei.reserve(static_cast<size_t>(me));
    dej.reserve(static_cast<size_t>(me));
    dw.reserve(static_cast<size_t>(me) * K);
    if (nu) ck(cudaMemcpyAsync(dU.p, p.free_spins.data(), sizeof(int) * nu, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(dei.p, p.ei.data(), sizeof(int) * me, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(dej.p, p.ej.data(), sizeof(int) * me, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(dw.p, p.w.data(), sizeof(int) * me * K, cudaMemcpyHostToDevice, c.stream), "H2D");
    const long long total = 1ll << nu;
    const long long chunk = std::min(total, kChunk);
    DevBuf<double> v;
    DevBuf<uint64_t> w;
    v.reserve(static_cast<size_t>(chunk) * K);
    w.reserve(static_cast<size_t>(chunk));
    const size_t sm = sizeof(int) * (2 * me + me * K + nu);
    for (long long t0 = 0; t0 < total; t0 += chunk) {
        const long long cnt = std::min(chunk, total - t0);
        k_enum_part<<<grid_for(cnt), 256, sm, c.stream>>>(dU.p, nu, fixed, t0, cnt, dei.p, dej.p, dw.p, me, K, v.p, w.p,
                                                          vmin);
        c.launches++;
        ck(cudaGetLastError(), "enumerate");
        if (!front) continue;  // minima only (reference_point_exact)
        if (total == cnt) {
            filter_values_device(c, v.p, w.p, 1, c.n, cnt, K, tmp, nullptr);
            take(c, tmp, out, K);
        } else {
            merge_into(c, out, v.p, w.p, cnt, K, tmp);
        }
    }
    ck(cudaStreamSynchronize(c.stream), "enumerate");
    for (auto* b : {&dU, &dei, &dej, &dw}) b->release();
    v.release();
    w.release();
}

// Vertex separator by BFS-ball sweeps: for every start vertex and ball size, S = ball
// vertices with a neighbour outside, A = rest of the ball, B = outside. Cost model: classes x
// (part configurations of A + of B). Also the trivial split (A = everything).
struct Split {
    std::vector<int> S, A, B;
    double cost = 0;
};

double split_cost(const Split& s)
{
    auto part = [](size_t q) { return std::ldexp(1.0, static_cast<int>(q)); };
    const double cls = part(s.S.size());
    return cls * (part(s.A.size()) + (s.B.empty() ? 0.0 : part(s.B.size())));
}

Split choose_split(int n, const std::vector<std::vector<int>>& adj)
{
    Split best;
    best.A.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) best.A[static_cast<size_t>(i)] = i;
    best.cost = split_cost(best);
    for (int s0 = 0; s0 < n; ++s0) {
        std::vector<int> order;
        std::vector<char> seen(static_cast<size_t>(n), 0);
        // BFS from s0, then any unreached component in index order
        for (int root = s0, scanned = 0; static_cast<int>(order.size()) < n; ++scanned) {
            if (!seen[static_cast<size_t>(root)]) {
                seen[static_cast<size_t>(root)] = 1;
                size_t head = order.size();
                order.push_back(root);
                while (head < order.size()) {
                    const int u = order[head++];
                    for (int v : adj[static_cast<size_t>(u)])
                        if (!seen[static_cast<size_t>(v)]) {
                            seen[static_cast<size_t>(v)] = 1;
                            order.push_back(v);
                        }
                }
            }
            root = scanned % n;
        }
        std::vector<char> in(static_cast<size_t>(n), 0);
        for (int t = 1; t < n; ++t) {
            in[static_cast<size_t>(order[static_cast<size_t>(t - 1)])] = 1;
            Split s;
            for (int u = 0; u < n; ++u) {
                if (!in[static_cast<size_t>(u)]) {
                    s.B.push_back(u);
                    continue;
                }
                bool boundary = false;
                for (int v : adj[static_cast<size_t>(u)]) boundary |= !in[static_cast<size_t>(v)];
                (boundary ? s.S : s.A).push_back(u);
            }
            s.cost = split_cost(s);
            if (s.cost < best.cost) best = s;
        }
    }
    return best;
}

}  // namespace

// Exact front of the resident instance into the resident archive; r_exact (K) optional.
void brute_force_device(Ctx& c, std::vector<double>* r_exact, bool front)
{
    const int n = c.n, K = c.k;
    if (n < 1) usage("enumeration needs n >= 1");
    if (n > 64) usage("exhaustive enumeration on the device supports n <= 64 (got n=" + std::to_string(n) + ")");
    if (!c.integer_weights) usage("exhaustive enumeration on the device needs integer weights");
    if (K > kMaxK) usage("the GPU path supports at most 16 objectives");
    std::vector<std::vector<int>> adj(static_cast<size_t>(n));
    for (int e = 0; e < c.m; ++e) {
        adj[static_cast<size_t>(c.h_ei[static_cast<size_t>(e)])].push_back(c.h_ej[static_cast<size_t>(e)]);
        adj[static_cast<size_t>(c.h_ej[static_cast<size_t>(e)])].push_back(c.h_ei[static_cast<size_t>(e)]);
    }
    Split sp = choose_split(n, adj);
    // spin 0 is pinned to +1 (oracle.hpp:34): drop it from whichever set holds it
    auto drop0 = [](std::vector<int>& v) { v.erase(std::remove(v.begin(), v.end(), 0), v.end()); };
    std::vector<int> Sfree = sp.S;
    drop0(Sfree);
    Part pa, pb;
    pa.free_spins = sp.A;
    pb.free_spins = sp.B;
    drop0(pa.free_spins);
    drop0(pb.free_spins);
    if (static_cast<int>(pa.free_spins.size()) > kMaxPartSpins || static_cast<int>(pb.free_spins.size()) > kMaxPartSpins ||
        Sfree.size() > 24)
        usage("exhaustive enumeration too large for this graph (no small vertex separator)");
    std::vector<char> inB(static_cast<size_t>(n), 0);
    for (int u : sp.B) inB[static_cast<size_t>(u)] = 1;
    for (int e = 0; e < c.m; ++e) {
        const int i = c.h_ei[static_cast<size_t>(e)], j = c.h_ej[static_cast<size_t>(e)];
        Part& p = (inB[static_cast<size_t>(i)] || inB[static_cast<size_t>(j)]) ? pb : pa;
        p.ei.push_back(i);
        p.ej.push_back(j);
        for (int l = 0; l < K; ++l)
            p.w.push_back(static_cast<int>(c.h_w[static_cast<size_t>(e) * K + l]));
    }
    const bool haveB = !sp.B.empty();
    DevArchive tmp;
    Front fa, fb, total;
    DevBuf<int> vmin;
    vmin.reserve(static_cast<size_t>(2 * K));
    std::vector<long long> rmin(static_cast<size_t>(K), LLONG_MAX);
    const long long classes = 1ll << Sfree.size();
    DevBuf<double> pv;
    DevBuf<uint64_t> pw;
    for (long long sigma = 0; sigma < classes; ++sigma) {
        uint64_t fixed = 1ull;  // s_0 = +1
        for (size_t q = 0; q < Sfree.size(); ++q)
            if ((sigma >> q) & 1) fixed |= 1ull << Sfree[q];
        std::vector<int> init(static_cast<size_t>(2 * K), INT_MAX);
        ck(cudaMemcpyAsync(vmin.p, init.data(), sizeof(int) * 2 * K, cudaMemcpyHostToDevice, c.stream), "H2D");
        part_front(c, pa, fixed, K, fa, tmp, vmin.p, front);
        if (haveB) part_front(c, pb, fixed, K, fb, tmp, vmin.p + K, front);  // B minima: second half
        std::vector<int> hm(static_cast<size_t>(2 * K));
        ck(cudaMemcpyAsync(hm.data(), vmin.p, sizeof(int) * 2 * K, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "sync");
        for (int l = 0; l < K; ++l) {
            long long a = hm[static_cast<size_t>(l)] == INT_MAX ? 0 : hm[static_cast<size_t>(l)];
            long long b = (!haveB || hm[static_cast<size_t>(K + l)] == INT_MAX) ? 0 : hm[static_cast<size_t>(K + l)];
            rmin[static_cast<size_t>(l)] = std::min(rmin[static_cast<size_t>(l)], a + b);
        }
        if (!front) continue;
        if (!haveB) {
            merge_into(c, total, fa.vals.p, fa.words.p, fa.F, K, tmp);
            continue;
        }
        // B part words carry the class bits too: OR is still exact (same bits)
        const long long per = std::max<long long>(1, kPairChunk / std::max<long long>(1, fb.F));
        Front cls;
        for (long long a0 = 0; a0 < fa.F; a0 += per) {
            const long long na = std::min(per, fa.F - a0);
            const long long M = na * fb.F;
            pv.reserve(static_cast<size_t>(M) * K);
            pw.reserve(static_cast<size_t>(M));
            k_pair_sums<<<grid_for(M), 256, 0, c.stream>>>(fa.vals.p, fa.words.p, a0, na, fb.vals.p, fb.words.p, fb.F, K,
                                                           pv.p, pw.p);
            c.launches++;
            merge_into(c, cls, pv.p, pw.p, M, K, tmp);
        }
        merge_into(c, total, cls.vals.p, cls.words.p, cls.F, K, tmp);
        cls.release();
    }
    if (front) {  // the result as the resident archive (lex-descending, lex-min owners)
        DevArchive& out = resident_archive(c);
        filter_values_device(c, total.vals.p, total.words.p, 1, c.n, total.F, K, out, nullptr);
    }
    ck(cudaStreamSynchronize(c.stream), "enumerate");
    if (r_exact) {
        r_exact->resize(static_cast<size_t>(K));
        for (int l = 0; l < K; ++l) (*r_exact)[static_cast<size_t>(l)] = static_cast<double>(rmin[static_cast<size_t>(l)]);
    }
    fa.release();
    fb.release();
    total.release();
    pv.release();
    pw.release();
    vmin.release();
    tmp.vals.release();
    tmp.words.release();
}

}  // namespace momc_b200
