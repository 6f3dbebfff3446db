// Pool CSV rows on the device: the record lines of save_pool_csv
// (solver.hpp:357-375) and load_pool_csv (solver.hpp:377-432). The two header lines are
// host work (Python mirror); the rows — 1e6..1e8 of them at C2..C5 — are formatted and
// parsed here: byte work bound by HBM, one thread per row, offsets from a device scan.
//   row  = run ',' weight ',' trajectory ',' timestamp_ns ',' hex(words) '\n'
//   hex  = per word, 16 lowercase nibbles from the most significant (solver.hpp:342-353)
// Parsing mirrors the reference's getline(',') + std::stoul / std::stoll (leading
// whitespace, optional sign, trailing garbage ignored, range errors) and its two messages
// ("malformed pool record", "bad spin field width"), reported for the first bad line.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <string>
#include <vector>

#include "ctx.cuh"

namespace momc_b200 {

namespace {

unsigned grid_for(long long n, int t = 256)
{
    long long b = (n + t - 1) / t;
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>(b, 148ll * 32)));
}

__device__ __forceinline__ int udigits(unsigned long long v)
{
    int d = 1;
    while (v >= 10) {
        v /= 10;
        ++d;
    }
    return d;
}

__device__ __forceinline__ int sdigits(long long v)
{
    return v < 0 ? 1 + udigits(0ull - static_cast<unsigned long long>(v)) : udigits(static_cast<unsigned long long>(v));
}

__device__ __forceinline__ char* put_u(char* p, unsigned long long v)
{
    const int d = udigits(v);
    for (int q = d - 1; q >= 0; --q) {
        p[q] = static_cast<char>('0' + v % 10);
        v /= 10;
    }
    return p + d;
}

__device__ __forceinline__ char* put_s(char* p, long long v)
{
    if (v < 0) {
        *p++ = '-';
        return put_u(p, 0ull - static_cast<unsigned long long>(v));
    }
    return put_u(p, static_cast<unsigned long long>(v));
}

__global__ void k_row_len(const uint32_t* __restrict__ run, const uint32_t* __restrict__ wt,
                          const uint32_t* __restrict__ tr, const int64_t* __restrict__ ts, long long M, int wpc,
                          unsigned long long* len)
{
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < M;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        len[i] = udigits(run[i]) + udigits(wt[i]) + udigits(tr[i]) + sdigits(ts[i]) + 4 + 16 * wpc + 1;
}

__global__ void k_row_write(const uint32_t* __restrict__ run, const uint32_t* __restrict__ wt,
                            const uint32_t* __restrict__ tr, const int64_t* __restrict__ ts,
                            const uint64_t* __restrict__ words, long long M, int wpc,
                            const unsigned long long* __restrict__ off, char* out)
{
    const char* digits = "0123456789abcdef";
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < M;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        char* p = out + off[i];
        p = put_u(p, run[i]);
        *p++ = ',';
        p = put_u(p, wt[i]);
        *p++ = ',';
        p = put_u(p, tr[i]);
        *p++ = ',';
        p = put_s(p, ts[i]);
        *p++ = ',';
        for (int w = 0; w < wpc; ++w) {
            const uint64_t v = words[i * wpc + w];
            for (int nib = 15; nib >= 0; --nib) *p++ = digits[(v >> (4 * nib)) & 0xF];
        }
        *p = '\n';
    }
}

// ---- parsing
constexpr int kSeg = 4096;  // bytes per newline-count segment

__global__ void k_nl_count(const char* __restrict__ t, long long len, unsigned long long* cnt)
{
    const long long seg = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long a = seg * kSeg;
    if (a >= len) return;
    const long long b = min(len, a + kSeg);
    unsigned long long c = 0;
    for (long long q = a; q < b; ++q) c += t[q] == '\n';
    cnt[seg] = c;
}

__global__ void k_nl_write(const char* __restrict__ t, long long len, const unsigned long long* __restrict__ base,
                           long long* pos)
{
    const long long seg = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long a = seg * kSeg;
    if (a >= len) return;
    const long long b = min(len, a + kSeg);
    unsigned long long o = base[seg];
    for (long long q = a; q < b; ++q)
        if (t[q] == '\n') pos[o++] = q;
}

__device__ __forceinline__ bool is_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

// std::stoul / std::stoll on the cell [p, e): false on "no conversion" or out of range
__device__ bool parse_ul(const char* p, const char* e, unsigned long long& out)
{
    while (p < e && is_space(*p)) ++p;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p >= e || *p < '0' || *p > '9') return false;
    unsigned long long v = 0;
    bool over = false;
    for (; p < e && *p >= '0' && *p <= '9'; ++p) {
        const unsigned d = *p - '0';
        if (v > (ULLONG_MAX - d) / 10) over = true;
        v = v * 10 + d;
    }
    if (over) return false;
    out = neg ? 0ull - v : v;  // strtoul negates in unsigned arithmetic
    return true;
}

__device__ bool parse_ll(const char* p, const char* e, long long& out)
{
    while (p < e && is_space(*p)) ++p;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p >= e || *p < '0' || *p > '9') return false;
    unsigned long long v = 0;
    const unsigned long long lim = neg ? 0x8000000000000000ull : 0x7FFFFFFFFFFFFFFFull;
    bool over = false;
    for (; p < e && *p >= '0' && *p <= '9'; ++p) {
        const unsigned d = *p - '0';
        if (v > (lim - d) / 10) over = true;
        if (!over) v = v * 10 + d;
    }
    if (over) return false;
    out = neg ? static_cast<long long>(0ull - v) : static_cast<long long>(v);
    return true;
}

// status: 0 empty line, 1 record, 2 malformed record, 3 bad spin field width
__device__ int parse_line(const char* s, const char* e, int n, int wpc, uint32_t* rec3, int64_t* ts, uint64_t* words)
{
    if (s == e) return 0;
    // five getline(row, cell, ',') calls: each fails when nothing is left to extract
    const char* cell[5];
    const char* cend[5];
    const char* p = s;
    for (int f = 0; f < 5; ++f) {
        if (p >= e) return 2;
        const char* q = p;
        while (q < e && *q != ',') ++q;
        cell[f] = p;
        cend[f] = q;
        p = q < e ? q + 1 : e;
    }
    unsigned long long v;
    for (int f = 0; f < 3; ++f) {
        if (!parse_ul(cell[f], cend[f], v)) return 2;
        if (rec3) rec3[f] = static_cast<uint32_t>(v);
    }
    long long t;
    if (!parse_ll(cell[3], cend[3], t)) return 2;
    if (ts) *ts = t;
    if (cend[4] - cell[4] != 16ll * wpc) return 3;
    if (words) {
        for (int w = 0; w < wpc; ++w) words[w] = 0;
        for (int b = 0; b < n; ++b) {
            const int word = b / 64;
            const int nib = 15 - (b % 64) / 4;
            const signed char ch = static_cast<signed char>(cell[4][word * 16 + nib]);
            const int val = ch <= '9' ? ch - '0' : ch - 'a' + 10;
            if ((val >> (b % 4)) & 1) words[word] |= 1ull << (b % 64);
        }
    }
    return 1;
}

__device__ __forceinline__ void line_span(const char* t, long long len, const long long* nl, long long nnl, long long q,
                                          const char*& s, const char*& e)
{
    const long long a = q == 0 ? 0 : nl[q - 1] + 1;
    const long long b = q < nnl ? nl[q] : len;
    s = t + a;
    e = t + b;
}

__global__ void k_parse_status(const char* __restrict__ t, long long len, const long long* __restrict__ nl,
                               long long nnl, long long L, int n, int wpc, unsigned* ok, unsigned long long* first_bad)
{
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < L;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const char *s, *e;
        line_span(t, len, nl, nnl, q, s, e);
        const int st = parse_line(s, e, n, wpc, nullptr, nullptr, nullptr);
        ok[q] = st == 1;
        if (st >= 2) atomicMin(first_bad, static_cast<unsigned long long>(q) << 2 | static_cast<unsigned long long>(st));
    }
}

__global__ void k_parse_write(const char* __restrict__ t, long long len, const long long* __restrict__ nl, long long nnl,
                              long long L, int n, int wpc, const unsigned* __restrict__ ok,
                              const unsigned* __restrict__ idx, uint32_t* run, uint32_t* wt, uint32_t* tr, int64_t* ts,
                              uint64_t* words)
{
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < L;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        if (!ok[q]) continue;
        const char *s, *e;
        line_span(t, len, nl, nnl, q, s, e);
        const long long o = idx[q];
        uint32_t r3[3];
        parse_line(s, e, n, wpc, r3, ts + o, words + o * wpc);
        run[o] = r3[0];
        wt[o] = r3[1];
        tr[o] = r3[2];
    }
}

struct ParsedPool {
    long long M = 0;
    int wpc = 0;
    DevBuf<uint32_t> run, wt, tr;
    DevBuf<int64_t> ts;
    DevBuf<uint64_t> words;
};

ParsedPool& parsed(Ctx& c)
{
    if (!c.csv_scratch) c.csv_scratch = std::shared_ptr<void>(new ParsedPool(), [](void* p) {
        auto* q = static_cast<ParsedPool*>(p);
        q->run.release();
        q->wt.release();
        q->tr.release();
        q->ts.release();
        q->words.release();
        delete q;
    });
    return *static_cast<ParsedPool*>(c.csv_scratch.get());
}

}  // namespace

// rows of save_pool_csv for M records (host arrays) into `out` (host, cap bytes); returns the
// byte count (with out == nullptr only the count)
size_t format_pool_rows(Ctx& c, const uint32_t* run, const uint32_t* wt, const uint32_t* tr, const int64_t* ts,
                        const uint64_t* words, long long M, int n, char* out, size_t cap)
{
    if (n < 1) usage("pool spin count must be positive");
    if (M == 0) return 0;
    const int wpc = (n + 63) / 64;
    DevBuf<uint32_t> dr, dw, dt;
    DevBuf<int64_t> ds;
    DevBuf<uint64_t> dwords;
    DevBuf<unsigned long long> len, off;
    dr.reserve(static_cast<size_t>(M));
    dw.reserve(static_cast<size_t>(M));
    dt.reserve(static_cast<size_t>(M));
    ds.reserve(static_cast<size_t>(M));
    len.reserve(static_cast<size_t>(M));
    off.reserve(static_cast<size_t>(M));
    ck(cudaMemcpyAsync(dr.p, run, sizeof(uint32_t) * M, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(dw.p, wt, sizeof(uint32_t) * M, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(dt.p, tr, sizeof(uint32_t) * M, cudaMemcpyHostToDevice, c.stream), "H2D");
    ck(cudaMemcpyAsync(ds.p, ts, sizeof(int64_t) * M, cudaMemcpyHostToDevice, c.stream), "H2D");
    k_row_len<<<grid_for(M), 256, 0, c.stream>>>(dr.p, dw.p, dt.p, ds.p, M, wpc, len.p);
    c.launches++;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, off.p, static_cast<int>(M), c.stream);
    DevBuf<unsigned char> tmp;
    tmp.reserve(tb + 1);
    ck(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, off.p, static_cast<int>(M), c.stream), "scan");
    unsigned long long last[2];
    ck(cudaMemcpyAsync(&last[0], off.p + M - 1, 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(&last[1], len.p + M - 1, 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "format");
    const size_t total = static_cast<size_t>(last[0] + last[1]);
    if (out) {
        if (cap < total) usage("output buffer too small for the pool rows");
        dwords.reserve(static_cast<size_t>(M) * wpc);
        ck(cudaMemcpyAsync(dwords.p, words, sizeof(uint64_t) * M * wpc, cudaMemcpyHostToDevice, c.stream), "H2D");
        DevBuf<char> text;
        text.reserve(total);
        k_row_write<<<grid_for(M), 256, 0, c.stream>>>(dr.p, dw.p, dt.p, ds.p, dwords.p, M, wpc, off.p, text.p);
        c.launches++;
        ck(cudaMemcpyAsync(out, text.p, total, cudaMemcpyDeviceToHost, c.stream), "D2H");
        ck(cudaStreamSynchronize(c.stream), "format");
        text.release();
    }
    for (auto* b : {&dr, &dw, &dt}) b->release();
    ds.release();
    dwords.release();
    len.release();
    off.release();
    tmp.release();
    return total;
}

// parse the record lines (the file after its two header lines; the first is line
// first_lineno) into the context's parsed-pool buffers; returns the record count
long long parse_pool_rows(Ctx& c, const char* text, size_t len, int n, int first_lineno, const std::string& path)
{
    if (n < 1) usage("pool spin count must be positive");
    ParsedPool& pp = parsed(c);
    pp.M = 0;
    pp.wpc = (n + 63) / 64;
    if (len == 0) return 0;
    DevBuf<char> dt;
    dt.reserve(len);
    ck(cudaMemcpyAsync(dt.p, text, len, cudaMemcpyHostToDevice, c.stream), "H2D");
    const long long segs = static_cast<long long>((len + kSeg - 1) / kSeg);
    DevBuf<unsigned long long> cnt, base;
    cnt.reserve(static_cast<size_t>(segs));
    base.reserve(static_cast<size_t>(segs));
    ck(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * segs, c.stream), "memset");
    k_nl_count<<<grid_for(segs, 128), 128, 0, c.stream>>>(dt.p, static_cast<long long>(len), cnt.p);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, base.p, static_cast<int>(segs), c.stream);
    DevBuf<unsigned char> tmp;
    tmp.reserve(tb + 1);
    ck(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, base.p, static_cast<int>(segs), c.stream), "scan");
    unsigned long long lastc[2];
    ck(cudaMemcpyAsync(&lastc[0], base.p + segs - 1, 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(&lastc[1], cnt.p + segs - 1, 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
    char lastch = 0;
    ck(cudaMemcpyAsync(&lastch, dt.p + len - 1, 1, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "parse");
    const long long nnl = static_cast<long long>(lastc[0] + lastc[1]);
    const long long L = nnl + (lastch != '\n' ? 1 : 0);  // std::getline: a final unterminated line counts
    DevBuf<long long> nl;
    nl.reserve(static_cast<size_t>(nnl) + 1);
    k_nl_write<<<grid_for(segs, 128), 128, 0, c.stream>>>(dt.p, static_cast<long long>(len), base.p, nl.p);
    DevBuf<unsigned> ok, idx;
    ok.reserve(static_cast<size_t>(L) + 1);
    idx.reserve(static_cast<size_t>(L) + 1);
    DevBuf<unsigned long long> bad;
    bad.reserve(1);
    const unsigned long long none = ~0ull;
    ck(cudaMemcpyAsync(bad.p, &none, 8, cudaMemcpyHostToDevice, c.stream), "H2D");
    k_parse_status<<<grid_for(L), 256, 0, c.stream>>>(dt.p, static_cast<long long>(len), nl.p, nnl, L, n, pp.wpc, ok.p,
                                                       bad.p);
    c.launches += 3;
    unsigned long long hb = 0;
    ck(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "parse");
    if (hb != ~0ull) {
        const long long line = static_cast<long long>(hb >> 2) + first_lineno;
        runtime(path + ":" + std::to_string(line) + ((hb & 3) == 3 ? ": bad spin field width" : ": malformed pool record"));
    }
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, ok.p, idx.p, static_cast<int>(L), c.stream);
    tmp.reserve(tb + 1);
    ck(cub::DeviceScan::ExclusiveSum(tmp.p, tb, ok.p, idx.p, static_cast<int>(L), c.stream), "scan");
    unsigned lastm[2];
    ck(cudaMemcpyAsync(&lastm[0], idx.p + L - 1, 4, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaMemcpyAsync(&lastm[1], ok.p + L - 1, 4, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "parse");
    const long long M = static_cast<long long>(lastm[0]) + lastm[1];
    pp.run.reserve(static_cast<size_t>(M) + 1);
    pp.wt.reserve(static_cast<size_t>(M) + 1);
    pp.tr.reserve(static_cast<size_t>(M) + 1);
    pp.ts.reserve(static_cast<size_t>(M) + 1);
    pp.words.reserve(static_cast<size_t>(M) * pp.wpc + 1);
    k_parse_write<<<grid_for(L), 256, 0, c.stream>>>(dt.p, static_cast<long long>(len), nl.p, nnl, L, n, pp.wpc, ok.p,
                                                      idx.p, pp.run.p, pp.wt.p, pp.tr.p, pp.ts.p, pp.words.p);
    c.launches++;
    ck(cudaStreamSynchronize(c.stream), "parse");
    pp.M = M;
    dt.release();
    cnt.release();
    base.release();
    tmp.release();
    nl.release();
    ok.release();
    idx.release();
    bad.release();
    return M;
}

void parsed_pool_get(Ctx& c, uint32_t* run, uint32_t* wt, uint32_t* tr, int64_t* ts, uint64_t* words)
{
    ParsedPool& pp = parsed(c);
    const long long M = pp.M;
    if (M == 0) return;
    if (run) ck(cudaMemcpyAsync(run, pp.run.p, sizeof(uint32_t) * M, cudaMemcpyDeviceToHost, c.stream), "D2H");
    if (wt) ck(cudaMemcpyAsync(wt, pp.wt.p, sizeof(uint32_t) * M, cudaMemcpyDeviceToHost, c.stream), "D2H");
    if (tr) ck(cudaMemcpyAsync(tr, pp.tr.p, sizeof(uint32_t) * M, cudaMemcpyDeviceToHost, c.stream), "D2H");
    if (ts) ck(cudaMemcpyAsync(ts, pp.ts.p, sizeof(int64_t) * M, cudaMemcpyDeviceToHost, c.stream), "D2H");
    if (words)
        ck(cudaMemcpyAsync(words, pp.words.p, sizeof(uint64_t) * M * pp.wpc, cudaMemcpyDeviceToHost, c.stream), "D2H");
    ck(cudaStreamSynchronize(c.stream), "parsed pool");
}

}  // namespace momc_b200
