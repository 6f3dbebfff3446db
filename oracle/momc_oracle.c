/*
 * momc_oracle.c — CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Plain C11 restatement of /root/reference/proj/include/momc (rng, weights, scalarize,
 * solver, pareto) used as the parity checker for the CUDA path. Each function cites the
 * reference file:line it follows. It is pinned against the reference itself (built
 * unmodified into oracle/_ref/libmomc_ref.so) and the reference's golden vectors in
 * tests/test_oracle_pin.py. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it; the product path never does.
 *
 * FP64 evaluation order follows oracle/eigen_shim/Eigen/Dense (compiled with
 * -ffp-contract=off): products rounded before every add, k-ascending GEMM sums.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng.hpp */
/* rng.hpp:22-38 Philox4x32::block (10 rounds, key bumped after each round) */
void oracle_philox(uint64_t key, const uint32_t in[4], uint32_t out[4])
{
    uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.hpp:42-50 mix64 (SplitMix64 finaliser) */
static uint64_t mix64(uint64_t z)
{
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

/* rng.hpp:54-57 derive_key */
uint64_t oracle_derive_key(uint64_t seed, uint64_t ctx)
{
    return mix64(seed + 0x9E3779B97F4A7C15ull) ^ mix64(ctx * 0x9E3779B97F4A7C15ull + 1);
}

/* solver.hpp:98-104 run_key */
uint64_t oracle_run_key(uint64_t seed, uint32_t run)
{
    return oracle_derive_key(oracle_derive_key(seed, 0x736F6C76u), run);
}

/* rng.hpp:208-211 tag_word */
uint32_t oracle_tag_word(uint32_t tag, uint32_t step) { return (tag << 26) | (step & 0x03FFFFFFu); }

/* rng.hpp:62-89 ZigguratTables (same libm calls, same order => identical tables) */
static uint32_t zkn[128];
static double zwn[128], zfn[128];
static pthread_once_t zonce = PTHREAD_ONCE_INIT;
static void zig_init(void)
{
    const double m1 = 2147483648.0;
    const double vn = 9.91256303526217e-3;
    double dn = 3.442619855899, tn = dn;
    const double q = vn / exp(-0.5 * dn * dn);
    zkn[0] = (uint32_t)((dn / q) * m1);
    zkn[1] = 0;
    zwn[0] = q / m1;
    zwn[127] = dn / m1;
    zfn[0] = 1.0;
    zfn[127] = exp(-0.5 * dn * dn);
    for (int i = 126; i >= 1; --i) {
        dn = sqrt(-2.0 * log(vn / dn + exp(-0.5 * dn * dn)));
        zkn[i + 1] = (uint32_t)((dn / tn) * m1);
        tn = dn;
        zfn[i] = exp(-0.5 * dn * dn);
        zwn[i] = dn / m1;
    }
}
void oracle_ziggurat_tables(uint32_t* kn, double* wn, double* fn)
{
    pthread_once(&zonce, zig_init);
    memcpy(kn, zkn, sizeof zkn);
    memcpy(wn, zwn, sizeof zwn);
    memcpy(fn, zfn, sizeof zfn);
}

/* rng.hpp:105-192 Stream: counter {block#, id_lo, id_mid, id_hi}, words consumed 0..3 */
typedef struct {
    uint64_t key;
    uint32_t ctr[4];
    uint32_t buf[4];
    int pos;
} stream_t;

static void stream_init(stream_t* s, uint64_t key, uint32_t hi, uint32_t mid, uint32_t lo)
{
    s->key = key;
    s->ctr[0] = 0; s->ctr[1] = lo; s->ctr[2] = mid; s->ctr[3] = hi;
    s->pos = 4;
}
static uint32_t next_u32(stream_t* s)
{
    if (s->pos == 4) {
        oracle_philox(s->key, s->ctr, s->buf);
        ++s->ctr[0];
        s->pos = 0;
    }
    return s->buf[s->pos++];
}
static uint64_t next_u64(stream_t* s)
{
    const uint64_t lo = next_u32(s);
    const uint64_t hi = next_u32(s);
    return lo | (hi << 32);
}
static double next_u01(stream_t* s) { return (double)(next_u64(s) >> 11) * 0x1.0p-53; }
static double next_u01_open(stream_t* s) { return (double)((next_u64(s) >> 11) + 1) * 0x1.0p-53; }
static double next_symmetric(stream_t* s, double h) { return h * (2.0 * next_u01(s) - 1.0); }
static uint64_t next_below(stream_t* s, uint64_t b)
{
    return (uint64_t)(((unsigned __int128)next_u64(s) * b) >> 64);
}
/* rng.hpp:156-185 next_normal (128-layer Marsaglia-Tsang ziggurat) */
static double next_normal(stream_t* s)
{
    for (;;) {
        const int32_t hz = (int32_t)next_u32(s);
        const uint32_t iz = (uint32_t)hz & 127u;
        const uint32_t mag = hz < 0 ? (uint32_t)(-(int64_t)hz) : (uint32_t)hz;
        if (mag < zkn[iz]) return hz * zwn[iz];
        if (iz == 0) {
            const double r = 3.442619855899;
            for (;;) {
                const double x = -log(next_u01_open(s)) / r;
                const double y = -log(next_u01_open(s));
                if (y + y >= x * x) return hz > 0 ? r + x : -(r + x);
            }
        }
        const double x = hz * zwn[iz];
        if (zfn[iz] + next_u01(s) * (zfn[iz - 1] - zfn[iz]) < exp(-0.5 * x * x)) return x;
    }
}

void oracle_stream_u32(uint64_t key, uint32_t hi, uint32_t mid, uint32_t lo, int count, uint32_t* out)
{
    stream_t s; stream_init(&s, key, hi, mid, lo);
    for (int i = 0; i < count; ++i) out[i] = next_u32(&s);
}
void oracle_stream_normals(uint64_t key, uint32_t hi, uint32_t mid, uint32_t lo, int count, double* out)
{
    pthread_once(&zonce, zig_init);
    stream_t s; stream_init(&s, key, hi, mid, lo);
    for (int i = 0; i < count; ++i) out[i] = next_normal(&s);
}
void oracle_stream_below(uint64_t key, uint32_t hi, uint32_t mid, uint32_t lo, uint64_t bound, int count,
                         uint64_t* out)
{
    stream_t s; stream_init(&s, key, hi, mid, lo);
    for (int i = 0; i < count; ++i) out[i] = next_below(&s, bound);
}

/* ------------------------------------------------------------------ weights.hpp */
static uint64_t binomial(int n, int k)
{  /* weights.hpp:12-21 */
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    uint64_t r = 1;
    for (int i = 1; i <= k; ++i) r = r * (uint64_t)(n - k + i) / (uint64_t)i;
    return r;
}
/* weights.hpp:110-117 resolution_for_interior_count; -1 on bad input */
int oracle_resolution_for_interior_count(int k, int count)
{
    if (k < 2 || count < 1) return -1;
    for (int h = k; h < 100000; ++h)
        if (binomial(h - 1, k - 1) >= (uint64_t)count) return h;
    return -1;
}
/* weights.hpp:75-96 das_dennis (lex-descending) + :100-107 interior_filter */
static void dd_rec(int k, int h, int pos, int rem, int* num, int interior, int* out, long long* cnt, long long cap)
{
    if (pos == k - 1) {
        num[pos] = rem;
        if (interior) {
            for (int j = 0; j < k; ++j)
                if (num[j] == 0) return;
        }
        if (*cnt < cap) memcpy(out + *cnt * k, num, sizeof(int) * (size_t)k);
        ++*cnt;
        return;
    }
    for (int v = rem; v >= 0; --v) {
        num[pos] = v;
        dd_rec(k, h, pos + 1, rem - v, num, interior, out, cnt, cap);
    }
}
long long oracle_das_dennis(int k, int h, int interior, int* out, long long cap)
{
    if (k < 2 || h < 1 || k > 64) return -1;
    int num[64];
    long long cnt = 0;
    dd_rec(k, h, 0, h, num, interior, out, &cnt, cap);
    return cnt;
}

/* ------------------------------------------------------------------ scalarize.hpp */
/* scalarize.hpp:22-39: J(c)_ij = ((0 + c0*w0) + c1*w1) + ..., c_k = num_k / H;
 * c0 = 1 / max_i |sum_j J_ij| (row sums j ascending). J is written row-major (symmetric).
 * Returns 0, or 2 for a degenerate normalisation. */
int oracle_scalarize(int n, int k, int m, const int* ei, const int* ej, const double* w, const int* nums, int H,
                     double* J, double* c0_out)
{
    memset(J, 0, sizeof(double) * (size_t)n * (size_t)n);
    for (int e = 0; e < m; ++e) {
        double v = 0;
        for (int l = 0; l < k; ++l) v += ((double)nums[l] / H) * w[(size_t)e * k + l];
        J[(size_t)ei[e] * n + ej[e]] = v;
        J[(size_t)ej[e] * n + ei[e]] = v;
    }
    double denom = 0;
    int first = 1;
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s = s + J[(size_t)i * n + j];
        const double a = fabs(s);
        if (first || a > denom) denom = a; /* maxCoeff: std::max running fold */
        first = 0;
    }
    if (!(denom > 0.0) || !isfinite(denom)) return 2;
    *c0_out = 1.0 / denom;
    return 0;
}

/* ------------------------------------------------------------------ solver.hpp */
typedef struct {
    int variant; /* 0 bsb, 1 dsb, 2 simcim */
    int n_iterations;
    double dt, a0, alpha;
    int batch_size;
    double init_scale;
    uint64_t seed;
    int threads;
} oracle_cfg;

/* One trajectory, solver.hpp:108-124 (init) + :152-183 (sb_step) + :188-214 (simcim_step)
 * + :221-234 (integrate_block). x/y: n doubles out. Returns 0, or the 1-based step at which
 * the state first became non-finite (solver.hpp:138-143 check_finite). */
int oracle_integrate_one(const double* J, int n, double c0, const oracle_cfg* cfg, uint64_t key, uint32_t weight,
                         uint32_t traj, double* x, double* y)
{
    pthread_once(&zonce, zig_init);
    stream_t sx, sy;
    stream_init(&sx, key, weight, traj, oracle_tag_word(1, 0));
    stream_init(&sy, key, weight, traj, oracle_tag_word(2, 0));
    for (int i = 0; i < n; ++i) x[i] = next_symmetric(&sx, cfg->init_scale);
    for (int i = 0; i < n; ++i) y[i] = next_symmetric(&sy, cfg->init_scale);
    double* coupled = (double*)malloc(sizeof(double) * (size_t)n * 3);
    double* noise = coupled + n;
    double* phi = noise + n;
    int bad = 0;
    const int T = cfg->n_iterations;
    for (int t = 0; t < T && !bad; ++t) {
        const double a_t = (double)(t + 1) / (double)T; /* solver.hpp:70-76 pump_schedule (a0 ignored) */
        for (int j = 0; j < n; ++j)
            phi[j] = cfg->variant == 1 ? (x[j] < 0.0 ? -1.0 : 1.0) : x[j];
        for (int i = 0; i < n; ++i) { /* GEMM row: k ascending from +0.0 */
            double s = 0.0;
            for (int j = 0; j < n; ++j) s = s + J[(size_t)i * n + j] * phi[j];
            coupled[i] = s;
        }
        if (cfg->alpha > 0.0) { /* solver.hpp:128-136 fill_step_noise */
            stream_t sn;
            stream_init(&sn, key, weight, traj, oracle_tag_word(3, (uint32_t)t));
            for (int i = 0; i < n; ++i) noise[i] = next_normal(&sn);
        }
        if (cfg->variant == 2) {
            const double pump = -0.5 * (1.0 - a_t); /* solver.hpp:217 simcim_schedule */
            const double beta = 0.9;
            for (int i = 0; i < n; ++i) {
                double d = pump * x[i] - c0 * coupled[i];
                if (cfg->alpha > 0.0) d = d + cfg->alpha * noise[i];
                y[i] = beta * y[i] + (1.0 - beta) * d;
            }
            for (int i = 0; i < n; ++i) x[i] = x[i] + cfg->dt * y[i];
        } else {
            const double drift = cfg->a0 - a_t;
            for (int i = 0; i < n; ++i) {
                double d = -drift * x[i] - c0 * coupled[i];
                if (cfg->alpha > 0.0) d = d + cfg->alpha * noise[i];
                y[i] = y[i] + cfg->dt * d;
            }
            const double s = cfg->dt * cfg->a0;
            for (int i = 0; i < n; ++i) x[i] = x[i] + s * y[i];
            for (int i = 0; i < n; ++i) y[i] = fabs(x[i]) > 1.0 ? 0.0 : y[i];
        }
        for (int i = 0; i < n; ++i) { /* cwiseMax(-1).cwiseMin(1): std::max / std::min */
            double v = x[i];
            v = (v < -1.0) ? -1.0 : v;
            v = (1.0 < v) ? 1.0 : v;
            x[i] = v;
        }
        for (int i = 0; i < n; ++i)
            if (!isfinite(x[i]) || !isfinite(y[i])) bad = t + 1;
    }
    free(coupled);
    return bad;
}

/* solver.hpp:237-244 read_spins + :288-297 set_config packing (bit b set iff s_b = +1) */
static void pack_x(const double* x, int n, uint64_t* w)
{
    const int wpc = (n + 63) / 64;
    for (int i = 0; i < wpc; ++i) w[i] = 0;
    for (int b = 0; b < n; ++b)
        if (!(x[b] < 0.0)) w[b / 64] |= 1ull << (b % 64);
}

typedef struct {
    const double* Js; /* L blocks, row-major n x n each */
    const double* c0s;
    int n, L, runs, tasks_per_run, chunks;
    const oracle_cfg* cfg;
    uint64_t* words;
    int next;
    pthread_mutex_t mu;
    int err_step, err_run, err_weight;
} sampler_ctx;

static void* sampler_worker(void* arg)
{
    sampler_ctx* c = (sampler_ctx*)arg;
    const int n = c->n, wpc = (n + 63) / 64, batch = c->cfg->batch_size;
    double* x = (double*)malloc(sizeof(double) * (size_t)n * 2);
    double* y = x + n;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        const int task = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (task >= c->runs * c->tasks_per_run) break;
        const int run = task / c->tasks_per_run, rt = task % c->tasks_per_run;
        const int l = rt / c->chunks, ch = rt % c->chunks;
        const int first = ch * 512, count = batch - first < 512 ? batch - first : 512;
        const uint64_t key = oracle_run_key(c->cfg->seed, (uint32_t)run);
        for (int t = 0; t < count; ++t) {
            const int bad = oracle_integrate_one(c->Js + (size_t)l * n * n, n, c->c0s[l], c->cfg, key,
                                                 (uint32_t)l, (uint32_t)(first + t), x, y);
            if (bad) {
                pthread_mutex_lock(&c->mu);
                if (!c->err_step || run < c->err_run || (run == c->err_run && l < c->err_weight)) {
                    c->err_step = bad; c->err_run = run; c->err_weight = l;
                }
                pthread_mutex_unlock(&c->mu);
                break;
            }
            const size_t idx = ((size_t)run * c->L + l) * batch + first + t;
            pack_x(x, n, c->words + idx * wpc);
        }
    }
    free(x);
    return NULL;
}

/* solver.hpp:439-529 run_sampler: scalarise every weight (scalarize.hpp:62-71), then
 * (weight x 512-chunk) tasks per run over `threads` workers; canonical index
 * (run*L + l)*batch + traj. Returns 0, 2 (degenerate coupling) or 1 (numerical failure:
 * *err_info = {step, run, weight}). */
int oracle_run_sampler(int n, int k, int m, const int* ei, const int* ej, const double* w, const int* nums, int L,
                       int H, const oracle_cfg* cfg, int runs, int threads, uint64_t* words, int* err_info)
{
    double* Js = (double*)malloc(sizeof(double) * (size_t)L * n * n);
    double* c0s = (double*)malloc(sizeof(double) * (size_t)L);
    for (int l = 0; l < L; ++l) {
        if (oracle_scalarize(n, k, m, ei, ej, w, nums + (size_t)l * k, H, Js + (size_t)l * n * n, c0s + l)) {
            free(Js); free(c0s);
            return 2;
        }
    }
    sampler_ctx c;
    memset(&c, 0, sizeof c);
    c.Js = Js; c.c0s = c0s; c.n = n; c.L = L; c.runs = runs; c.cfg = cfg; c.words = words;
    c.chunks = (cfg->batch_size + 511) / 512;
    c.tasks_per_run = L * c.chunks;
    pthread_mutex_init(&c.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, sampler_worker, &c);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&c.mu);
    free(Js); free(c0s);
    if (c.err_step) {
        if (err_info) { err_info[0] = c.err_step; err_info[1] = c.err_run; err_info[2] = c.err_weight; }
        return 1;
    }
    return 0;
}

/* ------------------------------------------------------------------ instance.hpp / pareto.hpp eval */
/* instance.hpp:183-194 cut_values: edges in order, C_k += w_k when s_i != s_j (from 0.0) */
void oracle_cut_values(int n, int k, int m, const int* ei, const int* ej, const double* w, const uint64_t* words,
                       size_t count, double* out)
{
    const int wpc = (n + 63) / 64;
    for (size_t c = 0; c < count; ++c) {
        const uint64_t* wd = words + c * wpc;
        double* o = out + c * k;
        for (int l = 0; l < k; ++l) o[l] = 0.0;
        for (int e = 0; e < m; ++e) {
            const int si = (wd[ei[e] / 64] >> (ei[e] % 64)) & 1, sj = (wd[ej[e] / 64] >> (ej[e] % 64)) & 1;
            if (si != sj)
                for (int l = 0; l < k; ++l) o[l] += w[(size_t)e * k + l];
        }
    }
}

/* pareto.hpp:330-363 evaluate_cuts: JS = J_k S (k-ascending), h = 0.5 * S_c . JS_c (i ascending),
 * C_k = 0.5 * (W_k - h), W_k = layer_sum (instance.hpp:131-137, edge order). */
void oracle_evaluate_cuts(int n, int k, int m, const int* ei, const int* ej, const double* w,
                          const uint64_t* words, size_t count, double* out)
{
    const int wpc = (n + 63) / 64;
    double* J = (double*)calloc((size_t)n * n, sizeof(double));
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    for (int l = 0; l < k; ++l) {
        memset(J, 0, sizeof(double) * (size_t)n * n);
        double W = 0;
        for (int e = 0; e < m; ++e) {
            J[(size_t)ei[e] * n + ej[e]] = w[(size_t)e * k + l];
            J[(size_t)ej[e] * n + ei[e]] = w[(size_t)e * k + l];
            W += w[(size_t)e * k + l];
        }
        for (size_t c = 0; c < count; ++c) {
            const uint64_t* wd = words + c * wpc;
            for (int i = 0; i < n; ++i) s[i] = (wd[i / 64] >> (i % 64)) & 1 ? 1.0 : -1.0;
            double dot = 0.0;
            for (int i = 0; i < n; ++i) {
                double js = 0.0;
                for (int j = 0; j < n; ++j) js = js + J[(size_t)i * n + j] * s[j];
                dot = dot + s[i] * js;
            }
            const double h = 0.5 * dot;
            out[c * k + l] = 0.5 * (W - h);
        }
    }
    free(J); free(s);
}

/* ------------------------------------------------------------------ pareto.hpp filter */
static int g_k; /* qsort context (single-threaded use) */
static const double* g_vals;

static int cmp_lex_desc_idx(const void* a, const void* b)
{
    const double* x = g_vals + (size_t)(*(const size_t*)a) * g_k;
    const double* y = g_vals + (size_t)(*(const size_t*)b) * g_k;
    for (int l = 0; l < g_k; ++l) {
        if (x[l] > y[l]) return -1;
        if (x[l] < y[l]) return 1;
    }
    return 0;
}
static int vec_eq(const double* a, const double* b, int k)
{
    for (int l = 0; l < k; ++l)
        if (a[l] != b[l]) return 0;
    return 1;
}
/* pareto.hpp:49-57 dominates_max */
static int dominates_max(const double* a, const double* b, int k)
{
    int strict = 0;
    for (int l = 0; l < k; ++l) {
        if (a[l] < b[l]) return 0;
        if (a[l] > b[l]) strict = 1;
    }
    return strict;
}

/* Non-dominated subset of `cnt` DISTINCT vectors (row-major, k wide) sorted lexicographically
 * descending: pareto.hpp:148-237 fast_front_ordered semantics (any dominator precedes its
 * victim in that order, so a scan against the kept archive is exact). keep[i] = 1/0. */
static void front_sorted(const double* v, size_t cnt, int k, unsigned char* keep)
{
    size_t* arch = (size_t*)malloc(sizeof(size_t) * (cnt ? cnt : 1));
    size_t na = 0;
    for (size_t i = 0; i < cnt; ++i) {
        int dom = 0;
        for (size_t a = 0; a < na && !dom; ++a) dom = dominates_max(v + arch[a] * k, v + i * k, k);
        keep[i] = (unsigned char)!dom;
        if (!dom) arch[na++] = i;
    }
    free(arch);
}

/* sort rows lex-descending and drop exact duplicates (pareto.hpp:274-275); returns count */
static size_t sort_unique_desc(double* v, size_t cnt, int k)
{
    size_t* ord = (size_t*)malloc(sizeof(size_t) * (cnt ? cnt : 1));
    for (size_t i = 0; i < cnt; ++i) ord[i] = i;
    g_k = k; g_vals = v;
    qsort(ord, cnt, sizeof(size_t), cmp_lex_desc_idx);
    double* t = (double*)malloc(sizeof(double) * (cnt ? cnt : 1) * k);
    size_t u = 0;
    for (size_t i = 0; i < cnt; ++i) {
        const double* r = v + ord[i] * k;
        if (u && vec_eq(t + (u - 1) * k, r, k)) continue;
        memcpy(t + u * k, r, sizeof(double) * k);
        ++u;
    }
    memcpy(v, t, sizeof(double) * u * k);
    free(t); free(ord);
    return u;
}

/* pareto.hpp:253-293 non_dominated_filter(vector<ObjectiveVector>) for cut-sense vectors:
 * sort + unique + front; output (in place) the front sorted lex-descending. Returns F. */
size_t oracle_filter_values(double* vals, size_t cnt, int k)
{
    const size_t u = sort_unique_desc(vals, cnt, k);
    unsigned char* keep = (unsigned char*)malloc(u ? u : 1);
    front_sorted(vals, u, k, keep);
    size_t f = 0;
    for (size_t i = 0; i < u; ++i)
        if (keep[i]) memmove(vals + f++ * k, vals + i * k, sizeof(double) * k);
    free(keep);
    return f;
}

typedef struct {
    const uint64_t* w;
    int wpc;
} cfgcmp_ctx;
static cfgcmp_ctx g_cc;
static int cmp_words(const void* a, const void* b)
{
    const uint64_t* x = g_cc.w + (size_t)(*(const size_t*)a) * g_cc.wpc;
    const uint64_t* y = g_cc.w + (size_t)(*(const size_t*)b) * g_cc.wpc;
    for (int i = 0; i < g_cc.wpc; ++i) {
        if (x[i] < y[i]) return -1;
        if (x[i] > y[i]) return 1;
    }
    return 0;
}
/* instance.hpp:63-67 SpinConfiguration operator< : lexicographic over spins (index 0 first,
 * -1 < +1). Returns <0 when config a precedes b. */
static int spin_lex_cmp(const uint64_t* a, const uint64_t* b, int n)
{
    for (int i = 0; i < n; ++i) {
        const int sa = (a[i / 64] >> (i % 64)) & 1, sb = (b[i / 64] >> (i % 64)) & 1;
        if (sa != sb) return sa < sb ? -1 : 1;
    }
    return 0;
}

/* pareto.hpp:370-410 non_dominated_filter(pool, inst): dedup (:309-326), evaluate_cuts
 * (:330-363), collapse equal vectors onto the lex-smallest config (:383-387), front,
 * archive sorted lex-descending. Outputs F values (F x k) and configs (F x wpc); out
 * buffers must hold min(M, cap) rows. Returns F. */
size_t oracle_filter_pool(int n, int k, int m, const int* ei, const int* ej, const double* w,
                          const uint64_t* words, size_t M, double* out_vals, uint64_t* out_words)
{
    const int wpc = (n + 63) / 64;
    size_t* ord = (size_t*)malloc(sizeof(size_t) * (M ? M : 1));
    for (size_t i = 0; i < M; ++i) ord[i] = i;
    g_cc.w = words; g_cc.wpc = wpc;
    qsort(ord, M, sizeof(size_t), cmp_words);
    uint64_t* uw = (uint64_t*)malloc(sizeof(uint64_t) * (M ? M : 1) * wpc);
    size_t U = 0;
    for (size_t i = 0; i < M; ++i) {
        const uint64_t* r = words + ord[i] * wpc;
        if (U && memcmp(uw + (U - 1) * wpc, r, sizeof(uint64_t) * wpc) == 0) continue;
        memcpy(uw + U * wpc, r, sizeof(uint64_t) * wpc);
        ++U;
    }
    free(ord);
    double* cv = (double*)malloc(sizeof(double) * (U ? U : 1) * k);
    oracle_evaluate_cuts(n, k, m, ei, ej, w, uw, U, cv);
    /* collapse: order by value desc; within equal values keep the lex-smallest config */
    size_t* o2 = (size_t*)malloc(sizeof(size_t) * (U ? U : 1));
    for (size_t i = 0; i < U; ++i) o2[i] = i;
    g_k = k; g_vals = cv;
    qsort(o2, U, sizeof(size_t), cmp_lex_desc_idx);
    double* vv = (double*)malloc(sizeof(double) * (U ? U : 1) * k);
    size_t* owner = (size_t*)malloc(sizeof(size_t) * (U ? U : 1));
    size_t V = 0;
    for (size_t i = 0; i < U; ++i) {
        const size_t c = o2[i];
        if (V && vec_eq(vv + (V - 1) * k, cv + c * k, k)) {
            if (spin_lex_cmp(uw + c * wpc, uw + owner[V - 1] * wpc, n) < 0) owner[V - 1] = c;
            continue;
        }
        memcpy(vv + V * k, cv + c * k, sizeof(double) * k);
        owner[V++] = c;
    }
    unsigned char* keep = (unsigned char*)malloc(V ? V : 1);
    front_sorted(vv, V, k, keep);
    size_t F = 0;
    for (size_t i = 0; i < V; ++i) {
        if (!keep[i]) continue;
        memcpy(out_vals + F * k, vv + i * k, sizeof(double) * k);
        memcpy(out_words + F * wpc, uw + owner[i] * wpc, sizeof(uint64_t) * wpc);
        ++F;
    }
    free(keep); free(owner); free(vv); free(o2); free(cv); free(uw);
    return F;
}

/* ------------------------------------------------------------------ pareto.hpp hypervolume */
/* exact HV of points (gains, cnt x k) — restates the dispatch of pareto.hpp:540-552:
 * K=1 max (:544-548), K=2 sweep (:430-442), K=3 dimension sweep (:458-480) over a 2-d
 * staircase, K>=4 WFG recursion (:482-524). */
static double hv2(double* g, size_t cnt)
{
    g_k = 2; g_vals = g;
    size_t* o = (size_t*)malloc(sizeof(size_t) * (cnt ? cnt : 1));
    for (size_t i = 0; i < cnt; ++i) o[i] = i;
    qsort(o, cnt, sizeof(size_t), cmp_lex_desc_idx);
    double hv = 0, best1 = 0;
    for (size_t i = 0; i < cnt; ++i) {
        const double* p = g + o[i] * 2;
        if (p[1] > best1) {
            hv += p[0] * (p[1] - best1);
            best1 = p[1];
        }
    }
    free(o);
    return hv;
}

static int cmp_g2_desc(const void* a, const void* b)
{
    const double x = g_vals[(*(const size_t*)a) * 3 + 2], y = g_vals[(*(const size_t*)b) * 3 + 2];
    return x > y ? -1 : (x < y ? 1 : 0);
}

/* staircase as arrays: keys g0 strictly descending, values g1 strictly ascending */
static double hv3(double* g, size_t cnt)
{
    size_t* o = (size_t*)malloc(sizeof(size_t) * (cnt ? cnt : 1));
    for (size_t i = 0; i < cnt; ++i) o[i] = i;
    g_vals = g;
    qsort(o, cnt, sizeof(size_t), cmp_g2_desc); /* std::sort: stability irrelevant for the result */
    double* sk = (double*)malloc(sizeof(double) * (cnt + 1));
    double* sv = (double*)malloc(sizeof(double) * (cnt + 1));
    size_t ns = 0;
    double hv = 0;
    size_t i = 0;
    while (i < cnt) {
        const double level = g[o[i] * 3 + 2];
        for (; i < cnt && g[o[i] * 3 + 2] == level; ++i) {
            const double a = g[o[i] * 3], b = g[o[i] * 3 + 1];
            /* lower_bound(a) under greater<>: first key <= a */
            size_t lb = 0;
            while (lb < ns && sk[lb] > a) ++lb;
            const double covered = lb == 0 ? 0.0 : sv[lb - 1];
            if (b <= covered) continue;
            size_t e = lb;
            while (e < ns && sv[e] <= b) ++e; /* erase [lb, e) */
            if (e == lb && lb < ns && sk[lb] == a) { /* std::map operator[] overwrites */
                sv[lb] = b;
                continue;
            }
            memmove(sk + lb + 1, sk + e, sizeof(double) * (ns - e));
            memmove(sv + lb + 1, sv + e, sizeof(double) * (ns - e));
            ns = ns - (e - lb) + 1;
            sk[lb] = a;
            sv[lb] = b;
        }
        const double next = i < cnt ? g[o[i] * 3 + 2] : 0.0;
        double area = 0, prev = 0;
        for (size_t s = 0; s < ns; ++s) {
            area += sk[s] * (sv[s] - prev);
            prev = sv[s];
        }
        hv += area * (level - next);
    }
    free(sk); free(sv); free(o);
    return hv;
}

static double hv_wfg(double* g, size_t cnt, int k);

static double inclusive(const double* p, int k)
{
    double v = 1;
    for (int l = 0; l < k; ++l) v *= p[l];
    return v;
}

/* pareto.hpp:492-511 exclusive_volume */
static double exclusive(const double* p, const double* rest, size_t nrest, int k)
{
    if (nrest == 0) return inclusive(p, k);
    double* lim = (double*)malloc(sizeof(double) * nrest * k);
    for (size_t q = 0; q < nrest; ++q)
        for (int l = 0; l < k; ++l) lim[q * k + l] = rest[q * k + l] < p[l] ? rest[q * k + l] : p[l];
    const size_t u = sort_unique_desc(lim, nrest, k);
    unsigned char* keep = (unsigned char*)malloc(u ? u : 1);
    front_sorted(lim, u, k, keep);
    size_t f = 0;
    for (size_t i = 0; i < u; ++i)
        if (keep[i]) memmove(lim + f++ * k, lim + i * k, sizeof(double) * k);
    free(keep);
    const double v = inclusive(p, k) - hv_wfg(lim, f, k);
    free(lim);
    return v;
}

/* pareto.hpp:513-524 hv_wfg_gains */
static double hv_wfg(double* g, size_t cnt, int k)
{
    if (cnt == 0) return 0;
    if (cnt == 1) return inclusive(g, k);
    if (k == 2) return hv2(g, cnt);
    g_k = k; g_vals = g;
    size_t* o = (size_t*)malloc(sizeof(size_t) * cnt);
    for (size_t i = 0; i < cnt; ++i) o[i] = i;
    qsort(o, cnt, sizeof(size_t), cmp_lex_desc_idx);
    double* s = (double*)malloc(sizeof(double) * cnt * k);
    for (size_t i = 0; i < cnt; ++i) memcpy(s + i * k, g + o[i] * k, sizeof(double) * k);
    free(o);
    double hv = 0;
    for (size_t i = 0; i < cnt; ++i) hv += exclusive(s + i * k, s + (i + 1) * k, cnt - i - 1, k);
    free(s);
    return hv;
}

/* hypervolume(archive, r) (pareto.hpp:540-552) after validate_reference (:103-118).
 * Returns 0, or 2 when r is not dominated (*bad = entry index * 64 + objective). */
int oracle_hypervolume(const double* vals, size_t F, int k, const double* r, double* out, long long* bad)
{
    if (F == 0) return 2;
    for (size_t i = 0; i < F; ++i)
        for (int l = 0; l < k; ++l)
            if (r[l] > vals[i * k + l]) {
                if (bad) *bad = (long long)i * 64 + l;
                return 2;
            }
    double* g = (double*)malloc(sizeof(double) * F * k);
    for (size_t i = 0; i < F; ++i)
        for (int l = 0; l < k; ++l) g[i * k + l] = vals[i * k + l] - r[l];
    double hv;
    if (k == 1) {
        hv = 0;
        for (size_t i = 0; i < F; ++i) hv = hv > g[i] ? hv : g[i];
    } else if (k == 2) {
        hv = hv2(g, F);
    } else if (k == 3) {
        hv = hv3(g, F);
    } else {
        hv = hv_wfg(g, F, k);
    }
    free(g);
    *out = hv;
    return 0;
}

/* pareto.hpp:620-642 reference_point_sampled: per-objective min of cut_values over `count`
 * configs from Stream(derive_key(seed, 0x70617265), c, 0, tag_word(reference_sample)). */
void oracle_reference_point_sampled(int n, int k, int m, const int* ei, const int* ej, const double* w, int count,
                                    uint64_t seed, double* r)
{
    const uint64_t key = oracle_derive_key(seed, 0x70617265u);
    const int wpc = (n + 63) / 64;
    uint64_t wd[64];
    double cv[64];
    for (int l = 0; l < k; ++l) r[l] = INFINITY;
    for (int c = 0; c < count; ++c) {
        stream_t s;
        stream_init(&s, key, (uint32_t)c, 0, oracle_tag_word(8, 0));
        for (int i = 0; i < wpc; ++i) wd[i] = next_u64(&s);
        if (n % 64) wd[wpc - 1] &= (1ull << (n % 64)) - 1;
        oracle_cut_values(n, k, m, ei, ej, w, wd, 1, cv);
        for (int l = 0; l < k; ++l) r[l] = cv[l] < r[l] ? cv[l] : r[l];
    }
}
