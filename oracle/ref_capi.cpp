// C-ABI wrapper around the UNMODIFIED reference headers — TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/build_ref.sh from /root/reference/proj/include (never copied) plus
// the Eigen-subset shim in oracle/eigen_shim, into oracle/_ref/libmomc_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs
// load it; the product path (paper_2604_26477_b200) never does.
//
// Every entry point forwards to the reference function named in its comment.
// Errors: 0 = ok, 2 = std::invalid_argument (usage), 1 = any other exception;
// the message is copied into `err`.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "momc/oracle.hpp"
#include "momc/pipeline.hpp"

using namespace momc;

namespace {

void put_err(char* err, std::size_t errlen, const char* msg)
{
    if (err && errlen) {
        std::strncpy(err, msg, errlen - 1);
        err[errlen - 1] = 0;
    }
}

template <class F>
int guarded(char* err, std::size_t errlen, F&& f)
{
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

struct CfgC {
    int variant;  // 0 bsb, 1 dsb, 2 simcim
    int n_iterations;
    double dt, a0, alpha;
    int batch_size;
    double init_scale;
    std::uint64_t seed;
    int threads;
};

SolverConfig to_cfg(const CfgC* c)
{
    SolverConfig s;
    s.variant = static_cast<SolverVariant>(c->variant);
    s.n_iterations = c->n_iterations;
    s.dt = c->dt;
    s.a0 = c->a0;
    s.alpha = c->alpha;
    s.batch_size = c->batch_size;
    s.init_scale = c->init_scale;
    s.seed = c->seed;
    s.threads = c->threads;
    return s;
}

std::vector<WeightVector> to_weights(const int* nums, int L, int k, int H)
{
    std::vector<WeightVector> w;
    w.reserve(static_cast<std::size_t>(L));
    for (int l = 0; l < L; ++l) {
        std::vector<int> v(nums + static_cast<std::size_t>(l) * k, nums + static_cast<std::size_t>(l + 1) * k);
        w.emplace_back(std::move(v), H);
    }
    return w;
}

SpinConfiguration unpack(const std::uint64_t* w, int n)
{
    std::vector<std::int8_t> s(static_cast<std::size_t>(n));
    for (int b = 0; b < n; ++b) s[static_cast<std::size_t>(b)] = (w[b / 64] >> (b % 64)) & 1u ? 1 : -1;
    return SpinConfiguration(std::move(s));
}

void pack(const SpinConfiguration& s, std::uint64_t* w)
{
    const int wpc = (s.size() + 63) / 64;
    for (int i = 0; i < wpc; ++i) w[i] = 0;
    for (int b = 0; b < s.size(); ++b) {
        if (s[b] > 0) w[b / 64] |= 1ull << (b % 64);
    }
}

SamplePool make_pool(const std::uint64_t* words, std::size_t M, int n)
{
    SamplePool pool(n);
    pool.resize(M);
    const int wpc = (n + 63) / 64;
    for (std::size_t i = 0; i < M; ++i) {
        pool.set_record(i, {0, 0, static_cast<std::uint32_t>(i), 0});
        pool.set_config(i, unpack(words + i * static_cast<std::size_t>(wpc), n));
    }
    return pool;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ rng.hpp
void momcref_philox(std::uint64_t key, const std::uint32_t* ctr, std::uint32_t* out)
{  // rng.hpp:22 Philox4x32::block
    const auto r = rng::Philox4x32::block(key, {ctr[0], ctr[1], ctr[2], ctr[3]});
    for (int i = 0; i < 4; ++i) out[i] = r[static_cast<std::size_t>(i)];
}
std::uint64_t momcref_derive_key(std::uint64_t seed, std::uint64_t ctx) { return rng::derive_key(seed, ctx); }
std::uint64_t momcref_run_key(std::uint64_t seed, std::uint32_t run) { return detail::run_key(seed, run); }
std::uint32_t momcref_tag_word(std::uint32_t tag, std::uint32_t step)
{
    return rng::tag_word(static_cast<rng::Tag>(tag), step);
}
void momcref_stream_u32(std::uint64_t key, std::uint32_t hi, std::uint32_t mid, std::uint32_t lo, int count,
                        std::uint32_t* out)
{
    rng::Stream s(key, hi, mid, lo);
    for (int i = 0; i < count; ++i) out[i] = s.next_u32();
}
void momcref_stream_normals(std::uint64_t key, std::uint32_t hi, std::uint32_t mid, std::uint32_t lo, int count,
                            double* out)
{  // rng.hpp:156 next_normal
    rng::Stream s(key, hi, mid, lo);
    for (int i = 0; i < count; ++i) out[i] = s.next_normal();
}
void momcref_stream_symmetric(std::uint64_t key, std::uint32_t hi, std::uint32_t mid, std::uint32_t lo, double h,
                              int count, double* out)
{  // rng.hpp:143 next_symmetric
    rng::Stream s(key, hi, mid, lo);
    for (int i = 0; i < count; ++i) out[i] = s.next_symmetric(h);
}
void momcref_ziggurat_tables(std::uint32_t* kn, double* wn, double* fn)
{  // rng.hpp:62 ZigguratTables
    const auto& z = rng::detail::ziggurat();
    for (int i = 0; i < 128; ++i) {
        kn[i] = z.kn[i];
        wn[i] = z.wn[i];
        fn[i] = z.fn[i];
    }
}

// ------------------------------------------------------------------ weights.hpp
int momcref_resolution_for_interior_count(int k, int count, char* err, std::size_t errlen)
{
    int h = -1;
    const int rc = guarded(err, errlen, [&] { h = resolution_for_interior_count(k, count); });
    return rc ? -rc : h;
}
// das_dennis (weights.hpp:75) [+ interior_filter (:100)]; returns the count, fills up to `cap` rows
long long momcref_das_dennis(int k, int h, int interior, int* out, long long cap, char* err, std::size_t errlen)
{
    long long count = 0;
    const int rc = guarded(err, errlen, [&] {
        auto lat = das_dennis(k, h);
        if (interior) lat = interior_filter(lat);
        count = static_cast<long long>(lat.size());
        for (long long i = 0; i < count && i < cap; ++i)
            for (int j = 0; j < k; ++j) out[i * k + j] = lat[static_cast<std::size_t>(i)].numerator(j);
    });
    return rc ? -rc : count;
}

// ------------------------------------------------------------------ instance.hpp
void* momcref_instance_new(int n, int k, int m, const int* ei, const int* ej, const double* w, char* err,
                           std::size_t errlen)
{
    MultiObjectiveInstance* p = nullptr;
    guarded(err, errlen, [&] {
        std::vector<Edge> edges(static_cast<std::size_t>(m));
        for (int e = 0; e < m; ++e) {
            edges[static_cast<std::size_t>(e)].i = ei[e];
            edges[static_cast<std::size_t>(e)].j = ej[e];
            edges[static_cast<std::size_t>(e)].w.assign(w + static_cast<std::size_t>(e) * k,
                                                        w + static_cast<std::size_t>(e + 1) * k);
        }
        p = new MultiObjectiveInstance(n, k, std::move(edges));
    });
    return p;
}
void* momcref_instance_load(const char* path, char* err, std::size_t errlen)
{  // instance.hpp:486 load_instance
    MultiObjectiveInstance* p = nullptr;
    guarded(err, errlen, [&] { p = new MultiObjectiveInstance(load_instance(path)); });
    return p;
}
void* momcref_instance_generate_uniform(int n, double density, int k, int kind, double lo, double hi,
                                        std::uint64_t seed, char* err, std::size_t errlen)
{  // instance.hpp:259 generate_uniform_instance
    MultiObjectiveInstance* p = nullptr;
    guarded(err, errlen, [&] {
        const WeightSpec spec = kind == 0 ? WeightSpec::uniform_int(static_cast<long>(lo), static_cast<long>(hi))
                                          : WeightSpec::uniform_real(lo, hi);
        p = new MultiObjectiveInstance(generate_uniform_instance(n, density, k, spec, seed));
    });
    return p;
}
void* momcref_instance_generate_correlated(int n, double density, double rho, std::uint64_t seed, char* err,
                                           std::size_t errlen)
{  // instance.hpp:364 generate_correlated_instance
    MultiObjectiveInstance* p = nullptr;
    guarded(err, errlen, [&] { p = new MultiObjectiveInstance(generate_correlated_instance(n, density, rho, seed)); });
    return p;
}
int momcref_measured_correlation(void* h, int pool_size, std::uint64_t seed, double* out, char* err, std::size_t errlen)
{  // instance.hpp:338
    return guarded(err, errlen, [&] {
        *out = measured_correlation(*static_cast<const MultiObjectiveInstance*>(h), pool_size, seed);
    });
}
void momcref_instance_dims(void* h, int* n, int* k, int* m)
{
    const auto* p = static_cast<const MultiObjectiveInstance*>(h);
    *n = p->n();
    *k = p->k();
    *m = p->num_edges();
}
void momcref_instance_edges(void* h, int* ei, int* ej, double* w)
{
    const auto* p = static_cast<const MultiObjectiveInstance*>(h);
    const int k = p->k();
    int e = 0;
    for (const auto& edge : p->edges()) {
        ei[e] = edge.i;
        ej[e] = edge.j;
        for (int l = 0; l < k; ++l) w[static_cast<std::size_t>(e) * k + l] = edge.w[static_cast<std::size_t>(l)];
        ++e;
    }
}
int momcref_instance_save(void* h, const char* path, char* err, std::size_t errlen)
{  // instance.hpp:473 save_instance
    return guarded(err, errlen, [&] { save_instance(*static_cast<const MultiObjectiveInstance*>(h), path); });
}
void momcref_instance_free(void* h) { delete static_cast<MultiObjectiveInstance*>(h); }

int momcref_cut_values(void* h, const std::uint64_t* words, std::size_t count, double* out, char* err,
                       std::size_t errlen)
{  // instance.hpp:183 cut_values, one config at a time
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        const int wpc = (inst.n() + 63) / 64;
        for (std::size_t c = 0; c < count; ++c) {
            const auto v = cut_values(inst, unpack(words + c * static_cast<std::size_t>(wpc), inst.n()));
            for (int l = 0; l < inst.k(); ++l) out[c * static_cast<std::size_t>(inst.k()) + static_cast<std::size_t>(l)] = v[l];
        }
    });
}

// ------------------------------------------------------------------ scalarize.hpp
int momcref_scalarize(void* h, const int* nums, int H, double* out_J, double* out_c0, char* err,
                      std::size_t errlen)
{  // scalarize.hpp:22 scalarize
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        const auto w = to_weights(nums, 1, inst.k(), H);
        const auto sc = scalarize(inst, w[0]);
        std::memcpy(out_J, sc.matrix.data(), sizeof(double) * static_cast<std::size_t>(inst.n()) * inst.n());
        *out_c0 = sc.c0;
    });
}

// ------------------------------------------------------------------ solver.hpp
int momcref_integrate_block(const double* J, int n, double c0, const CfgC* cfg, std::uint64_t key,
                            std::uint32_t weight, std::uint32_t traj, int count, double* out_x, double* out_y,
                            char* err, std::size_t errlen)
{  // solver.hpp:221 integrate_block
    return guarded(err, errlen, [&] {
        ScalarizedCoupling sc;
        sc.matrix.resize(n, n);
        std::memcpy(sc.matrix.data(), J, sizeof(double) * static_cast<std::size_t>(n) * n);
        sc.c0 = c0;
        const auto st = integrate_block(sc, to_cfg(cfg), StreamKey{key, weight, traj}, count);
        std::memcpy(out_x, st.x.data(), sizeof(double) * static_cast<std::size_t>(n) * count);
        std::memcpy(out_y, st.y.data(), sizeof(double) * static_cast<std::size_t>(n) * count);
    });
}
int momcref_init_state(const CfgC* cfg, int n, int count, std::uint64_t key, std::uint32_t weight,
                       std::uint32_t traj, double* out_x, double* out_y, char* err, std::size_t errlen)
{  // solver.hpp:108 init_state
    return guarded(err, errlen, [&] {
        const auto st = init_state(to_cfg(cfg), n, count, StreamKey{key, weight, traj});
        std::memcpy(out_x, st.x.data(), sizeof(double) * static_cast<std::size_t>(n) * count);
        std::memcpy(out_y, st.y.data(), sizeof(double) * static_cast<std::size_t>(n) * count);
    });
}
// run_sampler (solver.hpp:439). out_words: runs*L*batch*wpc; out_rec: 3 u32 per sample
// (run, weight, trajectory); out_stamp: timestamp_ns per sample (may be null);
// out_t: {model_construction_seconds, sampling_seconds}
int momcref_run_sampler(void* h, const int* nums, int L, int H, const CfgC* cfg, int runs, std::uint64_t* out_words,
                        std::uint32_t* out_rec, std::int64_t* out_stamp, double* out_t, char* err,
                        std::size_t errlen)
{
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        const auto pool = run_sampler(inst, to_weights(nums, L, inst.k(), H), to_cfg(cfg), runs);
        std::memcpy(out_words, pool.packed_words().data(), sizeof(std::uint64_t) * pool.packed_words().size());
        for (std::size_t i = 0; i < pool.size(); ++i) {
            const auto& r = pool.record(i);
            if (out_rec) {
                out_rec[3 * i] = r.run;
                out_rec[3 * i + 1] = r.weight;
                out_rec[3 * i + 2] = r.trajectory;
            }
            if (out_stamp) out_stamp[i] = r.timestamp_ns;
        }
        out_t[0] = pool.model_construction_seconds;
        out_t[1] = pool.sampling_seconds;
    });
}

// ------------------------------------------------------------------ pareto.hpp
// non_dominated_filter(pool, inst) (pareto.hpp:370) -> archive handle
void* momcref_filter_pool(void* h, const std::uint64_t* words, std::size_t M, int algo, char* err,
                          std::size_t errlen)
{
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    ParetoArchive* a = nullptr;
    guarded(err, errlen, [&] {
        const auto pool = make_pool(words, M, inst.n());
        a = new ParetoArchive(non_dominated_filter(pool, inst, static_cast<FilterAlgorithm>(algo)));
    });
    return a;
}
// non_dominated_filter(vector<ObjectiveVector>) (pareto.hpp:253); sense 0 cut, 1 hamiltonian
void* momcref_filter_values(const double* vals, std::size_t M, int k, int sense, int algo, char* err,
                            std::size_t errlen)
{
    ParetoArchive* a = nullptr;
    guarded(err, errlen, [&] {
        std::vector<ObjectiveVector> pool;
        pool.reserve(M);
        for (std::size_t i = 0; i < M; ++i)
            pool.emplace_back(std::vector<double>(vals + i * static_cast<std::size_t>(k), vals + (i + 1) * static_cast<std::size_t>(k)),
                              sense ? Sense::hamiltonian : Sense::cut);
        a = new ParetoArchive(non_dominated_filter(pool, static_cast<FilterAlgorithm>(algo)));
    });
    return a;
}
void* momcref_brute_force_pareto(void* h, char* err, std::size_t errlen)
{  // oracle.hpp:25
    ParetoArchive* a = nullptr;
    guarded(err, errlen, [&] { a = new ParetoArchive(brute_force_pareto(*static_cast<const MultiObjectiveInstance*>(h))); });
    return a;
}
void momcref_archive_dims(void* h, long long* F, int* k, int* n)
{
    const auto* a = static_cast<const ParetoArchive*>(h);
    *F = static_cast<long long>(a->size());
    *k = a->entries.empty() ? 0 : static_cast<int>(a->entries.front().value.size());
    *n = a->entries.empty() ? 0 : a->entries.front().config.size();
}
void momcref_archive_get(void* h, double* values, std::uint64_t* words, double* filtering_s)
{
    const auto* a = static_cast<const ParetoArchive*>(h);
    const int k = a->entries.empty() ? 0 : static_cast<int>(a->entries.front().value.size());
    const int n = a->entries.empty() ? 0 : a->entries.front().config.size();
    const int wpc = (n + 63) / 64;
    for (std::size_t i = 0; i < a->size(); ++i) {
        for (int l = 0; l < k; ++l) values[i * static_cast<std::size_t>(k) + static_cast<std::size_t>(l)] = a->entries[i].value[static_cast<std::size_t>(l)];
        if (words && n > 0) pack(a->entries[i].config, words + i * static_cast<std::size_t>(wpc));
    }
    if (filtering_s) *filtering_s = a->filtering_seconds;
}
void momcref_archive_free(void* h) { delete static_cast<ParetoArchive*>(h); }

// hypervolume (pareto.hpp:540; forced algorithm :557 when algo >= 0)
int momcref_hypervolume(const double* vals, long long F, int k, const double* r, int algo, double* out, char* err,
                        std::size_t errlen)
{
    return guarded(err, errlen, [&] {
        ParetoArchive a;
        for (long long i = 0; i < F; ++i)
            a.entries.push_back({std::vector<double>(vals + i * k, vals + (i + 1) * k), {}});
        const std::vector<double> rv(r, r + k);
        *out = algo < 0 ? hypervolume(a, rv) : hypervolume(a, rv, static_cast<HvAlgorithm>(algo));
    });
}
// detail::evaluate_cuts (pareto.hpp:330)
int momcref_evaluate_cuts(void* h, const std::uint64_t* words, std::size_t U, double* out, char* err,
                          std::size_t errlen)
{
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        const int wpc = (inst.n() + 63) / 64;
        std::vector<SpinConfiguration> cfgs;
        cfgs.reserve(U);
        for (std::size_t i = 0; i < U; ++i) cfgs.push_back(unpack(words + i * static_cast<std::size_t>(wpc), inst.n()));
        const auto cuts = detail::evaluate_cuts(inst, cfgs);
        for (std::size_t i = 0; i < U; ++i)
            for (int l = 0; l < inst.k(); ++l) out[i * static_cast<std::size_t>(inst.k()) + static_cast<std::size_t>(l)] = cuts[i][static_cast<std::size_t>(l)];
    });
}
int momcref_reference_point_sampled(void* h, int count, std::uint64_t seed, double* r, char* err, std::size_t errlen)
{  // pareto.hpp:620
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        const auto v = reference_point_sampled(inst, count, seed);
        for (std::size_t l = 0; l < v.size(); ++l) r[l] = v[l];
    });
}
int momcref_reference_point_exact(void* h, double* r, char* err, std::size_t errlen)
{  // pareto.hpp:603
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        const auto v = reference_point_exact(inst);
        for (std::size_t l = 0; l < v.size(); ++l) r[l] = v[l];
    });
}
// samples_to_reach (pareto.hpp:763); *out = -1 when never reached
int momcref_samples_to_reach(void* h, const std::uint64_t* words, std::size_t M, const double* r, double target,
                             long long* out, char* err, std::size_t errlen)
{
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        const auto pool = make_pool(words, M, inst.n());
        const auto hit = samples_to_reach(pool, inst, std::vector<double>(r, r + inst.k()), target);
        *out = hit ? static_cast<long long>(*hit) : -1;
    });
}

// convergence_trace (pareto.hpp:716); record i = {0, 0, i, stamps[i]}
int momcref_convergence_trace(void* h, const std::uint64_t* words, const long long* stamps, std::size_t M,
                              const double* r, int checkpoints, double* elapsed, double* hv, long long* samples,
                              char* err, std::size_t errlen)
{
    const auto& inst = *static_cast<const MultiObjectiveInstance*>(h);
    return guarded(err, errlen, [&] {
        auto pool = make_pool(words, M, inst.n());
        for (std::size_t i = 0; i < M; ++i) pool.set_record(i, {0, 0, static_cast<std::uint32_t>(i), stamps[i]});
        const auto t = convergence_trace(pool, inst, std::vector<double>(r, r + inst.k()), checkpoints);
        for (std::size_t i = 0; i < t.size(); ++i) {
            elapsed[i] = t[i].elapsed_s;
            hv[i] = t[i].hv;
            samples[i] = static_cast<long long>(t[i].samples);
        }
    });
}

// ------------------------------------------------------------------ CSV formats
// save_pool_csv (solver.hpp:357) of a pool built from words + records (rec3 = run, weight,
// trajectory per record) + stamps + timings
int momcref_save_pool_csv(const std::uint64_t* words, const std::uint32_t* rec3, const long long* stamps,
                          std::size_t M, int n, double mc, double ss, const char* path, char* err, std::size_t errlen)
{
    return guarded(err, errlen, [&] {
        SamplePool pool(n);
        pool.resize(M);
        const int wpc = (n + 63) / 64;
        for (std::size_t i = 0; i < M; ++i) {
            pool.set_record(i, {rec3[3 * i], rec3[3 * i + 1], rec3[3 * i + 2], stamps[i]});
            pool.set_config(i, unpack(words + i * static_cast<std::size_t>(wpc), n));
        }
        pool.model_construction_seconds = mc;
        pool.sampling_seconds = ss;
        save_pool_csv(pool, path);
    });
}
// load_pool_csv (solver.hpp:377): with cap < M only *M / *n / timings are returned
int momcref_load_pool_csv(const char* path, std::size_t* M, int* n, double* mc, double* ss, std::uint64_t* words,
                          std::uint32_t* rec3, long long* stamps, std::size_t cap, char* err, std::size_t errlen)
{
    return guarded(err, errlen, [&] {
        const auto pool = load_pool_csv(path);
        *M = pool.size();
        *n = pool.n();
        *mc = pool.model_construction_seconds;
        *ss = pool.sampling_seconds;
        if (cap < pool.size()) return;
        const int wpc = pool.words_per_config();
        for (std::size_t i = 0; i < pool.size(); ++i) {
            const auto& r = pool.record(i);
            rec3[3 * i] = r.run;
            rec3[3 * i + 1] = r.weight;
            rec3[3 * i + 2] = r.trajectory;
            stamps[i] = r.timestamp_ns;
            for (int w = 0; w < wpc; ++w) words[i * wpc + w] = pool.packed_words()[i * wpc + w];
        }
    });
}
// save_archive_csv (pareto.hpp:787): words == nullptr -> objective-only entries
int momcref_save_archive_csv(const double* vals, const std::uint64_t* words, std::size_t F, int k, int n, double fs,
                             const double* r, int nr, const char* path, char* err, std::size_t errlen)
{
    return guarded(err, errlen, [&] {
        ParetoArchive a;
        const int wpc = (n + 63) / 64;
        for (std::size_t i = 0; i < F; ++i) {
            ParetoArchive::Entry e;
            e.value.assign(vals + i * k, vals + (i + 1) * k);
            if (words) e.config = unpack(words + i * static_cast<std::size_t>(wpc), n);
            a.entries.push_back(std::move(e));
        }
        a.filtering_seconds = fs;
        a.reference.assign(r, r + nr);
        save_archive_csv(a, path);
    });
}
// load_archive_csv (pareto.hpp:823): with cap < F only the sizes are returned; has_cfg[i]
// marks entries with a configuration
int momcref_load_archive_csv(const char* path, std::size_t* F, int* k, int* n, double* fs, int* nr, double* r,
                             double* vals, std::uint64_t* words, unsigned char* has_cfg, std::size_t cap, char* err,
                             std::size_t errlen)
{
    return guarded(err, errlen, [&] {
        const auto a = load_archive_csv(path);
        *F = a.entries.size();
        *k = a.k();
        int nn = 0;
        for (const auto& e : a.entries) nn = std::max(nn, e.config.size());
        *n = nn;
        *fs = a.filtering_seconds;
        *nr = static_cast<int>(a.reference.size());
        for (std::size_t i = 0; i < a.reference.size() && i < 16; ++i) r[i] = a.reference[i];
        if (cap < a.entries.size()) return;
        const int wpc = (nn + 63) / 64;
        for (std::size_t i = 0; i < a.entries.size(); ++i) {
            const auto& e = a.entries[i];
            for (int l = 0; l < *k; ++l) vals[i * *k + l] = e.value[static_cast<std::size_t>(l)];
            has_cfg[i] = e.config.size() > 0;
            if (wpc && e.config.size() > 0) pack(e.config, words + i * wpc);
        }
    });
}

// ------------------------------------------------------------------ pipeline.hpp
// bench (pipeline.hpp:309) on a generated (instance_path == "" ) or loaded instance;
// writes format_report() into `report` and the pool words into out_words when non-null.
int momcref_bench(const char* instance_path, int n, double density, int k, std::uint64_t instance_seed,
                  const CfgC* cfg, int weight_count, int weight_resolution, int runs, const char* ref,
                  int checkpoints, char* report, std::size_t report_len, char* err, std::size_t errlen)
{
    return guarded(err, errlen, [&] {
        BenchConfig bc;
        bc.instance_path = instance_path ? instance_path : "";
        bc.n = n;
        bc.density = density;
        bc.k = k;
        bc.instance_seed = instance_seed;
        bc.solver = to_cfg(cfg);
        bc.weights.count = weight_count;
        bc.weights.resolution = weight_resolution;
        bc.runs = runs;
        bc.ref = ref;
        bc.checkpoints = checkpoints;
        const auto res = bench(bc);
        put_err(report, report_len, format_report(res.report).c_str());
    });
}

}  // extern "C"
