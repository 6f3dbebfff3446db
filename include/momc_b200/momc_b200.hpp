// momc_b200.hpp — C++ drop-in for the reference's hot-path interface (proj/include/momc),
// backed by the B200 C-ABI (include/momc_b200.h, libmomc_b200.so).
//
// Same types (momc::MultiObjectiveInstance, WeightVector, SolverConfig, SamplePool,
// ParetoArchive, ObjectiveVector from the reference headers), same signatures, same
// exceptions (std::invalid_argument for usage errors, std::runtime_error otherwise, with the
// reference's message text), in namespace momc::b200. A caller switches by replacing
// `momc::run_sampler(...)` with `momc::b200::run_sampler(...)` (or a using-declaration);
// see INTEGRATION.md. Replaced functions:
//   run_sampler                       solver.hpp:439-529
//   non_dominated_filter (pool)       pareto.hpp:370-410
//   non_dominated_filter (vectors)    pareto.hpp:253-293
//   detail::evaluate_cuts             pareto.hpp:330-363
//   hypervolume                       pareto.hpp:540-552
//   reference_point_sampled           pareto.hpp:620-642
//   scalarize                         scalarize.hpp:22-39   (as coupling(): J(c) and c0)
//   brute_force_pareto                oracle.hpp:25-77      (n <= 64 with a small separator)
//   reference_point_exact             pareto.hpp:603-617
#ifndef MOMC_B200_HPP
#define MOMC_B200_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "momc/pareto.hpp"
#include "momc/solver.hpp"
#include "momc_b200.h"

namespace momc::b200 {

namespace detail {

inline void raise(int rc, const char* err)
{
    if (rc == MOMC_OK) return;
    if (rc == MOMC_EUSAGE) throw std::invalid_argument(err);
    throw std::runtime_error(err);
}

struct InstanceArrays {
    std::vector<int32_t> ei, ej;
    std::vector<double> w;
    momc_instance_view view{};
    explicit InstanceArrays(const MultiObjectiveInstance& inst)
    {
        const int k = inst.k();
        for (const auto& e : inst.edges()) {
            ei.push_back(e.i);
            ej.push_back(e.j);
            w.insert(w.end(), e.w.begin(), e.w.end());
        }
        view = {inst.n(), k, inst.num_edges(), ei.data(), ej.data(), w.data()};
    }
};

inline std::pair<std::vector<int32_t>, int> weight_arrays(const std::vector<WeightVector>& weights, int k)
{
    std::vector<int32_t> nums;
    const int H = weights.empty() ? 1 : weights.front().resolution();
    for (const auto& wv : weights) {
        if (wv.size() != k) throw std::invalid_argument("weight vector length does not match objective count");
        if (wv.resolution() != H) throw std::invalid_argument("all weight vectors must share one resolution");
        for (int q = 0; q < k; ++q) nums.push_back(wv.numerator(q));
    }
    return {nums, H};
}

inline momc_solver_cfg cfg_of(const SolverConfig& c)
{
    return {static_cast<int>(c.variant), c.n_iterations, c.dt, c.a0, c.alpha, c.batch_size, c.init_scale, c.seed,
            c.threads};
}

inline SpinConfiguration unpack(const uint64_t* w, int n)
{
    std::vector<std::int8_t> s(static_cast<size_t>(n));
    for (int b = 0; b < n; ++b) s[static_cast<size_t>(b)] = (w[b / 64] >> (b % 64)) & 1u ? 1 : -1;
    return SpinConfiguration(std::move(s));
}

inline void pack(const SpinConfiguration& s, uint64_t* w)
{
    const int wpc = (s.size() + 63) / 64;
    for (int i = 0; i < wpc; ++i) w[i] = 0;
    for (int b = 0; b < s.size(); ++b)
        if (s[b] > 0) w[b / 64] |= 1ull << (b % 64);
}

}  // namespace detail

// One device context (stream + resident buffers). Movable, not copyable.
class Context {
public:
    explicit Context(int device = 0)
    {
        char err[1024] = {0};
        detail::raise(momc_b200_ctx_create(device, &h_, err, sizeof err), err);
    }
    ~Context()
    {
        if (h_) momc_b200_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    Context(Context&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    momc_ctx* get() const noexcept { return h_; }

private:
    momc_ctx* h_ = nullptr;
};

inline Context& default_context()
{
    static Context ctx(0);
    return ctx;
}

// solver.hpp:439-529
inline SamplePool run_sampler(const MultiObjectiveInstance& inst, const std::vector<WeightVector>& weights,
                              const SolverConfig& config, int runs, Context& ctx = default_context())
{
    config.validate();
    if (weights.empty()) throw std::invalid_argument("run_sampler needs at least one weight vector");
    if (runs < 1) throw std::invalid_argument("runs must be >= 1");
    detail::InstanceArrays ia(inst);
    auto [nums, H] = detail::weight_arrays(weights, inst.k());
    const int L = static_cast<int>(weights.size());
    const size_t M = static_cast<size_t>(runs) * L * config.batch_size;
    const int wpc = (inst.n() + 63) / 64;
    std::vector<uint64_t> words(M * wpc);
    std::vector<int64_t> stamps(M);
    double secs[2] = {0, 0};
    const momc_solver_cfg c = detail::cfg_of(config);
    char err[1024] = {0};
    detail::raise(momc_b200_run_sampler(ctx.get(), &ia.view, nums.data(), L, H, &c, runs, words.data(), stamps.data(),
                                        secs, err, sizeof err),
                  err);
    SamplePool pool(inst.n());
    pool.resize(M);
    for (size_t i = 0; i < M; ++i) {
        const size_t per_run = static_cast<size_t>(L) * config.batch_size;
        const auto run = static_cast<uint32_t>(i / per_run);
        const auto l = static_cast<uint32_t>((i % per_run) / config.batch_size);
        const auto t = static_cast<uint32_t>(i % config.batch_size);
        pool.set_record(i, {run, l, t, stamps[i]});
        pool.set_config(i, detail::unpack(&words[i * wpc], inst.n()));
    }
    pool.model_construction_seconds = secs[0];
    pool.sampling_seconds = secs[1];
    return pool;
}

inline ParetoArchive fetch_archive(Context& ctx, int k, int n)
{
    const int64_t F = momc_b200_archive_size(ctx.get());
    const int wpc = (n + 63) / 64;
    std::vector<double> vals(static_cast<size_t>(F) * k);
    std::vector<uint64_t> words(static_cast<size_t>(F) * (wpc ? wpc : 1));
    char err[1024] = {0};
    detail::raise(momc_b200_archive_get(ctx.get(), vals.data(), n ? words.data() : nullptr, err, sizeof err), err);
    ParetoArchive a;
    a.entries.reserve(static_cast<size_t>(F));
    for (int64_t i = 0; i < F; ++i) {
        ParetoArchive::Entry e;
        e.value.assign(vals.begin() + i * k, vals.begin() + (i + 1) * k);
        if (n) e.config = detail::unpack(&words[static_cast<size_t>(i) * wpc], n);
        a.entries.push_back(std::move(e));
    }
    return a;
}

// pareto.hpp:370-410 (the GPU front is exact; `algo` is accepted for signature parity)
inline ParetoArchive non_dominated_filter(const SamplePool& pool, const MultiObjectiveInstance& inst,
                                          FilterAlgorithm algo = FilterAlgorithm::fast, Context& ctx = default_context())
{
    (void)algo;
    if (pool.empty()) throw std::invalid_argument("non-dominated filter needs a non-empty pool");
    if (pool.n() != inst.n()) throw std::invalid_argument("pool does not match instance");
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    int64_t F = 0;
    double fs = 0;
    detail::raise(momc_b200_filter_pool(ctx.get(), pool.packed_words().data(), pool.size(), &F, &fs, err, sizeof err),
                  err);
    ParetoArchive a = fetch_archive(ctx, inst.k(), inst.n());
    a.filtering_seconds = fs;
    return a;
}

// pareto.hpp:253-293
inline ParetoArchive non_dominated_filter(const std::vector<ObjectiveVector>& pool,
                                          FilterAlgorithm algo = FilterAlgorithm::fast, Context& ctx = default_context())
{
    (void)algo;
    if (pool.empty()) throw std::invalid_argument("non-dominated filter needs a non-empty pool");
    const Sense sense = pool.front().sense();
    const int k = pool.front().size();
    std::vector<double> vals;
    vals.reserve(pool.size() * static_cast<size_t>(k));
    for (const auto& v : pool) {
        if (v.sense() != sense || v.size() != k) throw std::invalid_argument("pool mixes objective senses or lengths");
        vals.insert(vals.end(), v.values().begin(), v.values().end());
    }
    int64_t F = 0;
    char err[1024] = {0};
    detail::raise(momc_b200_filter_values(ctx.get(), vals.data(), pool.size(), k, sense == Sense::hamiltonian ? 1 : 0,
                                          &F, err, sizeof err),
                  err);
    return fetch_archive(ctx, k, 0);
}

// pareto.hpp:540-552
inline double hypervolume(const ParetoArchive& archive, const std::vector<double>& r, Context& ctx = default_context())
{
    if (archive.entries.empty()) throw std::invalid_argument("hypervolume of an empty archive");
    const int k = static_cast<int>(r.size());
    std::vector<double> vals;
    for (const auto& e : archive.entries) {
        if (static_cast<int>(e.value.size()) != k)
            throw std::invalid_argument("reference point length does not match archive");
        vals.insert(vals.end(), e.value.begin(), e.value.end());
    }
    double out = 0;
    char err[1024] = {0};
    detail::raise(momc_b200_hypervolume(ctx.get(), vals.data(), static_cast<int64_t>(archive.entries.size()), k,
                                        r.data(), &out, err, sizeof err),
                  err);
    return out;
}

// pareto.hpp:330-363
inline std::vector<std::vector<double>> evaluate_cuts(const MultiObjectiveInstance& inst,
                                                      const std::vector<SpinConfiguration>& configs,
                                                      Context& ctx = default_context())
{
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    const int wpc = (inst.n() + 63) / 64;
    std::vector<uint64_t> words(configs.size() * wpc);
    for (size_t i = 0; i < configs.size(); ++i) detail::pack(configs[i], &words[i * wpc]);
    std::vector<double> out(configs.size() * inst.k());
    detail::raise(momc_b200_evaluate_cuts(ctx.get(), words.data(), configs.size(), out.data(), err, sizeof err), err);
    std::vector<std::vector<double>> cuts(configs.size());
    for (size_t i = 0; i < configs.size(); ++i)
        cuts[i].assign(out.begin() + static_cast<long>(i * inst.k()), out.begin() + static_cast<long>((i + 1) * inst.k()));
    return cuts;
}

// pareto.hpp:620-642
inline std::vector<double> reference_point_sampled(const MultiObjectiveInstance& inst, int count, std::uint64_t seed,
                                                   Context& ctx = default_context())
{
    if (count < 1) throw std::invalid_argument("sampled reference needs count >= 1");
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    std::vector<double> r(static_cast<size_t>(inst.k()));
    detail::raise(momc_b200_reference_point_sampled(ctx.get(), count, seed, r.data(), err, sizeof err), err);
    return r;
}

// oracle.hpp:25-77. The reference caps n at 22 (enumerate.hpp:17); the device enumeration
// splits the graph at a small vertex separator and needs integer weights instead (n <= 64).
inline ParetoArchive brute_force_pareto(const MultiObjectiveInstance& inst, Context& ctx = default_context())
{
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    int64_t F = 0;
    detail::raise(momc_b200_brute_force_pareto(ctx.get(), &F, nullptr, err, sizeof err), err);
    return fetch_archive(ctx, inst.k(), inst.n());
}

// pareto.hpp:603-617
inline std::vector<double> reference_point_exact(const MultiObjectiveInstance& inst, Context& ctx = default_context())
{
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    std::vector<double> r(static_cast<size_t>(inst.k()));
    detail::raise(momc_b200_reference_point_exact(ctx.get(), r.data(), err, sizeof err), err);
    return r;
}

}  // namespace momc::b200

#endif
