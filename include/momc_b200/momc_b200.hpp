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
//   scalarize / build_block_system    scalarize.hpp:22-39, :62-71 (J(c) built on the device, copied
//                                                           back into the reference's Eigen types)
//   brute_force_pareto                oracle.hpp:25-77      (n <= 64 with a small separator)
//   reference_point_exact             pareto.hpp:603-617
//   samples_to_reach                  pareto.hpp:763-781
//   convergence_trace                 pareto.hpp:716-757
//   bench                             pipeline.hpp:309-393  (BenchResult: report, pool, archive, trace)
// Several GPUs: run_sampler / non_dominated_filter / bench also take a DeviceGroup (one
// context per device; MOMC_GPUS selects the devices of default_group()), which replaces the
// reference's task pool (solver.hpp:455-522) and merges the per-device fronts (NCCL).
// The reference's own headers (and so Eigen, or oracle/eigen_shim) must be on the include
// path: the drop-in returns the reference's types.
#ifndef MOMC_B200_HPP
#define MOMC_B200_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <chrono>
#include <cstdlib>
#include <optional>

#include "momc/pareto.hpp"
#include "momc/pipeline.hpp"
#include "momc/scalarize.hpp"
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
        if (h_ && owned_) momc_b200_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    Context(Context&& o) noexcept : h_(o.h_), owned_(o.owned_) { o.h_ = nullptr; }
    momc_ctx* get() const noexcept { return h_; }
    // a non-owning view of a context owned elsewhere (a DeviceGroup member)
    static Context borrow(momc_ctx* h) noexcept { return Context(h, false); }

private:
    Context(momc_ctx* h, bool owned) noexcept : h_(h), owned_(owned) {}
    momc_ctx* h_ = nullptr;
    bool owned_ = true;
};

inline Context& default_context()
{
    static Context ctx(0);
    return ctx;
}

// Several devices, one context each (momc_b200_group_*). Movable, not copyable.
class DeviceGroup {
public:
    // devices empty: MOMC_GPUS ("N" or a list "0,2,5"), else device 0
    explicit DeviceGroup(const std::vector<int>& devices = {})
    {
        char err[1024] = {0};
        detail::raise(momc_b200_group_create(devices.empty() ? nullptr : devices.data(), static_cast<int>(devices.size()),
                                             &h_, err, sizeof err),
                      err);
    }
    ~DeviceGroup()
    {
        if (h_) momc_b200_group_destroy(h_);
    }
    DeviceGroup(const DeviceGroup&) = delete;
    DeviceGroup& operator=(const DeviceGroup&) = delete;
    DeviceGroup(DeviceGroup&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    momc_group* get() const noexcept { return h_; }
    int size() const noexcept { return momc_b200_group_size(h_); }
    int transport() const noexcept { return momc_b200_group_transport(h_); }
    momc_ctx* root() const noexcept { return momc_b200_group_ctx(h_, 0); }

private:
    momc_group* h_ = nullptr;
};

inline DeviceGroup& default_group()
{
    static DeviceGroup g;
    return g;
}

namespace detail {

// canonical (run, weight, trajectory) records + packed configs -> the reference's SamplePool
inline SamplePool make_pool(int n, int L, int batch, size_t M, const std::vector<uint64_t>& words,
                            const std::vector<int64_t>& stamps)
{
    const int wpc = (n + 63) / 64;
    SamplePool pool(n);
    pool.resize(M);
    const size_t per_run = static_cast<size_t>(L) * batch;
    for (size_t i = 0; i < M; ++i) {
        const auto run = static_cast<uint32_t>(i / per_run);
        const auto l = static_cast<uint32_t>((i % per_run) / batch);
        const auto t = static_cast<uint32_t>(i % batch);
        pool.set_record(i, {run, l, t, stamps[i]});
        pool.set_config(i, unpack(&words[i * wpc], n));
    }
    return pool;
}

// MOMC_GPUS listing more than one device routes the context-less calls through default_group()
inline bool env_multi_gpu()
{
    const char* e = std::getenv("MOMC_GPUS");
    if (!e || !*e) return false;
    const std::string s(e);
    return s.find(',') != std::string::npos || std::atoi(s.c_str()) > 1;
}

}  // namespace detail

// solver.hpp:439-529, one device
inline SamplePool run_sampler(const MultiObjectiveInstance& inst, const std::vector<WeightVector>& weights,
                              const SolverConfig& config, int runs, Context& ctx)
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
    SamplePool pool = detail::make_pool(inst.n(), L, config.batch_size, M, words, stamps);
    pool.model_construction_seconds = secs[0];
    pool.sampling_seconds = secs[1];
    return pool;
}

// solver.hpp:439-529 over several devices: the blocks are split across the group's devices
inline SamplePool run_sampler(const MultiObjectiveInstance& inst, const std::vector<WeightVector>& weights,
                              const SolverConfig& config, int runs, DeviceGroup& group)
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
    detail::raise(momc_b200_group_run_sampler(group.get(), &ia.view, nums.data(), L, H, &c, runs, words.data(),
                                              stamps.data(), secs, err, sizeof err),
                  err);
    SamplePool pool = detail::make_pool(inst.n(), L, config.batch_size, M, words, stamps);
    pool.model_construction_seconds = secs[0];
    pool.sampling_seconds = secs[1];
    return pool;
}

inline SamplePool run_sampler(const MultiObjectiveInstance& inst, const std::vector<WeightVector>& weights,
                              const SolverConfig& config, int runs)
{
    if (detail::env_multi_gpu()) return run_sampler(inst, weights, config, runs, default_group());
    return run_sampler(inst, weights, config, runs, default_context());
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
                                          FilterAlgorithm algo, Context& ctx)
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

// pareto.hpp:370-410 over several devices: row shares filtered per device, fronts merged
inline ParetoArchive non_dominated_filter(const SamplePool& pool, const MultiObjectiveInstance& inst,
                                          FilterAlgorithm algo, DeviceGroup& group)
{
    (void)algo;
    if (pool.empty()) throw std::invalid_argument("non-dominated filter needs a non-empty pool");
    if (pool.n() != inst.n()) throw std::invalid_argument("pool does not match instance");
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_group_set_instance(group.get(), &ia.view, err, sizeof err), err);
    int64_t F = 0;
    double fs = 0;
    detail::raise(
        momc_b200_group_filter_pool(group.get(), pool.packed_words().data(), pool.size(), &F, &fs, err, sizeof err),
        err);
    const int64_t n_out = momc_b200_archive_size(group.root());
    const int k = inst.k(), n = inst.n(), wpc = (n + 63) / 64;
    std::vector<double> vals(static_cast<size_t>(n_out) * k);
    std::vector<uint64_t> words(static_cast<size_t>(n_out) * wpc);
    detail::raise(momc_b200_archive_get(group.root(), vals.data(), words.data(), err, sizeof err), err);
    ParetoArchive a;
    for (int64_t i = 0; i < n_out; ++i) {
        ParetoArchive::Entry e;
        e.value.assign(vals.begin() + i * k, vals.begin() + (i + 1) * k);
        e.config = detail::unpack(&words[static_cast<size_t>(i) * wpc], n);
        a.entries.push_back(std::move(e));
    }
    a.filtering_seconds = fs;
    return a;
}

inline ParetoArchive non_dominated_filter(const SamplePool& pool, const MultiObjectiveInstance& inst,
                                          FilterAlgorithm algo = FilterAlgorithm::fast)
{
    if (detail::env_multi_gpu()) return non_dominated_filter(pool, inst, algo, default_group());
    return non_dominated_filter(pool, inst, algo, default_context());
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

// scalarize.hpp:22-39: J(c) and c0 built by the device scalarisation kernel (the same
// rounding order as the reference), copied back into the reference's Eigen types
inline ScalarizedCoupling scalarize(const MultiObjectiveInstance& inst, const WeightVector& c,
                                    Context& ctx = default_context())
{
    if (c.size() != inst.k()) throw std::invalid_argument("weight vector length does not match objective count");
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    auto [nums, H] = detail::weight_arrays({c}, inst.k());
    detail::raise(momc_b200_set_weights(ctx.get(), nums.data(), 1, H, err, sizeof err), err);
    const int n = inst.n();
    std::vector<double> J(static_cast<size_t>(n) * n);
    double c0 = 0;
    detail::raise(momc_b200_get_coupling(ctx.get(), 0, J.data(), &c0, err, sizeof err), err);
    ScalarizedCoupling sc;
    sc.matrix = Eigen::MatrixXd::Zero(n, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) sc.matrix(i, j) = J[static_cast<size_t>(i) * n + j];
    sc.c0 = c0;
    return sc;
}

// scalarize.hpp:62-71
inline BlockSystem build_block_system(const MultiObjectiveInstance& inst, const std::vector<WeightVector>& weights,
                                      Context& ctx = default_context())
{
    if (weights.empty()) throw std::invalid_argument("block system needs at least one weight vector");
    BlockSystem sys;
    sys.block_dim = inst.n();
    sys.blocks.reserve(weights.size());
    for (const auto& w : weights) sys.blocks.push_back(scalarize(inst, w, ctx));
    return sys;
}

// pareto.hpp:763-781: first 1-based sample count (canonical order) whose running archive
// reaches target_hv within 1e-9 relative; nullopt when never
inline std::optional<std::size_t> samples_to_reach(const SamplePool& pool, const MultiObjectiveInstance& inst,
                                                   const std::vector<double>& r, double target_hv,
                                                   Context& ctx = default_context())
{
    if (pool.empty()) throw std::invalid_argument("empty pool");
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    int64_t out = -1;
    detail::raise(momc_b200_samples_to_reach(ctx.get(), pool.packed_words().data(), pool.size(), r.data(), target_hv,
                                             &out, err, sizeof err),
                  err);
    if (out < 0) return std::nullopt;
    return static_cast<std::size_t>(out);
}

// pareto.hpp:716-757: HV of the running archive (replay by timestamp) at `checkpoints`
// evenly spaced milestones
inline std::vector<TracePoint> convergence_trace(const SamplePool& pool, const MultiObjectiveInstance& inst,
                                                 const std::vector<double>& r, int checkpoints,
                                                 Context& ctx = default_context())
{
    if (pool.empty()) throw std::invalid_argument("convergence trace needs a non-empty pool");
    if (checkpoints < 1) throw std::invalid_argument("checkpoints must be >= 1");
    detail::InstanceArrays ia(inst);
    char err[1024] = {0};
    detail::raise(momc_b200_set_instance(ctx.get(), &ia.view, err, sizeof err), err);
    std::vector<int64_t> stamps(pool.size());
    for (size_t i = 0; i < pool.size(); ++i) stamps[i] = pool.record(i).timestamp_ns;
    const auto C = static_cast<size_t>(checkpoints);
    std::vector<double> el(C), hv(C);
    std::vector<int64_t> ns(C);
    detail::raise(momc_b200_convergence_trace(ctx.get(), pool.packed_words().data(), stamps.data(), pool.size(),
                                              r.data(), checkpoints, el.data(), hv.data(), ns.data(), err, sizeof err),
                  err);
    std::vector<TracePoint> trace(C);
    for (size_t i = 0; i < C; ++i) trace[i] = {el[i], hv[i], static_cast<std::size_t>(ns[i])};
    return trace;
}

namespace detail {

// pipeline.hpp:309-393 with the hot path on `root` (one device) or on `group`
inline BenchResult bench_impl(const BenchConfig& cfg, momc_ctx* root, momc_group* group)
{
    if (cfg.runs < 1) throw std::invalid_argument("runs must be >= 1");
    const auto [exact_ref, sample_count] = parse_ref_mode(cfg.ref);
    cfg.solver.validate();
    Context ctx = Context::borrow(root);
    const auto t0 = std::chrono::steady_clock::now();
    BenchResult result;
    RunReport& rep = result.report;
    std::optional<MultiObjectiveInstance> inst_opt;
    if (!cfg.instance_path.empty()) {
        inst_opt.emplace(load_instance(cfg.instance_path));
        rep.instance_source = cfg.instance_path;
    } else if (cfg.target_rho != 0) {
        inst_opt.emplace(generate_correlated_instance(cfg.n, cfg.density, cfg.target_rho, cfg.instance_seed));
        rep.instance_source = "generated";
        rep.density = cfg.density;
        rep.target_rho = cfg.target_rho;
        rep.instance_seed = cfg.instance_seed;
    } else {
        inst_opt.emplace(generate_uniform_instance(cfg.n, cfg.density, cfg.k, WeightSpec{}, cfg.instance_seed));
        rep.instance_source = "generated";
        rep.density = cfg.density;
        rep.instance_seed = cfg.instance_seed;
    }
    const MultiObjectiveInstance& inst = *inst_opt;
    const auto weights = build_weights(inst.k(), cfg.weights);
    const double obtain_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep.n = inst.n();
    rep.k = inst.k();
    rep.edge_count = inst.edges().size();
    rep.variant = variant_name(cfg.solver.variant);
    rep.iterations = cfg.solver.n_iterations;
    rep.dt = cfg.solver.dt;
    rep.alpha = cfg.solver.alpha;
    rep.batch = cfg.solver.batch_size;
    rep.init_scale = cfg.solver.init_scale;
    rep.runs = cfg.runs;
    rep.seed = cfg.solver.seed;
    rep.threads = cfg.solver.threads;
    rep.weight_resolution = select_resolution(inst.k(), cfg.weights);
    rep.weight_count = weights.size();

    std::vector<double> r_fixed;
    if (exact_ref) r_fixed = reference_point_exact(inst, ctx);
    InstanceArrays ia(inst);
    auto [nums, H] = weight_arrays(weights, inst.k());
    const int L = static_cast<int>(weights.size());
    const size_t M = static_cast<size_t>(cfg.runs) * L * cfg.solver.batch_size;
    const int wpc = (inst.n() + 63) / 64;
    std::vector<uint64_t> words(M * wpc);
    std::vector<int64_t> stamps(M);
    const momc_solver_cfg c = cfg_of(cfg.solver);
    momc_bench_report br{};
    char err[1024] = {0};
    if (group) {
        raise(momc_b200_group_bench(group, &ia.view, nums.data(), L, H, &c, cfg.runs, sample_count,
                                    exact_ref ? r_fixed.data() : nullptr, words.data(), stamps.data(), &br, err,
                                    sizeof err),
              err);
    } else {
        raise(momc_b200_bench(root, &ia.view, nums.data(), L, H, &c, cfg.runs, sample_count,
                              exact_ref ? r_fixed.data() : nullptr, words.data(), &br, err, sizeof err),
              err);
        raise(momc_b200_pool_get(root, nullptr, stamps.data(), err, sizeof err), err);
    }
    result.pool = make_pool(inst.n(), L, cfg.solver.batch_size, M, words, stamps);
    result.pool.model_construction_seconds = br.model_construction_s;
    result.pool.sampling_seconds = br.sampling_s;
    rep.model_construction_s = obtain_s + br.model_construction_s;
    rep.sampling_s = br.sampling_s;
    rep.pool_size = result.pool.size();
    result.archive = fetch_archive(ctx, inst.k(), inst.n());
    result.archive.filtering_seconds = br.dedup_s + br.eval_s + br.collapse_s + br.front_s + br.order_s;
    rep.archive_size = result.archive.size();
    const std::vector<double> r(br.reference, br.reference + inst.k());
    result.archive.set_reference(r);
    rep.reference = r;
    rep.reference_mode = exact_ref ? "exact" : "sampled:" + std::to_string(sample_count);
    rep.hv = br.hv;
    rep.pareto_filtering_s = br.pareto_filtering_s;
    if (exact_ref && inst.n() <= kEnumerationCap) {
        const auto exact_front = brute_force_pareto(inst, ctx);
        rep.oracle = true;
        rep.hv_max = hypervolume(exact_front, r, ctx);
        rep.hv_ratio = hv_ratio(rep.hv, rep.hv_max);
        rep.hv_difference = hv_difference(rep.hv_max, rep.hv);
        const auto hit = samples_to_reach(result.pool, inst, r, rep.hv_max, ctx);
        rep.samples_to_optimal = hit ? static_cast<long long>(*hit) : -1;
    }
    if (cfg.checkpoints > 0) result.trace = convergence_trace(result.pool, inst, r, cfg.checkpoints, ctx);
    rep.end_to_end_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return result;
}

}  // namespace detail

// pipeline.hpp:309-393
inline BenchResult bench(const BenchConfig& cfg, Context& ctx) { return detail::bench_impl(cfg, ctx.get(), nullptr); }
inline BenchResult bench(const BenchConfig& cfg, DeviceGroup& group)
{
    return detail::bench_impl(cfg, group.root(), group.get());
}
inline BenchResult bench(const BenchConfig& cfg)
{
    if (detail::env_multi_gpu()) return bench(cfg, default_group());
    return bench(cfg, default_context());
}

}  // namespace momc::b200

#endif
