// C++ drop-in parity: the reference (CPU, shim build) against momc::b200 (GPU) through the
// same C++ signatures, in the style of proj/tests/test_solver.cpp / test_pareto.cpp.
// Built by tests/cpp/build_dropin.sh (needs /root/reference); run by tests/test_gpu_dropin.py.
#include <cstdio>
#include <cstdlib>

#include "momc/oracle.hpp"
#include "momc/pipeline.hpp"
#include "momc_b200/momc_b200.hpp"

using namespace momc;

static int failures = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        if (!(c)) {                                                          \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);       \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

int main(int argc, char** argv)
{
    const char* hh = argc > 1 ? argv[1] : "data/heavyhex42_k4_seed7.txt";
    {  // README config: same_samples + identical archive + hv
        const auto inst = generate_uniform_instance(10, 0.5, 3, WeightSpec{}, 54);
        const auto lattice = interior_filter(das_dennis(3, 12));
        SolverConfig cfg;
        cfg.batch_size = 500;
        cfg.seed = 54;
        const auto cpu = run_sampler(inst, lattice, cfg, 1);
        const auto gpu = b200::run_sampler(inst, lattice, cfg, 1);
        CHECK(same_samples(cpu, gpu));
        const auto a = non_dominated_filter(cpu, inst);
        const auto b = b200::non_dominated_filter(gpu, inst);
        CHECK(a.size() == 14 && b.size() == 14);
        bool same = a.size() == b.size();
        for (size_t i = 0; same && i < a.size(); ++i)
            same = a.entries[i].value == b.entries[i].value && a.entries[i].config == b.entries[i].config;
        CHECK(same);
        CHECK(b200::hypervolume(b, {0, 0, 0}) == hypervolume(a, {0, 0, 0}));
        CHECK(b200::hypervolume(b, {0, 0, 0}) == 1141902.0);
    }
    {  // heavy-hex K=4, dSB, ragged batch, two runs
        const auto inst = load_instance(hh);
        const auto lattice = interior_filter(das_dennis(4, 13));
        SolverConfig cfg;
        cfg.variant = SolverVariant::discrete_sb;
        cfg.batch_size = 700;
        cfg.seed = 7;
        cfg.threads = 0;
        const auto cpu = run_sampler(inst, lattice, cfg, 2);
        const auto gpu = b200::run_sampler(inst, lattice, cfg, 2);
        CHECK(same_samples(cpu, gpu));
        const auto a = non_dominated_filter(cpu, inst);
        const auto b = b200::non_dominated_filter(gpu, inst);
        bool same = a.size() == b.size();
        for (size_t i = 0; same && i < a.size(); ++i)
            same = a.entries[i].value == b.entries[i].value && a.entries[i].config == b.entries[i].config;
        CHECK(same);
        auto r = reference_point_sampled(inst, 4096, 7);
        CHECK(r == b200::reference_point_sampled(inst, 4096, 7));
        clamp_reference(r, a);
        CHECK(b200::hypervolume(b, r) == hypervolume(a, r));
        std::vector<SpinConfiguration> cfgs;
        for (size_t i = 0; i < 2000; ++i) cfgs.push_back(gpu.config(i));
        CHECK(b200::evaluate_cuts(inst, cfgs) == momc::detail::evaluate_cuts(inst, cfgs));
    }
    {  // exact front by enumeration (oracle.hpp:25-77), reference_point_exact (pareto.hpp:603-617)
        const auto inst = generate_uniform_instance(18, 0.3, 3, WeightSpec::uniform_int(-10, 10), 3);
        const auto a = brute_force_pareto(inst);
        const auto b = b200::brute_force_pareto(inst);
        bool same = a.size() == b.size() && a.size() > 0;
        for (size_t i = 0; same && i < a.size(); ++i)
            same = a.entries[i].value == b.entries[i].value && a.entries[i].config == b.entries[i].config;
        CHECK(same);
        CHECK(reference_point_exact(inst) == b200::reference_point_exact(inst));
    }
    {  // exceptions keep the reference's types and messages
        const auto inst = generate_uniform_instance(4, 1.0, 2, WeightSpec{}, 1);
        SolverConfig cfg;
        try {
            b200::run_sampler(inst, {}, cfg, 1);
            CHECK(false);
        } catch (const std::invalid_argument& e) {
            CHECK(std::string(e.what()) == "run_sampler needs at least one weight vector");
        }
        try {
            ParetoArchive a;
            a.entries.push_back({{1, 2}, {}});
            b200::hypervolume(a, {2, 0});
            CHECK(false);
        } catch (const std::invalid_argument& e) {
            CHECK(std::string(e.what()) == "reference point not dominated by archive entry 0 (objective 0)");
        }
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
