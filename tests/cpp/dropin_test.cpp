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
    {  // bench (pipeline.hpp:309-393): the README report, field for field
        BenchConfig bc;
        bc.n = 10;
        bc.density = 0.5;
        bc.k = 3;
        bc.instance_seed = 54;
        bc.weights.count = 55;
        bc.solver.batch_size = 500;
        bc.solver.seed = 54;
        bc.checkpoints = 20;
        const auto cpu = bench(bc);
        const auto gpu = b200::bench(bc);
        const RunReport& a = cpu.report;
        const RunReport& b = gpu.report;
        CHECK(same_samples(cpu.pool, gpu.pool));
        CHECK(b.pool_size == 27500 && b.archive_size == 14);
        CHECK(b.hv == 1141902.0 && b.hv_max == 1141902.0 && b.samples_to_optimal == 6054);
        CHECK(a.hv == b.hv && a.hv_max == b.hv_max && a.hv_ratio == b.hv_ratio && a.hv_difference == b.hv_difference);
        CHECK(a.samples_to_optimal == b.samples_to_optimal && a.oracle == b.oracle);
        CHECK(a.reference == b.reference && a.reference_mode == b.reference_mode);
        CHECK(a.n == b.n && a.k == b.k && a.edge_count == b.edge_count && a.weight_count == b.weight_count &&
              a.weight_resolution == b.weight_resolution && a.variant == b.variant && a.runs == b.runs);
        bool same = cpu.archive.size() == gpu.archive.size();
        for (size_t i = 0; same && i < cpu.archive.size(); ++i)
            same = cpu.archive.entries[i].value == gpu.archive.entries[i].value &&
                   cpu.archive.entries[i].config == gpu.archive.entries[i].config;
        CHECK(same);
        CHECK(gpu.trace.size() == 20);
        // the trace replays by timestamp: compare both implementations on the same (GPU) pool
        const auto inst = generate_uniform_instance(10, 0.5, 3, WeightSpec{}, 54);
        const auto t_ref = convergence_trace(gpu.pool, inst, b.reference, 20);
        const auto t_b200 = b200::convergence_trace(gpu.pool, inst, b.reference, 20);
        bool st = t_ref.size() == t_b200.size();
        for (size_t i = 0; st && i < t_ref.size(); ++i)
            st = t_ref[i].hv == t_b200[i].hv && t_ref[i].samples == t_b200[i].samples &&
                 t_ref[i].elapsed_s == t_b200[i].elapsed_s;
        CHECK(st);
        // samples_to_reach (pareto.hpp:763-781): the README's 6,054, and a target never reached
        CHECK(b200::samples_to_reach(gpu.pool, inst, b.reference, b.hv_max) == samples_to_reach(cpu.pool, inst, a.reference, a.hv_max));
        CHECK(!b200::samples_to_reach(gpu.pool, inst, b.reference, 2.0 * b.hv_max).has_value());
        // sampled reference mode, two runs
        bc.ref = "sampled:4096";
        bc.runs = 2;
        bc.checkpoints = 0;
        const auto cpu2 = bench(bc);
        const auto gpu2 = b200::bench(bc);
        CHECK(cpu2.report.hv == gpu2.report.hv && cpu2.report.reference == gpu2.report.reference &&
              cpu2.report.archive_size == gpu2.report.archive_size && !gpu2.report.oracle);
    }
    {  // scalarize / build_block_system (scalarize.hpp:22-71): J(c) and c0 bit-equal
        const auto inst = load_instance(hh);
        const auto lattice = interior_filter(das_dennis(4, 13));
        const std::vector<WeightVector> some(lattice.begin(), lattice.begin() + 7);
        const auto a = build_block_system(inst, some);
        const auto b = b200::build_block_system(inst, some);
        bool same = a.blocks.size() == b.blocks.size() && a.block_dim == b.block_dim;
        for (size_t l = 0; same && l < a.blocks.size(); ++l) {
            same = a.blocks[l].c0 == b.blocks[l].c0;
            for (int i = 0; same && i < inst.n(); ++i)
                for (int j = 0; same && j < inst.n(); ++j) same = a.blocks[l].matrix(i, j) == b.blocks[l].matrix(i, j);
        }
        CHECK(same);
        try {
            b200::build_block_system(inst, {});
            CHECK(false);
        } catch (const std::invalid_argument& e) {
            CHECK(std::string(e.what()) == "block system needs at least one weight vector");
        }
    }
    {  // a device group (two contexts; on a one-GPU box both on device 0, peer-copy merge):
       // the sharded pool, the merged archive and the bench report equal one device's
        const auto inst = load_instance(hh);
        const auto lattice = interior_filter(das_dennis(4, 13));
        SolverConfig cfg;
        cfg.variant = SolverVariant::discrete_sb;
        cfg.batch_size = 333;
        cfg.seed = 11;
        b200::DeviceGroup g2(std::vector<int>{0, 0});
        CHECK(g2.size() == 2 && g2.transport() == MOMC_GROUP_COPY);
        const auto cpu = run_sampler(inst, lattice, cfg, 2);
        const auto one = b200::run_sampler(inst, lattice, cfg, 2);
        const auto two = b200::run_sampler(inst, lattice, cfg, 2, g2);
        CHECK(same_samples(cpu, two) && same_samples(one, two));
        const auto a = non_dominated_filter(cpu, inst);
        const auto b = b200::non_dominated_filter(two, inst, FilterAlgorithm::fast, g2);
        bool same = a.size() == b.size() && a.size() > 0;
        for (size_t i = 0; same && i < a.size(); ++i)
            same = a.entries[i].value == b.entries[i].value && a.entries[i].config == b.entries[i].config;
        CHECK(same);
        BenchConfig bc;
        bc.instance_path = hh;
        bc.weights.resolution = 13;
        bc.solver = cfg;
        bc.runs = 2;
        bc.ref = "sampled:4096";
        const auto r1 = b200::bench(bc);
        const auto r2 = b200::bench(bc, g2);
        CHECK(same_samples(r1.pool, r2.pool));
        CHECK(r1.report.hv == r2.report.hv && r1.report.reference == r2.report.reference &&
              r1.report.archive_size == r2.report.archive_size);
        bool sa = r1.archive.size() == r2.archive.size();
        for (size_t i = 0; sa && i < r1.archive.size(); ++i)
            sa = r1.archive.entries[i].value == r2.archive.entries[i].value &&
                 r1.archive.entries[i].config == r2.archive.entries[i].config;
        CHECK(sa);
        b200::DeviceGroup g3(std::vector<int>{0, 0, 0});
        const auto r3 = b200::bench(bc, g3);
        CHECK(same_samples(r1.pool, r3.pool) && r1.report.hv == r3.report.hv);
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
