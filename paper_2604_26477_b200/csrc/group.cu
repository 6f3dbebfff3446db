// Several devices behind one C-ABI handle (momc_group): the reference's task pool over
// (run, weight, 512-trajectory chunk) tasks (run_sampler, solver.hpp:455-522) becomes one
// context per device, each sampling a contiguous share of the flattened blocks; every RNG
// stream is position-independent (solver.hpp:86-94), so the shards concatenate to the
// single-device pool bit for bit. Filtering runs per device to a local front; the fronts
// are gathered on member 0 and merged by the same device filter, which keeps the lex-min
// owner of each value (filter(A u B) = filter(filter(A) u filter(B)), test_pareto.cpp).
//
// Transport of the fronts: NCCL all-gather (communicators from ncclCommInitAll over the
// group's devices, libnccl.so.2 loaded at run time so that a host process that already
// carries torch's NCCL reuses it) when the devices are distinct; otherwise (the same device
// listed twice, e.g. a functional test on a one-GPU box, or MOMC_GROUP_TRANSPORT=copy)
// peer copies into member 0.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.cuh"
#include "pareto.cuh"

using namespace momc_b200;

namespace {

// the few NCCL entry points the merge needs, resolved from libnccl.so.2 at run time
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    bool load(std::string& why)
    {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (lib) break;
        }
        if (!lib) {
            why = "libnccl.so.2 not found";
            return false;
        }
        CommInitAll = reinterpret_cast<decltype(CommInitAll)>(dlsym(lib, "ncclCommInitAll"));
        AllGather = reinterpret_cast<decltype(AllGather)>(dlsym(lib, "ncclAllGather"));
        GroupStart = reinterpret_cast<decltype(GroupStart)>(dlsym(lib, "ncclGroupStart"));
        GroupEnd = reinterpret_cast<decltype(GroupEnd)>(dlsym(lib, "ncclGroupEnd"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(dlsym(lib, "ncclCommDestroy"));
        GetErrorString = reinterpret_cast<decltype(GetErrorString)>(dlsym(lib, "ncclGetErrorString"));
        if (!CommInitAll || !AllGather || !GroupStart || !GroupEnd || !CommDestroy || !GetErrorString) {
            why = "libnccl.so.2 lacks a needed symbol";
            return false;
        }
        return true;
    }
    void check(ncclResult_t r, const char* what) const
    {
        if (r != ncclSuccess) runtime(std::string("NCCL error in ") + what + ": " + GetErrorString(r));
    }
};

// [F x K] doubles then [F x wpc] words, as one byte buffer of `cap` rows per member
__global__ void k_pack_front(const double* __restrict__ v, const uint64_t* __restrict__ w, long long F, int K, int wpc,
                             long long cap, uint64_t* __restrict__ out)
{
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= cap) return;
    for (int q = 0; q < K; ++q) out[i * K + q] = i < F ? __double_as_longlong(v[i * K + q]) : 0ull;
    for (int q = 0; q < wpc; ++q) out[cap * K + i * wpc + q] = i < F ? w[i * wpc + q] : 0ull;
}

}  // namespace

struct momc_group {
    std::vector<momc_ctx*> m;   // one context per listed device
    std::vector<int> devices;
    int transport = 0;          // MOMC_GROUP_{SINGLE, NCCL, COPY}
    NcclApi nccl;
    std::vector<ncclComm_t> comms;
    std::vector<long long> shard_rows;  // first pool row of each member's shard (last sample)
    ~momc_group()
    {
        for (ncclComm_t c : comms)
            if (c && nccl.CommDestroy) nccl.CommDestroy(c);
        for (momc_ctx* c : m) momc_b200_ctx_destroy(c);
    }
};

namespace {

// f(i, ctx) on every member, one host thread per member (each binds its own device); the
// first exception is rethrown on the caller's thread
template <class F>
void each(momc_group& g, F&& f)
{
    if (g.m.size() == 1) {
        bind(*g.m[0]);
        f(0, *g.m[0]);
        return;
    }
    std::vector<std::exception_ptr> errs(g.m.size());
    std::vector<std::thread> th;
    for (size_t i = 0; i < g.m.size(); ++i)
        th.emplace_back([&, i] {
            try {
                bind(*g.m[i]);
                f(static_cast<int>(i), *g.m[i]);
            } catch (...) {
                errs[i] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

std::vector<int> parse_devices(const int* devices, int ndev)
{
    std::vector<int> d;
    if (devices && ndev > 0) return std::vector<int>(devices, devices + ndev);
    const char* env = std::getenv("MOMC_GPUS");
    if (!env || !*env) return {0};
    const std::string s(env);
    if (s.find(',') == std::string::npos) {  // a count: devices 0 .. N-1
        const int n = std::atoi(s.c_str());
        if (n < 1) usage("MOMC_GPUS must be a device count >= 1 or a comma-separated device list");
        for (int i = 0; i < n; ++i) d.push_back(i);
        return d;
    }
    size_t p = 0;
    while (p <= s.size()) {
        const size_t q = s.find(',', p);
        const std::string tok = s.substr(p, q == std::string::npos ? std::string::npos : q - p);
        if (tok.empty()) usage("MOMC_GPUS: empty device entry");
        d.push_back(std::atoi(tok.c_str()));
        if (q == std::string::npos) break;
        p = q + 1;
    }
    return d;
}

// Gathers every member's resident front on member 0 and merges it there into member 0's
// resident archive (ordered like the single-device archive). Returns its size.
long long gather_merge(momc_group& g)
{
    Ctx& root = *g.m[0];
    const size_t N = g.m.size();
    const int K = root.k, wpc = (root.n + 63) / 64;
    std::vector<long long> F(N);
    for (size_t i = 0; i < N; ++i) F[i] = resident_archive(*g.m[i]).F;
    long long total = 0;
    for (long long f : F) total += f;
    bind(root);
    DevBuf<double> av;
    DevBuf<uint64_t> aw;
    av.reserve(static_cast<size_t>(std::max<long long>(total, 1)) * K);
    aw.reserve(static_cast<size_t>(std::max<long long>(total, 1)) * wpc);
    if (g.transport == MOMC_GROUP_NCCL) {
        // one padded all-gather: member i's rows land in every member's receive buffer
        const long long cap = std::max<long long>(*std::max_element(F.begin(), F.end()), 1);
        const size_t chunk = static_cast<size_t>(cap) * (K + wpc);
        std::vector<DevBuf<uint64_t>> send(N), recv(N);
        each(g, [&](int i, Ctx& c) {
            send[i].reserve(chunk);
            recv[i].reserve(chunk * N);
            DevArchive& a = resident_archive(c);
            k_pack_front<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c.stream>>>(a.vals.p, a.words.p, a.F, K, wpc,
                                                                                         cap, send[i].p);
            ck(cudaGetLastError(), "pack front");
            ++c.launches;
        });
        g.nccl.check(g.nccl.GroupStart(), "ncclGroupStart");
        for (size_t i = 0; i < N; ++i) {
            ck(cudaSetDevice(g.m[i]->device), "cudaSetDevice");
            g.nccl.check(g.nccl.AllGather(send[i].p, recv[i].p, chunk * sizeof(uint64_t), ncclUint8, g.comms[i],
                                          g.m[i]->stream),
                         "ncclAllGather");
        }
        g.nccl.check(g.nccl.GroupEnd(), "ncclGroupEnd");
        bind(root);
        long long off = 0;
        for (size_t i = 0; i < N; ++i) {  // member i's chunk of member 0's receive buffer
            const uint64_t* src = recv[0].p + i * chunk;
            if (F[i]) {
                ck(cudaMemcpyAsync(av.p + off * K, src, sizeof(double) * F[i] * K, cudaMemcpyDeviceToDevice, root.stream),
                   "D2D");
                ck(cudaMemcpyAsync(aw.p + off * wpc, src + cap * K, sizeof(uint64_t) * F[i] * wpc,
                                   cudaMemcpyDeviceToDevice, root.stream),
                   "D2D");
            }
            off += F[i];
        }
        for (size_t i = 0; i < N; ++i) ck(cudaStreamSynchronize(g.m[i]->stream), "all-gather");
        for (size_t i = 0; i < N; ++i) {  // free on the owning device
            bind(*g.m[i]);
            send[i].release();
            recv[i].release();
        }
        bind(root);
    } else {
        // peer copies into member 0 (the same device listed twice: plain device-to-device)
        long long off = 0;
        for (size_t i = 0; i < N; ++i) {
            DevArchive& a = resident_archive(*g.m[i]);
            ck(cudaStreamSynchronize(g.m[i]->stream), "front");
            if (F[i]) {
                ck(cudaMemcpyPeerAsync(av.p + off * K, root.device, a.vals.p, g.m[i]->device, sizeof(double) * F[i] * K,
                                       root.stream),
                   "peer copy");
                ck(cudaMemcpyPeerAsync(aw.p + off * wpc, root.device, a.words.p, g.m[i]->device,
                                       sizeof(uint64_t) * F[i] * wpc, root.stream),
                   "peer copy");
            }
            off += F[i];
        }
    }
    root.skip_order = false;
    DevArchive& out = resident_archive(root);
    filter_values_device(root, av.p, aw.p, wpc, root.n, total, K, out, nullptr);
    ck(cudaStreamSynchronize(root.stream), "merge");
    av.release();
    aw.release();
    return out.F;
}

// samples this member's share of the flattened (run, weight, chunk) blocks (compact pool)
void sample_shards(momc_group& g, const momc_solver_cfg* cfg, int runs, std::vector<double>& secs)
{
    Ctx& c0 = *g.m[0];
    const long long total = momc_b200_num_blocks(g.m[0], cfg, runs);
    const size_t N = g.m.size();
    g.shard_rows.assign(N, 0);
    secs.assign(N, 0.0);
    each(g, [&](int i, Ctx& c) {
        const long long base = total / static_cast<long long>(N), rem = total % static_cast<long long>(N);
        const long long b0 = i * base + std::min<long long>(i, rem);
        const long long b1 = b0 + base + (i < rem ? 1 : 0);
        if (b1 > b0) {
            sample(c, cfg, runs, b0, b1, &secs[static_cast<size_t>(i)], true);
        } else {
            c.pool_size = 0;
        }
        g.shard_rows[static_cast<size_t>(i)] = c.pool_row0;
    });
    (void)c0;
}

// the member fronts go through gather_merge (several members, or the forced one-rank NCCL path)
bool merges(const momc_group& g) { return g.m.size() > 1 || g.transport == MOMC_GROUP_NCCL; }

void filter_members(momc_group& g, std::vector<ParetoTimings>& tm)
{
    tm.assign(g.m.size(), ParetoTimings{});
    each(g, [&](int i, Ctx& c) {
        DevArchive& a = resident_archive(c);
        if (c.pool_size <= 0) {
            a.F = 0;
            a.K = c.k;
            a.wpc = (c.n + 63) / 64;
            return;
        }
        const bool so = c.skip_order;
        c.skip_order = merges(g);  // member fronts are merged: no archive order needed
        filter_pool_device(c, c.d_words.p, c.pool_size, a, &tm[static_cast<size_t>(i)]);
        c.skip_order = so;
        ck(cudaStreamSynchronize(c.stream), "front");
    });
}

// each member's compact shard into the host pool (canonical order), stamps per member
void gather_pool(momc_group& g, uint64_t* words, int64_t* stamps)
{
    const int wpc = (g.m[0]->n + 63) / 64;
    each(g, [&](int i, Ctx& c) {
        if (c.pool_size <= 0) return;
        const long long r0 = g.shard_rows[static_cast<size_t>(i)];
        pool_get(c, words ? words + r0 * wpc : nullptr, stamps ? stamps + r0 : nullptr);
    });
}

}  // namespace

extern "C" {

int momc_b200_group_create(const int* devices, int ndev, momc_group** out, char* err, size_t errlen)
{
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto g = std::make_unique<momc_group>();
        g->devices = parse_devices(devices, ndev);
        if (g->devices.empty()) usage("a device group needs at least one device");
        for (int d : g->devices) {
            momc_ctx* c = nullptr;
            char e[1024] = {0};
            const int rc = momc_b200_ctx_create(d, &c, e, sizeof e);
            if (rc != MOMC_OK) throw ApiError(rc, e);
            g->m.push_back(c);
        }
        const std::set<int> distinct(g->devices.begin(), g->devices.end());
        const char* tr = std::getenv("MOMC_GROUP_TRANSPORT");
        const bool want_copy = tr && std::string(tr) == "copy";
        // test hook: "nccl" forces the NCCL transport even for one device (a one-rank
        // all-gather), so the NCCL path runs on a one-GPU box
        const bool force_nccl = tr && std::string(tr) == "nccl";
        if (g->m.size() == 1 && !force_nccl) {
            g->transport = MOMC_GROUP_SINGLE;
        } else if (distinct.size() == g->devices.size() && (force_nccl || !want_copy)) {
            std::string why;
            if (!g->nccl.load(why)) runtime("device group: " + why);
            g->comms.assign(g->m.size(), nullptr);
            g->nccl.check(g->nccl.CommInitAll(g->comms.data(), static_cast<int>(g->m.size()), g->devices.data()),
                          "ncclCommInitAll");
            g->transport = MOMC_GROUP_NCCL;
        } else {
            g->transport = MOMC_GROUP_COPY;
        }
        *out = g.release();
    });
}

void momc_b200_group_destroy(momc_group* g) { delete g; }

int momc_b200_group_size(momc_group* g) { return g ? static_cast<int>(g->m.size()) : 0; }

momc_ctx* momc_b200_group_ctx(momc_group* g, int i)
{
    return g && i >= 0 && i < static_cast<int>(g->m.size()) ? g->m[static_cast<size_t>(i)] : nullptr;
}

int momc_b200_group_transport(momc_group* g) { return g ? g->transport : -1; }

int momc_b200_group_set_instance(momc_group* g, const momc_instance_view* inst, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] { each(*g, [&](int, Ctx& c) { set_instance(c, inst); }); });
}

int momc_b200_group_set_weights(momc_group* g, const int32_t* nums, int L, int H, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] { each(*g, [&](int, Ctx& c) { set_weights(c, nums, L, H); }); });
}

int momc_b200_group_run_sampler(momc_group* g, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                                const momc_solver_cfg* cfg, int runs, uint64_t* out_words, int64_t* out_stamps_ns,
                                double* out_seconds, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        validate_cfg(cfg);
        if (L < 1) usage("run_sampler needs at least one weight vector");
        if (runs < 1) usage("runs must be >= 1");
        const auto t0 = std::chrono::steady_clock::now();
        each(*g, [&](int, Ctx& c) {
            set_instance(c, inst);
            set_weights(c, nums, L, H);
        });
        const auto t1 = std::chrono::steady_clock::now();
        std::vector<double> secs;
        sample_shards(*g, cfg, runs, secs);
        gather_pool(*g, out_words, out_stamps_ns);
        const auto t2 = std::chrono::steady_clock::now();
        if (out_seconds) {
            out_seconds[0] = std::chrono::duration<double>(t1 - t0).count();
            out_seconds[1] = std::chrono::duration<double>(t2 - t1).count();
        }
    });
}

int momc_b200_group_filter_pool(momc_group* g, const uint64_t* words, size_t M, int64_t* out_F, double* filtering_s,
                                char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        if (M == 0) usage("non-dominated filter needs a non-empty pool");
        const auto t0 = std::chrono::steady_clock::now();
        const int wpc = (g->m[0]->n + 63) / 64;
        const size_t N = g->m.size();
        each(*g, [&](int i, Ctx& c) {  // contiguous row shares, filtered where they land
            const size_t r0 = M * static_cast<size_t>(i) / N, r1 = M * static_cast<size_t>(i + 1) / N;
            DevArchive& a = resident_archive(c);
            if (r1 == r0) {
                a.F = 0;
                a.K = c.k;
                a.wpc = wpc;
                return;
            }
            upload_words(c, words + r0 * wpc, r1 - r0);
            const bool so = c.skip_order;
            c.skip_order = merges(*g);
            filter_pool_device(c, c.d_upload.p, static_cast<long long>(r1 - r0), a, nullptr);
            c.skip_order = so;
            ck(cudaStreamSynchronize(c.stream), "front");
        });
        const long long F = merges(*g) ? gather_merge(*g) : resident_archive(*g->m[0]).F;
        if (out_F) *out_F = F;
        if (filtering_s) *filtering_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

int momc_b200_group_bench(momc_group* g, const momc_instance_view* inst, const int32_t* nums, int L, int H,
                          const momc_solver_cfg* cfg, int runs, int ref_count, const double* fixed_ref,
                          uint64_t* out_pool, int64_t* out_stamps_ns, momc_bench_report* rep, char* err, size_t errlen)
{
    return guarded(err, errlen, [&] {
        if (runs < 1) usage("runs must be >= 1");
        validate_cfg(cfg);
        std::memset(rep, 0, sizeof *rep);
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        each(*g, [&](int, Ctx& c) {
            set_instance(c, inst);
            set_weights(c, nums, L, H);
        });
        rep->model_construction_s = std::chrono::duration<double>(clk::now() - t0).count();
        std::vector<double> secs;
        sample_shards(*g, cfg, runs, secs);
        rep->sampling_s = *std::max_element(secs.begin(), secs.end());
        const auto tf = clk::now();
        std::vector<ParetoTimings> tm;
        filter_members(*g, tm);
        Ctx& root = *g->m[0];
        long long pool = 0;
        for (momc_ctx* c : g->m) pool += std::max<long long>(c->pool_size, 0);
        rep->pool_size = pool;
        for (const auto& t : tm) {  // per-member stage times run concurrently: the slowest
            rep->unique_configs += t.unique_configs;
            rep->dedup_s = std::max(rep->dedup_s, t.dedup_s);
            rep->eval_s = std::max(rep->eval_s, t.eval_s);
            rep->collapse_s = std::max(rep->collapse_s, t.collapse_s);
            rep->front_s = std::max(rep->front_s, t.front_s);
            rep->order_s = std::max(rep->order_s, t.order_s);
            rep->front_method = std::max(rep->front_method, t.front_method);
        }
        if (merges(*g)) {
            rep->unique_vectors = 0;  // distinct vectors across shards are not counted after the merge
            gather_merge(*g);
        } else {
            rep->unique_vectors = tm[0].unique_vectors;
        }
        bind(root);
        DevArchive& a = resident_archive(root);
        rep->archive_size = a.F;
        rep->sampler_path = root.last_path;
        const auto tr = clk::now();
        std::vector<double> r(static_cast<size_t>(root.k));
        if (fixed_ref) {
            r.assign(fixed_ref, fixed_ref + root.k);
            rep->hv = hypervolume_device(root, a.vals.p, a.F, a.K, r, true);
        } else {
            rep->hv = hv_sampled_reference_device(root, a.vals.p, a.F, a.K, ref_count, cfg->seed, r, true);
        }
        const auto te = clk::now();
        rep->reference_s = 0;
        rep->hv_s = std::chrono::duration<double>(te - tr).count();
        for (int l = 0; l < root.k && l < 16; ++l) rep->reference[l] = r[static_cast<size_t>(l)];
        rep->pareto_filtering_s = std::chrono::duration<double>(te - tf).count();
        if (out_pool || out_stamps_ns) gather_pool(*g, out_pool, out_stamps_ns);
        rep->end_to_end_s = std::chrono::duration<double>(clk::now() - t0).count();
    });
}

}  // extern "C"
