// DRAM traffic of the kernels launched between momc_prof_begin() and momc_prof_end(), measured
// in-process with the CUPTI range profiler (auto ranges: one range per kernel launch, kernel
// replay). bench.py uses it in an untimed pass to report roofline.traffic for the dominant kernel
// from the run itself (dram__bytes_read.sum + dram__bytes_write.sum). Measurement tooling only: a
// separate library (libmomc_b200_prof.so, linked against CUPTI) that the product library never
// loads.
#include <cuda.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

const char* kMetrics[] = {"dram__bytes_read.sum", "dram__bytes_write.sum"};
constexpr size_t kNumMetrics = 2;
constexpr size_t kMaxRanges = 256;

struct State {
    bool active = false;
    bool user = false;
    CUpti_Profiler_Host_Object* host = nullptr;
    CUpti_RangeProfiler_Object* rp = nullptr;
    std::vector<uint8_t> config, counter_data;
    std::string err;
};
State g;

bool ok(CUptiResult r, const char* what)
{
    if (r == CUPTI_SUCCESS) return true;
    const char* s = nullptr;
    cuptiGetResultString(r, &s);
    g.err = std::string(what) + ": " + (s ? s : "CUPTI error");
    return false;
}

void cleanup()
{
    if (g.rp) {
        CUpti_RangeProfiler_Disable_Params p{CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
        p.pRangeProfilerObject = g.rp;
        cuptiRangeProfilerDisable(&p);
        g.rp = nullptr;
    }
    if (g.host) {
        CUpti_Profiler_Host_Deinitialize_Params p{CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
        p.pHostObject = g.host;
        cuptiProfilerHostDeinitialize(&p);
        g.host = nullptr;
    }
    g.active = false;
}

}  // namespace

extern "C" {

// Starts profiling the kernels of the current CUDA context of device `device`. user_range = 0:
// one range per kernel launch (auto ranges, kernel replay), everything from here to
// momc_prof_end; user_range = 1: one range around each momc_prof_pass_begin / _pass_end pair,
// the caller replaying its work until momc_prof_pass_end reports every pass submitted.
int momc_prof_begin_mode(int device, int user_range);
int momc_prof_begin(int device) { return momc_prof_begin_mode(device, 0); }

int momc_prof_begin_mode(int device, int user_range)
{
    g.err.clear();
    CUcontext ctx = nullptr;
    if (cuCtxGetCurrent(&ctx) != CUDA_SUCCESS || !ctx) {
        g.err = "no current CUDA context";
        return 1;
    }
    CUpti_Profiler_Initialize_Params ip{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
    if (!ok(cuptiProfilerInitialize(&ip), "cuptiProfilerInitialize")) return 1;
    CUpti_Device_GetChipName_Params cp{CUpti_Device_GetChipName_Params_STRUCT_SIZE};
    cp.deviceIndex = static_cast<size_t>(device);
    if (!ok(cuptiDeviceGetChipName(&cp), "cuptiDeviceGetChipName")) return 1;
    // counter availability of this context
    CUpti_Profiler_GetCounterAvailability_Params ap{CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
    ap.ctx = ctx;
    if (!ok(cuptiProfilerGetCounterAvailability(&ap), "counter availability size")) return 1;
    std::vector<uint8_t> avail(ap.counterAvailabilityImageSize);
    ap.pCounterAvailabilityImage = avail.data();
    if (!ok(cuptiProfilerGetCounterAvailability(&ap), "counter availability")) return 1;
    // host side: the configuration image of the two metrics
    CUpti_Profiler_Host_Initialize_Params hp{CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
    hp.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
    hp.pChipName = cp.pChipName;
    hp.pCounterAvailabilityImage = avail.data();
    if (!ok(cuptiProfilerHostInitialize(&hp), "cuptiProfilerHostInitialize")) return 1;
    g.host = hp.pHostObject;
    CUpti_Profiler_Host_ConfigAddMetrics_Params mp{CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
    mp.pHostObject = g.host;
    mp.ppMetricNames = kMetrics;
    mp.numMetrics = kNumMetrics;
    if (!ok(cuptiProfilerHostConfigAddMetrics(&mp), "config add metrics")) return cleanup(), 1;
    CUpti_Profiler_Host_GetConfigImageSize_Params sp{CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
    sp.pHostObject = g.host;
    if (!ok(cuptiProfilerHostGetConfigImageSize(&sp), "config image size")) return cleanup(), 1;
    g.config.assign(sp.configImageSize, 0);
    CUpti_Profiler_Host_GetConfigImage_Params gp{CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
    gp.pHostObject = g.host;
    gp.configImageSize = g.config.size();
    gp.pConfigImage = g.config.data();
    if (!ok(cuptiProfilerHostGetConfigImage(&gp), "config image")) return cleanup(), 1;
    // target side: range profiler on this context, counter data for up to kMaxRanges kernels
    CUpti_RangeProfiler_Enable_Params ep{CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
    ep.ctx = ctx;
    if (!ok(cuptiRangeProfilerEnable(&ep), "cuptiRangeProfilerEnable")) return cleanup(), 1;
    g.rp = ep.pRangeProfilerObject;
    CUpti_RangeProfiler_GetCounterDataSize_Params dp{CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
    dp.pRangeProfilerObject = g.rp;
    dp.pMetricNames = kMetrics;
    dp.numMetrics = kNumMetrics;
    dp.maxNumOfRanges = user_range ? 1 : kMaxRanges;
    dp.maxNumRangeTreeNodes = user_range ? 1 : kMaxRanges;
    if (!ok(cuptiRangeProfilerGetCounterDataSize(&dp), "counter data size")) return cleanup(), 1;
    g.counter_data.assign(dp.counterDataSize, 0);
    CUpti_RangeProfiler_CounterDataImage_Initialize_Params cip{
        CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
    cip.pRangeProfilerObject = g.rp;
    cip.counterDataSize = g.counter_data.size();
    cip.pCounterData = g.counter_data.data();
    if (!ok(cuptiRangeProfilerCounterDataImageInitialize(&cip), "counter data init")) return cleanup(), 1;
    CUpti_RangeProfiler_SetConfig_Params scp{CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
    scp.pRangeProfilerObject = g.rp;
    scp.configSize = g.config.size();
    scp.pConfig = g.config.data();
    scp.counterDataImageSize = g.counter_data.size();
    scp.pCounterDataImage = g.counter_data.data();
    scp.range = user_range ? CUPTI_UserRange : CUPTI_AutoRange;
    scp.replayMode = user_range ? CUPTI_UserReplay : CUPTI_KernelReplay;
    scp.maxRangesPerPass = user_range ? 1 : kMaxRanges;
    scp.numNestingLevels = 1;
    scp.minNestingLevel = 1;
    scp.passIndex = 0;
    scp.targetNestingLevel = 1;
    if (!ok(cuptiRangeProfilerSetConfig(&scp), "cuptiRangeProfilerSetConfig")) return cleanup(), 1;
    g.user = user_range != 0;
    g.active = true;
    if (!g.user) {
        CUpti_RangeProfiler_Start_Params stp{CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
        stp.pRangeProfilerObject = g.rp;
        if (!ok(cuptiRangeProfilerStart(&stp), "cuptiRangeProfilerStart")) return cleanup(), 1;
    }
    return 0;
}

// user-range mode: one pass of the profiled work
int momc_prof_pass_begin()
{
    CUpti_RangeProfiler_Start_Params stp{CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
    stp.pRangeProfilerObject = g.rp;
    if (!ok(cuptiRangeProfilerStart(&stp), "cuptiRangeProfilerStart")) return cleanup(), 1;
    CUpti_RangeProfiler_PushRange_Params pp{CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
    pp.pRangeProfilerObject = g.rp;
    pp.pRangeName = "work";
    if (!ok(cuptiRangeProfilerPushRange(&pp), "cuptiRangeProfilerPushRange")) return cleanup(), 1;
    return 0;
}

// 1 when every pass has been submitted, 0 when the work must be replayed, -1 on error
int momc_prof_pass_end()
{
    CUpti_RangeProfiler_PopRange_Params pp{CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
    pp.pRangeProfilerObject = g.rp;
    if (!ok(cuptiRangeProfilerPopRange(&pp), "cuptiRangeProfilerPopRange")) return cleanup(), -1;
    CUpti_RangeProfiler_Stop_Params sp{CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
    sp.pRangeProfilerObject = g.rp;
    if (!ok(cuptiRangeProfilerStop(&sp), "cuptiRangeProfilerStop")) return cleanup(), -1;
    return sp.isAllPassSubmitted ? 1 : 0;
}

// Stops, decodes, and returns for the kernel ranges whose name contains `name_substr` the
// summed DRAM bytes (read, write) and the number of matching launches. 0 on success.
int momc_prof_end(const char* name_substr, double* read_bytes, double* write_bytes, int* launches)
{
    if (!g.active) {
        if (g.err.empty()) g.err = "not profiling";
        return 1;
    }
    if (!g.user) {
        CUpti_RangeProfiler_Stop_Params sp{CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
        sp.pRangeProfilerObject = g.rp;
        if (!ok(cuptiRangeProfilerStop(&sp), "cuptiRangeProfilerStop")) return cleanup(), 1;
    }
    CUpti_RangeProfiler_DecodeData_Params dp{CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
    dp.pRangeProfilerObject = g.rp;
    if (!ok(cuptiRangeProfilerDecodeData(&dp), "cuptiRangeProfilerDecodeData")) return cleanup(), 1;
    CUpti_RangeProfiler_GetCounterDataInfo_Params ip{CUpti_RangeProfiler_GetCounterDataInfo_Params_STRUCT_SIZE};
    ip.pCounterDataImage = g.counter_data.data();
    ip.counterDataImageSize = g.counter_data.size();
    if (!ok(cuptiRangeProfilerGetCounterDataInfo(&ip), "counter data info")) return cleanup(), 1;
    double rd = 0, wr = 0;
    int n = 0;
    std::string names;  // reported when nothing matches
    for (size_t r = 0; r < ip.numTotalRanges; ++r) {
        CUpti_RangeProfiler_CounterData_GetRangeInfo_Params rp{
            CUpti_RangeProfiler_CounterData_GetRangeInfo_Params_STRUCT_SIZE};
        rp.pCounterDataImage = g.counter_data.data();
        rp.counterDataImageSize = g.counter_data.size();
        rp.rangeIndex = r;
        rp.rangeDelimiter = "/";
        if (!ok(cuptiRangeProfilerCounterDataGetRangeInfo(&rp), "range info")) return cleanup(), 1;
        if (names.size() < 600) names += std::string(rp.rangeName ? rp.rangeName : "(null)") + "; ";
        if (!g.user && (!rp.rangeName || !std::strstr(rp.rangeName, name_substr))) continue;
        double v[kNumMetrics] = {0, 0};
        CUpti_Profiler_Host_EvaluateToGpuValues_Params ep{CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
        ep.pHostObject = g.host;
        ep.pCounterDataImage = g.counter_data.data();
        ep.counterDataImageSize = g.counter_data.size();
        ep.rangeIndex = r;
        ep.ppMetricNames = kMetrics;
        ep.numMetrics = kNumMetrics;
        ep.pMetricValues = v;
        if (!ok(cuptiProfilerHostEvaluateToGpuValues(&ep), "evaluate")) return cleanup(), 1;
        rd += v[0];
        wr += v[1];
        ++n;
    }
    cleanup();
    if (n == 0) g.err = std::to_string(ip.numTotalRanges) + " ranges: " + names;
    *read_bytes = rd;
    *write_bytes = wr;
    *launches = n;
    return 0;
}

const char* momc_prof_error() { return g.err.c_str(); }

}  // extern "C"
