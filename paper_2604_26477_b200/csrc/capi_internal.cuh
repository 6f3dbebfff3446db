// Host-side building blocks of the C-ABI shared by capi.cu (one context) and group.cu
// (a group of contexts on several devices).
#pragma once
#include <cstring>
#include <utility>

#include "../../include/momc_b200.h"
#include "ctx.cuh"
#include "pareto.cuh"

struct momc_ctx : momc_b200::Ctx {};

namespace momc_b200 {

inline void put_err(char* err, size_t errlen, const char* msg)
{
    if (err && errlen) {
        std::strncpy(err, msg, errlen - 1);
        err[errlen - 1] = 0;
    }
}

// runs f, mapping ApiError to its code (2 usage / 1 runtime) and any other exception to 1,
// with the message in err
template <class F>
int guarded(char* err, size_t errlen, F&& f)
{
    try {
        f();
        return MOMC_OK;
    } catch (const ApiError& e) {
        put_err(err, errlen, e.what());
        return e.code;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return MOMC_ERUNTIME;
    }
}

void validate_cfg(const momc_solver_cfg* c);                      // SolverConfig::validate
void set_instance(Ctx& c, const momc_instance_view* iv);           // MultiObjectiveInstance ctor + CSR
void set_weights(Ctx& c, const int32_t* nums, int L, int H);       // build_block_system on the device
// sample blocks [b_begin, b_end) of a `runs`-run job; compact: the pool holds only their rows
void sample(Ctx& c, const momc_solver_cfg* cfg, int runs, long long b_begin, long long b_end, double* seconds,
            bool compact = false);
void pool_get(Ctx& c, uint64_t* words, int64_t* stamps);            // resident pool -> host
void upload_words(Ctx& c, const uint64_t* words, size_t M);        // host pool -> c.d_upload
std::pair<long long, long long> rows_of_blocks(int batch, int bt, long long b0, long long b1);
DevArchive& resident_archive(Ctx& c);

}  // namespace momc_b200
