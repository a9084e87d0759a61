// api.cu -- library-wide error reporting and diagnostics for the C ABI.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"

namespace rtsdf {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return RTSDF_ERR_CUDA;
    }
    return RTSDF_OK;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace rtsdf

extern "C" const char* rtsdf_version(void) { return "rtsdf-b200 0.1.0 (sm_100a)"; }
extern "C" const char* rtsdf_last_error(void) { return rtsdf::g_err; }
extern "C" int64_t rtsdf_launch_count(void) { return rtsdf::g_launches.load(); }
// graph replays run kernels the library counted once, at capture
extern "C" void rtsdf_count_launches(int64_t n) { rtsdf::count_launch((int)n); }
