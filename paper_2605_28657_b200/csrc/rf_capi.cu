// C-ABI plumbing: error reporting, version, device info.
#include <stdarg.h>
#include <stdio.h>

#include "rf_common.cuh"

namespace rf {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return RF_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return RF_ECUDA;
}

int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (!cached) cached = 148;
    }
    return cached;
}

}  // namespace rf

extern "C" int rf_abi_version(void) { return RF_ABI_VERSION; }
extern "C" const char *rf_last_error(void) { return rf::g_err; }
extern "C" int rf_device_sm_count(void) { return rf::sm_count(); }
