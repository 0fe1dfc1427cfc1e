// Library-wide C ABI pieces: error reporting, version, label width.
#include <cstdarg>
#include <cstring>

#include "gee_common.cuh"

namespace gee {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void clear_error() { g_err[0] = 0; }

int check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
        return GEE_ERR_CUDA;
    }
    return GEE_OK;
}

}  // namespace gee


extern "C" {

int gee_version(void) { return 100; }

const char *gee_last_error(void) { return gee::g_err; }

}  // extern "C"
