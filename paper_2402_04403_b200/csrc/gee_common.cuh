// Shared helpers for the GEE sm_100a kernels and their C ABI wrappers.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../include/gee_b200.h"

namespace gee {

void set_error(const char *fmt, ...);
void clear_error();

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Map a pending launch error to GEE_ERR_CUDA with a message naming `what`.
int check_launch(const char *what);

inline int sm_count()
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T>
__device__ __forceinline__ T ldg_stream(const T *p) { return __ldcs(p); }

// Read-only gather through the non-coherent path (labels, inv tables).
template <typename T>
__device__ __forceinline__ T ldg_ro(const T *p) { return __ldg(p); }

}  // namespace gee

#define GEE_REQUIRE(cond, code, ...)      \
    do {                                  \
        if (!(cond)) {                    \
            gee::set_error(__VA_ARGS__);  \
            return (code);                \
        }                                 \
    } while (0)

#define GEE_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            gee::set_error("%s failed: %s", #call, cudaGetErrorString(e_));         \
            return GEE_ERR_CUDA;                                                    \
        }                                                                           \
    } while (0)
