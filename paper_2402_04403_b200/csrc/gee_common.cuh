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

// Shared memory per SM (bytes) available to resident CTAs.
inline int smem_per_sm()
{
    static int b = 0;
    if (!b) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&b, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        if (b <= 0) b = 228 * 1024;
    }
    return b;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T>
__device__ __forceinline__ T ldg_stream(const T *p) { return __ldcs(p); }

// Read-only gather through the non-coherent path (labels, inv tables).
template <typename T>
__device__ __forceinline__ T ldg_ro(const T *p) { return __ldg(p); }

// ---------------------------------------------------------------- labels
// The edge kernels read labels from a "label table": one u8 (k <= 255), u16
// (k <= 65535) or int32 entry per slot, laid out as
//     [ hot tier: n_hot labels in degree-rank order | n labels by vertex id | 0 ]
// (gee_build_projection writes it; gee_hot.cu plans the hot tier).  A CSR
// target stores its slot directly: rank for a hot vertex, n_hot + v for a
// cold one; the trailing zero slot is the sentinel for padding arcs.
template <typename LT>
__device__ __forceinline__ uint32_t ld_label(const LT *p, uint64_t pol);
template <>
__device__ __forceinline__ uint32_t ld_label<uint8_t>(const uint8_t *p, uint64_t pol)
{
    uint16_t v;
    asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ uint32_t ld_label<uint16_t>(const uint16_t *p, uint64_t pol)
{
    uint16_t v;
    asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ uint32_t ld_label<int32_t>(const int32_t *p, uint64_t pol)
{
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

}  // namespace gee

// Checked builds (_build.build_library(checked=True) -> libgee_b200_checked.so,
// compiled with -DGEE_CHECKED): device-side bounds and invariant checks on
// the hot kernels' memory accesses; a violation prints the condition and
// traps the kernel.  compute-sanitizer is not available on the GPU pool, so
// the GPU test suite is also run against this build (profiles/).
#ifdef GEE_CHECKED
#define GEE_DCHECK(cond)                                                                              \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("GEE_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,    \
                   (int)blockIdx.x, (int)threadIdx.x);                                               \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define GEE_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

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
