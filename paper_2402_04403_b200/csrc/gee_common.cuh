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

// ---------------------------------------------------------------- labels
// Compact labels are packed into u32 words: `per` labels of `bits` bits per
// word (bits = smallest width holding k; per = 32 / bits).  K=50 packs five
// 6-bit labels per word, so C4's 134M labels take 107 MB and stay resident
// in the 126 MB L2.  bits == 32 (per == 1) reads raw int32 labels.
struct LabelFmt {
    uint32_t bits, per, mask;
    uint32_t magic, shift;  // t / per == (t * magic) >> shift for 0 <= t < 2^31
};

// magic = ceil(2^(31+l) / per) with 2^l >= per: < 2^32, and the rounding
// error t*(magic*per - 2^(31+l)) / (per 2^(31+l)) < 2^-l <= 1/per keeps the
// floor exact for every 31-bit t.
inline LabelFmt label_fmt(int bits)
{
    LabelFmt f;
    f.bits = (uint32_t)bits;
    f.per = 32u / f.bits;
    f.mask = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
    uint32_t l = 0;
    while ((1u << l) < f.per) l++;
    f.shift = 31 + l;
    f.magic = (uint32_t)(((1ull << f.shift) + f.per - 1) / f.per);
    return f;
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Label gather: read-only path, L2 evict_last so the streamed CSR/Z bytes
// do not push the label words out of L2.
__device__ __forceinline__ uint32_t ld_label_word(const uint32_t *p, uint64_t pol)
{
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ uint32_t gather_label(const uint32_t *__restrict__ words, uint32_t t,
                                                 const LabelFmt &f, uint64_t pol)
{
    const uint32_t wi = (uint32_t)(((uint64_t)t * f.magic) >> f.shift);
    const uint32_t sh = (t - wi * f.per) * f.bits;
    return (ld_label_word(words + wi, pol) >> sh) & f.mask;
}

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
