// K3: push edge map over a listed edge list (COO, SoA int32/int32/fp32).
//
// Restates serial_pass (reference _kernels.py:210-226): per listed edge
// (u, v, w) both updates, whatever `directed` says (encoder.py:106-120):
//     Z[u, Y[v]-1] += inv[Y[v]] * w     (skipped if Y[v] == 0)
//     Z[v, Y[u]-1] += inv[Y[u]] * w     (skipped if Y[u] == 0)
// With GEE_SOURCE_ONLY only the first update is applied, which is
// arc_pass_worker's rule for symmetric storage (_kernels.py:192-199,
// EdgeAccounting.SOURCE_ONLY, encoder.py:37-55).
//
// The scatter is fp32 red.global.add (REDG.E.ADD.F32.FTZ.RN), the B200
// equivalent of the reference's CAS-loop f64 atomic add (_kernels.py:92-106).
// Edges stream in with 128-bit loads (4 edges per thread-iteration); labels
// are u8/u16 gathers from the label table (gee_common.cuh) kept in L2 with
// an evict_last policy; inv[K+1] lives in shared memory.
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include "gee_common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int PUSH_THREADS = 256;

template <bool PRECOMBINE>
__device__ __forceinline__ void scatter(float *z, int64_t idx, float val, bool active)
{
    if constexpr (PRECOMBINE) {
        // Warp pre-combining: lanes hitting the same Z entry sum their
        // deltas first and one lane issues the red (hub rows).
        cg::coalesced_group act = cg::coalesced_threads();
        unsigned long long key = active ? (unsigned long long)idx : ~0ull;
        auto grp = cg::labeled_partition(act, key);
        float tot = cg::reduce(grp, active ? val : 0.0f, cg::plus<float>());
        if (active && grp.thread_rank() == 0) atomicAdd(z + idx, tot);
    } else {
        if (active) atomicAdd(z + idx, val);
    }
}

template <typename LT, bool WEIGHTED, bool SRC_ONLY, bool VEC, bool PRECOMBINE>
__global__ void __launch_bounds__(PUSH_THREADS)
k_push(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
       const float *__restrict__ w, int64_t s, const LT *__restrict__ labels,
       const float *__restrict__ inv, int32_t k, float *__restrict__ z, bool inv_smem)
{
    const uint64_t pol = gee::policy_evict_last();
    extern __shared__ float sinv[];
    if (inv_smem) {
        for (int c = threadIdx.x; c <= k; c += blockDim.x) sinv[c] = inv[c];
        __syncthreads();
    }
    const float *tab = inv_smem ? sinv : inv;

    auto edge = [&](int32_t u, int32_t v, float wt, bool valid) {
        uint32_t yv = valid ? gee::ld_label<LT>(labels + v, pol) : 0u;
        uint32_t yu = (valid && !SRC_ONLY) ? gee::ld_label<LT>(labels + u, pol) : 0u;
        if (yv > (uint32_t)k) yv = 0;  // raw int32 labels: drop out-of-range
        if (yu > (uint32_t)k) yu = 0;
        float dv = yv ? tab[yv] * wt : 0.f;
        scatter<PRECOMBINE>(z, (int64_t)u * k + ((int64_t)yv - 1), dv, yv != 0);
        if (!SRC_ONLY) {
            float du = yu ? tab[yu] * wt : 0.f;
            scatter<PRECOMBINE>(z, (int64_t)v * k + ((int64_t)yu - 1), du, yu != 0);
        }
    };

    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t done = 0;
    if (VEC) {
        const int64_t s4 = s >> 2;
        const int64_t iters = (s4 + stride - 1) / stride;  // uniform trip count (PRECOMBINE needs converged warps)
        for (int64_t it = 0; it < iters; it++) {
            int64_t q = t0 + it * stride;
            bool ok = q < s4;
            int4 u4 = make_int4(0, 0, 0, 0), v4 = make_int4(0, 0, 0, 0);
            float4 w4 = make_float4(1.f, 1.f, 1.f, 1.f);
            if (ok) {
                u4 = __ldcs(reinterpret_cast<const int4 *>(src) + q);
                v4 = __ldcs(reinterpret_cast<const int4 *>(dst) + q);
                if (WEIGHTED) w4 = __ldcs(reinterpret_cast<const float4 *>(w) + q);
            }
            edge(u4.x, v4.x, w4.x, ok);
            edge(u4.y, v4.y, w4.y, ok);
            edge(u4.z, v4.z, w4.z, ok);
            edge(u4.w, v4.w, w4.w, ok);
        }
        done = s4 << 2;
    }
    const int64_t rest = s - done;
    const int64_t iters = (rest + stride - 1) / stride;
    for (int64_t it = 0; it < iters; it++) {
        int64_t i = done + t0 + it * stride;
        bool ok = i < s;
        int32_t u = ok ? __ldcs(src + i) : 0, v = ok ? __ldcs(dst + i) : 0;
        float wt = (ok && WEIGHTED) ? __ldcs(w + i) : 1.f;
        edge(u, v, wt, ok);
    }
}

template <typename LT, bool WEIGHTED, bool SRC_ONLY, bool VEC, bool PRE>
int launch_push4(const int32_t *src, const int32_t *dst, const float *w, int64_t s, const void *labels,
                 const float *inv, int32_t k, float *z, cudaStream_t st)
{
    bool inv_smem = (size_t)(k + 1) * sizeof(float) <= 48 * 1024;
    size_t sh = inv_smem ? (size_t)(k + 1) * sizeof(float) : 0;
    int64_t per = VEC ? 4 : 1;
    int64_t want = (s + PUSH_THREADS * per - 1) / (PUSH_THREADS * per);
    int64_t cap = (int64_t)gee::sm_count() * 8;  // 8 resident CTAs of 256 per SM
    int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    k_push<LT, WEIGHTED, SRC_ONLY, VEC, PRE><<<grid, PUSH_THREADS, sh, st>>>(
        src, dst, w, s, static_cast<const LT *>(labels), inv, k, z, inv_smem);
    return gee::check_launch("k_push");
}

template <typename LT, bool WEIGHTED, bool SRC_ONLY>
int launch_push3(bool vec, bool pre, const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                 const void *labels, const float *inv, int32_t k, float *z, cudaStream_t st)
{
    if (vec)
        return pre ? launch_push4<LT, WEIGHTED, SRC_ONLY, true, true>(src, dst, w, s, labels, inv, k, z, st)
                   : launch_push4<LT, WEIGHTED, SRC_ONLY, true, false>(src, dst, w, s, labels, inv, k, z, st);
    return pre ? launch_push4<LT, WEIGHTED, SRC_ONLY, false, true>(src, dst, w, s, labels, inv, k, z, st)
               : launch_push4<LT, WEIGHTED, SRC_ONLY, false, false>(src, dst, w, s, labels, inv, k, z, st);
}

template <typename LT>
int launch_push2(bool weighted, bool src_only, bool vec, bool pre, const int32_t *src, const int32_t *dst,
                 const float *w, int64_t s, const void *labels, const float *inv, int32_t k, float *z,
                 cudaStream_t st)
{
    if (weighted)
        return src_only ? launch_push3<LT, true, true>(vec, pre, src, dst, w, s, labels, inv, k, z, st)
                        : launch_push3<LT, true, false>(vec, pre, src, dst, w, s, labels, inv, k, z, st);
    return src_only ? launch_push3<LT, false, true>(vec, pre, src, dst, w, s, labels, inv, k, z, st)
                    : launch_push3<LT, false, false>(vec, pre, src, dst, w, s, labels, inv, k, z, st);
}

}  // namespace

extern "C" int gee_embed_coo(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                             const void *table, int64_t label_off, const float *inv, int64_t n, int32_t k,
                             float *z, uint32_t flags, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && s >= 0 && label_off >= 0, GEE_ERR_INVALID, "n, s and label_off must be nonnegative");
    cudaStream_t st = gee::as_stream(stream);
    if (flags & GEE_ZERO_Z) {
        if (n > 0) GEE_CUDA(cudaMemsetAsync(z, 0, sizeof(float) * (size_t)n * (size_t)k, st));
    }
    if (s == 0 || n == 0) return GEE_OK;
    GEE_REQUIRE(src && dst && table && inv && z, GEE_ERR_INVALID, "NULL array argument");
    const bool vec = gee::aligned16(src) && gee::aligned16(dst) && (!w || gee::aligned16(w));
    const bool src_only = (flags & GEE_SOURCE_ONLY) != 0;
    const bool pre = (flags & GEE_PRECOMBINE) != 0;
    switch (gee_label_bytes(k)) {
    case 1:
        return launch_push2<uint8_t>(w != nullptr, src_only, vec, pre, src, dst, w, s,
                                     static_cast<const uint8_t *>(table) + label_off, inv, k, z, st);
    case 2:
        return launch_push2<uint16_t>(w != nullptr, src_only, vec, pre, src, dst, w, s,
                                      static_cast<const uint16_t *>(table) + label_off, inv, k, z, st);
    default:
        return launch_push2<int32_t>(w != nullptr, src_only, vec, pre, src, dst, w, s,
                                     static_cast<const int32_t *>(table) + label_off, inv, k, z, st);
    }
}
