// Label-gather stream: cls[e] = table[targets[e]] for every arc (the random
// half of the pull pass, isolated).  One persistent 1024-thread CTA per SM;
// each thread streams 16 targets (4 x 128-bit), issues 16 independent
// gathers through L1/L2 (evict-last) and writes 16 class bytes (one 128-bit
// store).  Nothing synchronises, so the gathers' latency is hidden by
// occupancy and per-thread memory-level parallelism.
#include <cstdlib>

#include "gee_common.cuh"

namespace {

constexpr int GTHREADS = 1024;
constexpr int GAPT = 16;

template <typename LT>
__global__ void __launch_bounds__(GTHREADS, 1)
k_gather(const int32_t *__restrict__ targets, int64_t arcs, const LT *__restrict__ table, int32_t hot0,
         uint8_t *__restrict__ cls)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LT *hot_s = reinterpret_cast<LT *>(smem_raw);
    {
        const int vec = (int)(((size_t)hot0 * sizeof(LT) + 15) / 16);
        const uint4 *src = reinterpret_cast<const uint4 *>(table);
        uint4 *dst = reinterpret_cast<uint4 *>(hot_s);
        for (int i = threadIdx.x; i < vec; i += GTHREADS) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const uint64_t pol = gee::policy_evict_last();
    const uint32_t h0 = (uint32_t)hot0;
    const int64_t chunks = arcs / GAPT;
    for (int64_t c = (int64_t)blockIdx.x * GTHREADS + threadIdx.x; c < chunks; c += (int64_t)gridDim.x * GTHREADS) {
        int32_t t[GAPT];
#pragma unroll
        for (int v = 0; v < GAPT / 4; v++) {
            const int4 t4 = __ldcs(reinterpret_cast<const int4 *>(targets + c * GAPT) + v);
            t[4 * v] = t4.x; t[4 * v + 1] = t4.y; t[4 * v + 2] = t4.z; t[4 * v + 3] = t4.w;
        }
        uint32_t l[GAPT];
#pragma unroll
        for (int i = 0; i < GAPT; i++) {
            const uint32_t ti = (uint32_t)t[i];
            const bool in_smem = ti < h0;
            l[i] = (uint32_t)hot_s[in_smem ? ti : 0u];
            if (!in_smem) l[i] = gee::ld_label<LT>(table + ti, pol);
        }
        uint4 o;
        o.x = l[0] | l[1] << 8 | l[2] << 16 | l[3] << 24;
        o.y = l[4] | l[5] << 8 | l[6] << 16 | l[7] << 24;
        o.z = l[8] | l[9] << 8 | l[10] << 16 | l[11] << 24;
        o.w = l[12] | l[13] << 8 | l[14] << 16 | l[15] << 24;
        __stcs(reinterpret_cast<uint4 *>(cls) + c, o);
    }
    for (int64_t e = chunks * GAPT + (int64_t)blockIdx.x * GTHREADS + threadIdx.x; e < arcs;
         e += (int64_t)gridDim.x * GTHREADS)
        cls[e] = (uint8_t)table[targets[e]];
}

}  // namespace

extern "C" int gee_gather_labels(const int32_t *targets, int64_t arcs, const void *table, int64_t n_hot, int32_t k,
                                 uint8_t *cls, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs k <= 255");
    if (arcs <= 0) return GEE_OK;
    GEE_REQUIRE(targets && table && cls, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(gee::aligned16(targets) && gee::aligned16(cls) && gee::aligned16(table), GEE_ERR_INVALID,
                "targets/cls/table must be 16-byte aligned");
    static int optin = 0;
    if (!optin) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
            optin = 48 * 1024;
    }
    // Hot labels are read through L1/L2: staging the hot tier's head in
    // shared memory measured 3x slower on C4 (33 ms vs 10.8 ms for 3.6e9
    // lookups: skewed LDS bank conflicts, and the carve-out starves L1).
    // GEE_GATHER_SMEM_HOT=1 re-enables it for experiments.
    int64_t hot0 = 0;
    if (getenv("GEE_GATHER_SMEM_HOT")) {
        hot0 = (optin - 64) & ~15;
        if (hot0 > n_hot) hot0 = n_hot & ~15;
    }
    const size_t sh = (size_t)hot0 + 16;
    auto kern = k_gather<uint8_t>;
    GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    kern<<<gee::sm_count(), GTHREADS, sh, gee::as_stream(stream)>>>(targets, arcs, static_cast<const uint8_t *>(table),
                                                                     (int32_t)hot0, cls);
    return gee::check_launch("k_gather");
}
