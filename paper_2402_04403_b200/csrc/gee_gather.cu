// Label-gather stream: cls[e] = table[targets[e]] for every arc (the random
// half of the pull pass, isolated).  One persistent 1024-thread CTA per SM;
// each thread streams 16 targets (2 x 256-bit loads that bypass L1), issues
// 16 independent predicated gathers through L1/L2 (L2 evict-last) and writes
// 16 class bytes (one 128-bit store).  Nothing synchronises, so the gathers'
// latency is hidden by occupancy and per-thread memory-level parallelism.
// Bound: L2->SM sector bandwidth (each L1-missing 1-byte lookup moves a
// 32-byte sector; C4 moves ~3.7e9 sectors).
#include <cstdlib>

#include "gee_common.cuh"

namespace {

constexpr int GTHREADS = 1024;
constexpr int GAPT = 16;

// Label load of a cold-or-L2 slot, issued only when `on` (predicated, so
// the 16 lookups of a thread stay independent and in flight together).
// L1MODE 0: default L1 policy; 1: L1::evict_last (keep the hot prefix).
template <int L1MODE>
__device__ __forceinline__ uint32_t ld_label_pred(const uint8_t *p, bool on, uint64_t pol)
{
    uint32_t v = 0;
    if (L1MODE == 1)
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                     "@q ld.global.nc.L1::evict_last.L2::cache_hint.u8 %0, [%1], %3;\n\t}"
                     : "+r"(v) : "l"(p), "r"((uint32_t)on), "l"(pol));
    else
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.u8 %0, [%1], %3;\n\t}"
                     : "+r"(v) : "l"(p), "r"((uint32_t)on), "l"(pol));
    return v;
}

// Target stream: TMODE 0 = ld.global.cs, 4 x 128-bit; 1 = 2 x 256-bit
// ld.global.nc.L1::no_allocate.L2::evict_first (sm_100 .v8.b32 loads).
template <int TMODE>
__device__ __forceinline__ void ld_targets16(const int32_t *p, int32_t (&t)[16])
{
    if (TMODE == 0) {
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const int4 t4 = __ldcs(reinterpret_cast<const int4 *>(p) + v);
            t[4 * v] = t4.x, t[4 * v + 1] = t4.y, t[4 * v + 2] = t4.z, t[4 * v + 3] = t4.w;
        }
    } else {
#pragma unroll
        for (int v = 0; v < 2; v++)
            asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(t[8 * v]), "=r"(t[8 * v + 1]), "=r"(t[8 * v + 2]), "=r"(t[8 * v + 3]),
                           "=r"(t[8 * v + 4]), "=r"(t[8 * v + 5]), "=r"(t[8 * v + 6]), "=r"(t[8 * v + 7])
                         : "l"(p + 8 * v));
    }
}

template <int L1MODE, int TMODE>
__global__ void __launch_bounds__(GTHREADS, 1)
k_gather(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table, int32_t hot0,
         uint8_t *__restrict__ cls)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint8_t *hot_s = smem_raw;  // table[0, hot0): the hottest ranks
    {
        const int vec = (hot0 + 15) / 16;
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
        ld_targets16<TMODE>(targets + c * GAPT, t);
        uint32_t l[GAPT];
#pragma unroll
        for (int i = 0; i < GAPT; i++) {
            const uint32_t ti = (uint32_t)t[i];
            const bool in_smem = ti < h0;
            const uint32_t g = ld_label_pred<L1MODE>(table + ti, !in_smem, pol);
            const uint32_t sv = hot_s[in_smem ? ti : 0u];
            l[i] = in_smem ? sv : g;
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
        cls[e] = table[targets[e]];
}

// Lane-contiguous variant: a warp takes 512 consecutive arcs per step and
// each of its 16 gather instructions covers 32 consecutive arcs, so when
// rows are sorted by slot (gee_sort_rows) a warp's lookups share sectors.
template <int L1MODE>
__global__ void __launch_bounds__(GTHREADS, 1)
k_gather_contig(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table,
                uint8_t *__restrict__ cls)
{
    const uint64_t pol = gee::policy_evict_last();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t steps = arcs / 512;
    for (int64_t st = gw; st < steps; st += warps) {
        const int32_t *tp = targets + st * 512 + lane;
        uint32_t t[16];
#pragma unroll
        for (int i = 0; i < 16; i++)
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(t[i]) : "l"(tp + 32 * i));
        uint32_t l[16];
#pragma unroll
        for (int i = 0; i < 16; i++) l[i] = ld_label_pred<L1MODE>(table + t[i], true, pol);
        uint8_t *cp = cls + st * 512 + lane;
#pragma unroll
        for (int i = 0; i < 16; i++) cp[32 * i] = (uint8_t)l[i];
    }
    for (int64_t e = steps * 512 + gw * 32 + lane; e < arcs; e += warps * 32) cls[e] = table[targets[e]];
}

// Tiered lane-contiguous gather: slots [0, hs) come from a shared-memory copy
// of the table head (immune to the L1 churn of the cold lookups), slots
// [hs, hl1) through L1 with evict_last, and the rest with L1::no_allocate so
// the cold tail does not evict the warm tier.  Lanes of one lookup
// instruction take consecutive arcs as in k_gather_contig.
template <bool SMEM, int SPLIT>
__global__ void __launch_bounds__(GTHREADS, 1)
k_gather_tiered(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table, uint32_t hs,
                uint32_t hl1, uint8_t *__restrict__ cls)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (SMEM) {
        const uint4 *src = reinterpret_cast<const uint4 *>(table);
        uint4 *dst = reinterpret_cast<uint4 *>(smem_raw);
        for (uint32_t i = threadIdx.x; i < hs / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    const uint64_t pol = gee::policy_evict_last();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t steps = arcs / 512;
    for (int64_t st = gw; st < steps; st += warps) {
        const int32_t *tp = targets + st * 512 + lane;
        uint32_t t[16];
#pragma unroll
        for (int i = 0; i < 16; i++)
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(t[i]) : "l"(tp + 32 * i));
        uint32_t l[16];
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const uint32_t ti = t[i];
            const bool in_s = SMEM && ti < hs;
            const bool warm = !in_s && ti < hl1;
            const bool cold = ti >= hl1 && !in_s;
            uint32_t a = 0, b = 0;
            if (SPLIT == 0) {  // one load, default L1 policy
                a = ld_label_pred<0>(table + ti, !in_s, pol);
            } else if (SPLIT == 1) {  // one load, L1 evict_last
                a = ld_label_pred<1>(table + ti, !in_s, pol);
            } else {
            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                         "@q ld.global.nc.L1::evict_last.L2::cache_hint.u8 %0, [%1], %3;\n\t}"
                         : "+r"(a) : "l"(table + ti), "r"((uint32_t)warm), "l"(pol));
            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                         "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %3;\n\t}"
                         : "+r"(b) : "l"(table + ti), "r"((uint32_t)cold), "l"(pol));
            }
            uint32_t sv = 0;
            if (SMEM) sv = smem_raw[in_s ? ti : 0u];
            l[i] = in_s ? sv : (a | b);
        }
        uint8_t *cp = cls + st * 512 + lane;
#pragma unroll
        for (int i = 0; i < 16; i++) cp[32 * i] = (uint8_t)l[i];
    }
    for (int64_t e = steps * 512 + gw * 32 + lane; e < arcs; e += warps * 32) cls[e] = table[targets[e]];
}

// Packed shared-memory head: the first `hl` slots of the table as PER labels
// of 32/PER bits per u32 word (K <= 15: 8, K <= 31: 6, K <= 63: 5, else 4
// per word), so a 96 KB head holds up to 2x the slots of a byte head.  The
// head is built from the u8 table at kernel start; lookups past it take one
// predicated load through L1 (evict_last) and L2 (evict_last).  Shared
// memory serves ~6 random lookups per SM clock, the L1->L2 path ~1.
template <int PER>
__global__ void __launch_bounds__(GTHREADS, 1)
k_gather_packed(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table, uint32_t hl,
                uint8_t *__restrict__ cls)
{
    constexpr uint32_t BITS = 32 / PER;
    constexpr uint32_t MASK = (1u << BITS) - 1u;
    extern __shared__ __align__(16) uint32_t head_w[];
    const uint32_t words = hl / PER;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) {
        uint32_t v = 0;
#pragma unroll
        for (int q = 0; q < PER; q++) v |= (uint32_t)__ldg(table + i * PER + q) << (BITS * q);
        head_w[i] = v;
    }
    __syncthreads();
    const uint64_t pol = gee::policy_evict_last();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t steps = arcs / 512;
    for (int64_t st = gw; st < steps; st += warps) {
        const int32_t *tp = targets + st * 512 + lane;
        uint32_t t[16];
#pragma unroll
        for (int i = 0; i < 16; i++)
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(t[i]) : "l"(tp + 32 * i));
        uint32_t l[16];
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const uint32_t ti = t[i];
            const bool in_s = ti < hl;
            const uint32_t g = ld_label_pred<1>(table + ti, !in_s, pol);
            const uint32_t wi = in_s ? ti / PER : 0u;
            const uint32_t sv = (head_w[wi] >> (BITS * (ti - wi * PER))) & MASK;
            l[i] = in_s ? sv : g;
        }
        uint8_t *cp = cls + st * 512 + lane;
#pragma unroll
        for (int i = 0; i < 16; i++) cp[32 * i] = (uint8_t)l[i];
    }
    for (int64_t e = steps * 512 + gw * 32 + lane; e < arcs; e += warps * 32) cls[e] = table[targets[e]];
}

}  // namespace

extern "C" int gee_gather_labels(const int32_t *targets, int64_t arcs, const void *table, int64_t n_hot, int32_t k,
                                 uint8_t *cls, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs k <= 255");
    if (arcs <= 0) return GEE_OK;
    GEE_REQUIRE(targets && table && cls, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(((uintptr_t)targets & 31) == 0 && gee::aligned16(cls) && gee::aligned16(table), GEE_ERR_INVALID,
                "targets must be 32-byte aligned, cls/table 16-byte aligned");
    static int optin = 0;
    if (!optin) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
            optin = 48 * 1024;
    }
    // Default (mode 10 for k <= 63, else 9): lane-contiguous lookups, which
    // share sectors when rows are sorted by slot, with the hottest slots of
    // the degree-ranked tier in a 96 KB shared-memory head (packed 5 labels
    // per word for k <= 63: 122 880 slots, C4 9.05 ms; bytes: 98 304 slots,
    // 9.22 ms) and the rest through L1 (evict_last) / L2 (evict_last).
    // C4: 9.23 ms against 9.77 ms without the head (mode 4) and 10.43 ms for
    // the 16-arcs-per-thread layout (mode 1); larger heads shrink the L1 that
    // holds the in-flight misses (160 KB: 10.5 ms, 180 KB: 13.3 ms;
    // profiles/r01_gather_tiers*.txt).  Without a hot tier: mode 4.
    // Experiments: GEE_GATHER_MODE (0-3 per-thread layouts, 4/5 contiguous,
    // 6-9 tiered), GEE_GATHER_SMEM_HOT=<bytes>, GEE_GATHER_L1_HOT=<slots>.
    int64_t hot0 = 98304;
    if (const char *e = getenv("GEE_GATHER_SMEM_HOT")) hot0 = atoll(e);
    if (hot0 > optin - 64) hot0 = optin - 64;
    if (hot0 > n_hot) hot0 = n_hot;
    hot0 &= ~(int64_t)15;
    int mode = hot0 >= 16384 ? (k <= 63 ? 10 : 9) : 4;
    if (const char *e = getenv("GEE_GATHER_MODE")) mode = atoi(e);
    if (mode == 10) {  // packed head: hot0 bytes of shared memory, 32/PER bits per label
        const int per = k <= 15 ? 8 : k <= 31 ? 6 : k <= 63 ? 5 : 4;
        int64_t hl = (hot0 / 4) * per;
        if (hl > n_hot) hl = n_hot;
        hl -= hl % per;
        const size_t sh = (size_t)(hl / per) * 4;
        auto kern = per == 8 ? k_gather_packed<8> : per == 6 ? k_gather_packed<6> : per == 5 ? k_gather_packed<5>
                                                                                           : k_gather_packed<4>;
        GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        int bt = GTHREADS;  // GEE_GATHER_BLOCK: fewer lookups in flight (experiment)
        if (const char *e = getenv("GEE_GATHER_BLOCK")) bt = atoi(e);
        kern<<<gee::sm_count(), bt, sh, gee::as_stream(stream)>>>(
            targets, arcs, static_cast<const uint8_t *>(table), (uint32_t)hl, cls);
        return gee::check_launch("k_gather_packed");
    }
    if (mode >= 6 && mode <= 9) {  // tiered: smem head (mode 7) + L1 evict_last warm tier + no-allocate tail
        int64_t hl1 = 1 << 18;
        if (const char *e = getenv("GEE_GATHER_L1_HOT")) hl1 = atoll(e);
        if (hl1 < hot0) hl1 = hot0;
        if (hl1 > 0x7fffffff) hl1 = 0x7fffffff;
        if (mode == 6 || hot0 < 16) mode = 6, hot0 = 0;
        const size_t sh = mode == 6 ? 0 : (size_t)hot0;
        // 6: L1 tiers only; 7: smem head + L1 tiers; 8 / 9: smem head + one load (L1 default / evict_last)
        auto kern = mode == 7   ? k_gather_tiered<true, 2>
                    : mode == 8 ? k_gather_tiered<true, 0>
                    : mode == 9 ? k_gather_tiered<true, 1>
                                : k_gather_tiered<false, 2>;
        GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        kern<<<gee::sm_count(), GTHREADS, sh, gee::as_stream(stream)>>>(
            targets, arcs, static_cast<const uint8_t *>(table), (uint32_t)hot0, (uint32_t)hl1, cls);
        return gee::check_launch("k_gather_tiered");
    }
    if (mode >= 4) {  // lane-contiguous lookups (rows sorted by slot)
        auto kc = mode == 5 ? k_gather_contig<1> : k_gather_contig<0>;
        // GEE_GATHER_BLOCK / GEE_GATHER_CTAS (per SM): co-residency experiments
        int bt = GTHREADS, per = 1;
        if (const char *e = getenv("GEE_GATHER_BLOCK")) bt = atoi(e);
        if (const char *e = getenv("GEE_GATHER_CTAS")) per = atoi(e);
        kc<<<gee::sm_count() * per, bt, 0, gee::as_stream(stream)>>>(targets, arcs,
                                                                     static_cast<const uint8_t *>(table), cls);
        return gee::check_launch("k_gather_contig");
    }
    const size_t sh = (size_t)hot0 + 16;
    auto kern = mode == 1 ? k_gather<0, 1> : mode == 2 ? k_gather<1, 0> : mode == 3 ? k_gather<1, 1> : k_gather<0, 0>;
    GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    kern<<<gee::sm_count(), GTHREADS, sh, gee::as_stream(stream)>>>(targets, arcs, static_cast<const uint8_t *>(table),
                                                                     (int32_t)hot0, cls);
    return gee::check_launch("k_gather");
}
