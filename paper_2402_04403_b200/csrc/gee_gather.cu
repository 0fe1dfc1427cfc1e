// Label-gather stream: cls[e] = table[targets[e]] for every arc (the random
// half of the pull pass, isolated).  One persistent 1024-thread CTA per SM.
// A warp takes 512 consecutive arcs per step: 16 coalesced target loads that
// bypass L1, then 16 lookup instructions of 32 consecutive arcs each (rows
// are sorted by slot, so neighbouring lanes share sectors), then 16 byte
// stores.  Nothing synchronises, so the lookups' latency is hidden by
// occupancy and per-thread memory-level parallelism.
// Bound: the L1 -> L2 request rate of the lookups that miss on-chip memory
// (one 32-byte sector request per lookup, ~1 per SM clock); shared memory
// serves ~6 random lookups per SM clock, hence the packed head below.
#include <cstdlib>

#include "gee_common.cuh"

namespace {

#ifndef GEE_GTHREADS
#define GEE_GTHREADS 1024
#endif
#ifndef GEE_GU
#define GEE_GU 16
#endif
constexpr int GTHREADS = GEE_GTHREADS;  // threads of the one persistent CTA per SM
constexpr int GU = GEE_GU;              // lookups per lane per step (a warp takes 32 GU arcs)
constexpr int GSTEP = 32 * GU;

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
    const int64_t steps = arcs / GSTEP;
    for (int64_t st = gw; st < steps; st += warps) {
        const int32_t *tp = targets + st * GSTEP + lane;
        uint32_t t[GU];
#pragma unroll
        for (int i = 0; i < GU; i++)
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(t[i]) : "l"(tp + 32 * i));
        uint32_t l[GU];
#pragma unroll
        for (int i = 0; i < GU; i++) l[i] = ld_label_pred<L1MODE>(table + t[i], true, pol);
        uint8_t *cp = cls + st * GSTEP + lane;
#pragma unroll
        for (int i = 0; i < GU; i++) cp[32 * i] = (uint8_t)l[i];
    }
    for (int64_t e = steps * GSTEP + gw * 32 + lane; e < arcs; e += warps * 32) cls[e] = table[targets[e]];
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
                uint8_t *__restrict__ cls, int32_t k)
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
    const int64_t steps = arcs / GSTEP;
    for (int64_t st = gw; st < steps; st += warps) {
        const int32_t *tp = targets + st * GSTEP + lane;
        uint32_t t[GU];
#pragma unroll
        for (int i = 0; i < GU; i++)
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(t[i]) : "l"(tp + 32 * i));
        uint32_t l[GU];
#pragma unroll
        for (int i = 0; i < GU; i++) {
            const uint32_t ti = t[i];
            const bool in_s = ti < hl;
            const uint32_t g = ld_label_pred<1>(table + ti, !in_s, pol);
            const uint32_t wi = in_s ? ti / PER : 0u;
            const uint32_t sv = (head_w[wi] >> (BITS * (ti - wi * PER))) & MASK;
            l[i] = in_s ? sv : g;
            GEE_DCHECK(wi < words && l[i] <= (uint32_t)k);
        }
        uint8_t *cp = cls + st * GSTEP + lane;
#pragma unroll
        for (int i = 0; i < GU; i++) cp[32 * i] = (uint8_t)l[i];
    }
    for (int64_t e = steps * GSTEP + gw * 32 + lane; e < arcs; e += warps * 32) cls[e] = table[targets[e]];
}

}  // namespace

extern "C" int gee_gather_labels_head(const int32_t *targets, int64_t arcs, const void *table, int64_t n_hot,
                                      int32_t k, int64_t head_bytes, uint8_t *cls, void *stream)
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
    // Shared-memory head: the hottest slots of the degree-ranked tier in
    // 96 KB, packed 32/PER bits per label (k <= 63: 5 per word, 122 880
    // slots; k <= 255: bytes, 98 304 slots).  C4: 9.05 ms packed, 9.22 ms
    // with bytes, 9.77 ms without a head (then every lookup goes through L1,
    // evict_last in L2).  Larger heads shrink the L1 that holds the lines of
    // the ~16K lookups in flight per SM (byte head 160 KB: 10.5 ms, 180 KB:
    // 13.3 ms; profiles/r01_gather_tiers*.txt).  Without a hot tier (or
    // head_bytes = 0): plain contiguous lookups.
    int64_t head = head_bytes < 0 ? 98304 : head_bytes;
    if (head > optin - 64) head = optin - 64;
    const int per = k <= 15 ? 8 : k <= 31 ? 6 : k <= 63 ? 5 : 4;
    int64_t hl = (head / 4) * per;
    if (hl > n_hot) hl = n_hot;
    hl -= hl % per;
    const auto *tab = static_cast<const uint8_t *>(table);
    if (hl < 16384) {
        k_gather_contig<0><<<gee::sm_count(), GTHREADS, 0, gee::as_stream(stream)>>>(targets, arcs, tab, cls);
        return gee::check_launch("k_gather_contig");
    }
    const size_t sh = (size_t)(hl / per) * 4;
    auto kern = per == 8 ? k_gather_packed<8> : per == 6 ? k_gather_packed<6> : per == 5 ? k_gather_packed<5>
                                                                                       : k_gather_packed<4>;
    GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    kern<<<gee::sm_count(), GTHREADS, sh, gee::as_stream(stream)>>>(targets, arcs, tab, (uint32_t)hl, cls, k);
    return gee::check_launch("k_gather_packed");
}

extern "C" int gee_gather_labels(const int32_t *targets, int64_t arcs, const void *table, int64_t n_hot, int32_t k,
                                 uint8_t *cls, void *stream)
{
    return gee_gather_labels_head(targets, arcs, table, n_hot, k, -1, cls, stream);
}
