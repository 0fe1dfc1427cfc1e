// Tile-major heavy region of the pull layout (graph preparation + its label
// gather).
//
// The label lookups of the split pull (gee_gather.cu) are bound by the
// L1 -> L2 request rate, ~1 lookup per SM clock, while lookups in shared
// memory run at the speed the targets stream from HBM (tools/
// tile_gather_bench.cu: 1290 G lookups/s against 270 G/s through L2).  Light
// rows have too few arcs to be regrouped, but the heavy rows (> 2048 arcs:
// half of C4's arcs) can be.  Their TARGETS are moved out of the row-major
// CSR into a region ordered by (slot tile, row, slot), where a tile is a run
// of `tile_slots` label-table slots that fits shared memory; their class
// bytes and weights stay row-major (row, tile, slot), which is what the
// heavy reducer streams.  Every (tile, row) span is padded to a multiple of
// 16 arcs (DeviceGraph.SPAN_ALIGN: 32, whole sectors of class bytes) in
// both orders, and group_dst maps each 16-arc group of the tile-major order
// to its group in the row-major order.  The gather of the region is then a
// pure stream: every CTA takes an equal arc range, stages the range's
// tile(s) in shared memory, looks every label up on chip and stores each
// lane's 4 class bytes at the group's row-major place.  Slots past the last
// tile (cold vertices) form a tail segment looked up through L2 with the
// same scatter.  Arc order inside a row does not matter to the exact
// integer sums, so Z is unchanged bit for bit.
#include <algorithm>

#include "gee_common.cuh"

namespace {

// bounds[b * n_heavy + j] = first arc of heavy row j whose slot is >= thr[b]
// (rows are sorted by slot).
__global__ void k_tile_bounds(const int64_t *__restrict__ offsets, const int32_t *__restrict__ heavy_rows,
                              int64_t n_heavy, const int32_t *__restrict__ targets, const int64_t *__restrict__ thr,
                              int32_t n_thr, int64_t *__restrict__ bounds)
{
    const int64_t total = n_heavy * n_thr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i % n_heavy;
        const int32_t b = (int32_t)(i / n_heavy);
        const int64_t row = heavy_rows[j];
        int64_t lo = offsets[row], hi = offsets[row + 1];
        const int64_t t = thr[b];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)(uint32_t)targets[mid] < t)
                lo = mid + 1;
            else
                hi = mid;
        }
        bounds[i] = lo;
    }
}

// One warp per span: out[dst_first .. + src_len) = in[src_first ..), then
// (sentinel, 0) up to dst_len.
__global__ void k_span_copy(int64_t n_spans, const int64_t *__restrict__ src_first, const int64_t *__restrict__ src_len,
                            const int64_t *__restrict__ dst_first, const int64_t *__restrict__ dst_len,
                            const int32_t *__restrict__ targets, const float *__restrict__ w, int32_t sentinel,
                            int32_t *__restrict__ out_t, float *__restrict__ out_w)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t GW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = gw; s < n_spans; s += GW) {
        const int64_t dl = dst_len[s];
        if (dl == 0) continue;
        const int64_t sf = src_first[s], sl = src_len[s], df = dst_first[s];
        for (int64_t i = lane; i < dl; i += 32) {
            const bool real = i < sl;
            if (targets) out_t[df + i] = real ? targets[sf + i] : sentinel;
            if (w) out_w[df + i] = real ? w[sf + i] : 0.f;
        }
    }
}

#ifndef GEE_TTHREADS
#define GEE_TTHREADS 1024
#endif
constexpr int TTHREADS = GEE_TTHREADS;
#ifndef GEE_TGU
#define GEE_TGU 4
#endif
constexpr int TGU = GEE_TGU;           // 16-byte target loads per lane per step
constexpr int TSTEP = 128 * TGU;       // arcs per warp step

// Tile gather: CTA b takes arcs [c0, c1) of the tile region (an equal share,
// in units of 16 arcs) and, tile by tile, stages the tile's labels in shared
// memory and streams its arcs: 16-byte target loads (L1 bypassed), four
// shared-memory lookups, one 4-byte class store per lane.  Slots outside the
// tile (the span padding's sentinel) give class 0.
__global__ void __launch_bounds__(TTHREADS, 1)
k_gather_tiles(const int32_t *__restrict__ targets, const int64_t *__restrict__ tile_start, int32_t n_tiles,
               int64_t region_start, const int32_t *__restrict__ gdst, const uint8_t *__restrict__ table,
               int64_t table_bytes, uint32_t tile_slots, uint8_t *__restrict__ cls, int32_t k)
{
    extern __shared__ __align__(16) uint8_t tile[];
    const int64_t a0 = tile_start[0], a1 = tile_start[n_tiles];
    const int64_t units = (a1 - a0) >> 4;
    const int64_t c0 = a0 + ((units * blockIdx.x / gridDim.x) << 4);
    const int64_t c1 = a0 + ((units * (blockIdx.x + 1) / gridDim.x) << 4);
    if (c0 >= c1) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // first tile that ends after c0
    int t = 0;
    while (t + 1 < n_tiles && tile_start[t + 1] <= c0) t++;
    for (; t < n_tiles; t++) {
        const int64_t lo = max(c0, tile_start[t]), hi = min(c1, tile_start[t + 1]);
        if (lo >= c1) break;
        if (lo >= hi) continue;
        __syncthreads();
        const int64_t base = (int64_t)t * tile_slots;
        for (uint32_t i = threadIdx.x; i < tile_slots / 16; i += blockDim.x) {
            const int64_t b = base + (int64_t)i * 16;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (b + 16 <= table_bytes) {
                v = *reinterpret_cast<const uint4 *>(table + b);
            } else if (b < table_bytes) {
                uint8_t tmp[16];
                for (int q = 0; q < 16; q++) tmp[q] = b + q < table_bytes ? table[b + q] : (uint8_t)0;
                v = *reinterpret_cast<const uint4 *>(tmp);
            }
            reinterpret_cast<uint4 *>(tile)[i] = v;
        }
        __syncthreads();
        const uint32_t ub = (uint32_t)base;
        for (int64_t a = lo + (int64_t)wid * TSTEP; a < hi; a += (int64_t)(TTHREADS / 32) * TSTEP) {
            uint4 tg[TGU];
            int32_t gd[TGU];
            bool on[TGU];
#pragma unroll
            for (int i = 0; i < TGU; i++) {
                const int64_t g = a + i * 128 + lane * 4;
                on[i] = g < hi;
                tg[i] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                gd[i] = 0;
                if (on[i]) {
                    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(tg[i].x), "=r"(tg[i].y), "=r"(tg[i].z), "=r"(tg[i].w)
                                 : "l"(targets + g));
                    gd[i] = __ldg(gdst + ((g - region_start) >> 4));
                }
            }
#pragma unroll
            for (int i = 0; i < TGU; i++) {
                if (!on[i]) continue;
                const uint32_t x = tg[i].x - ub, y = tg[i].y - ub, zz = tg[i].z - ub, ww = tg[i].w - ub;
                const uint32_t cx = x < tile_slots ? tile[x] : 0u, cy = y < tile_slots ? tile[y] : 0u;
                const uint32_t cz = zz < tile_slots ? tile[zz] : 0u, cw = ww < tile_slots ? tile[ww] : 0u;
                GEE_DCHECK(cx <= (uint32_t)k && cy <= (uint32_t)k && cz <= (uint32_t)k && cw <= (uint32_t)k);
                *reinterpret_cast<uint32_t *>(cls + ((int64_t)gd[i] << 4) + (lane & 3) * 4) =
                    cx | (cy << 8) | (cz << 16) | (cw << 24);
            }
        }
    }
}

// Tail of the heavy region (slots past the last tile): the same stream and
// scatter, with the lookups going to the label table through L1 / L2.
__global__ void __launch_bounds__(TTHREADS, 1)
k_gather_scatter(const int32_t *__restrict__ targets, int64_t first, int64_t end, int64_t region_start,
                 const int32_t *__restrict__ gdst, const uint8_t *__restrict__ table, uint8_t *__restrict__ cls,
                 int32_t k)
{
    const uint64_t pol = gee::policy_evict_last();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    for (int64_t a = first + gw * TSTEP; a < end; a += warps * TSTEP) {
        uint4 tg[TGU];
        int32_t gd[TGU];
        bool on[TGU];
#pragma unroll
        for (int i = 0; i < TGU; i++) {
            const int64_t g = a + i * 128 + lane * 4;
            on[i] = g < end;
            gd[i] = 0;
            if (on[i]) {
                asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(tg[i].x), "=r"(tg[i].y), "=r"(tg[i].z), "=r"(tg[i].w)
                             : "l"(targets + g));
                gd[i] = __ldg(gdst + ((g - region_start) >> 4));
            }
        }
        uint32_t c[TGU][4];
#pragma unroll
        for (int i = 0; i < TGU; i++) {
            if (!on[i]) continue;
            c[i][0] = gee::ld_label<uint8_t>(table + tg[i].x, pol);
            c[i][1] = gee::ld_label<uint8_t>(table + tg[i].y, pol);
            c[i][2] = gee::ld_label<uint8_t>(table + tg[i].z, pol);
            c[i][3] = gee::ld_label<uint8_t>(table + tg[i].w, pol);
        }
#pragma unroll
        for (int i = 0; i < TGU; i++) {
            if (!on[i]) continue;
            GEE_DCHECK(c[i][0] <= (uint32_t)k && c[i][1] <= (uint32_t)k && c[i][2] <= (uint32_t)k &&
                       c[i][3] <= (uint32_t)k);
            *reinterpret_cast<uint32_t *>(cls + ((int64_t)gd[i] << 4) + (lane & 3) * 4) =
                c[i][0] | (c[i][1] << 8) | (c[i][2] << 16) | (c[i][3] << 24);
        }
    }
}

}  // namespace

extern "C" {

int gee_tile_bounds(const int64_t *offsets, const int32_t *heavy_rows, int64_t n_heavy, const int32_t *targets,
                    const int64_t *thresholds, int32_t n_thresholds, int64_t *bounds, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n_heavy >= 0 && n_thresholds >= 1, GEE_ERR_INVALID, "bad sizes");
    if (n_heavy == 0) return GEE_OK;
    GEE_REQUIRE(offsets && heavy_rows && targets && thresholds && bounds, GEE_ERR_INVALID, "NULL array argument");
    const int64_t total = n_heavy * n_thresholds;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)gee::sm_count() * 16);
    k_tile_bounds<<<grid, 256, 0, gee::as_stream(stream)>>>(offsets, heavy_rows, n_heavy, targets, thresholds,
                                                            n_thresholds, bounds);
    return gee::check_launch("k_tile_bounds");
}

int gee_span_copy(int64_t n_spans, const int64_t *src_first, const int64_t *src_len, const int64_t *dst_first,
                  const int64_t *dst_len, const int32_t *targets, const float *w, int32_t sentinel, int32_t *out_targets,
                  float *out_w, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n_spans >= 0, GEE_ERR_INVALID, "n_spans must be nonnegative");
    if (n_spans == 0) return GEE_OK;
    GEE_REQUIRE(src_first && src_len && dst_first && dst_len && (!targets || out_targets) && (!w || out_w) &&
                    (targets || w),
                GEE_ERR_INVALID, "NULL array argument");
    const int grid = (int)std::min<int64_t>((n_spans * 32 + 255) / 256, (int64_t)gee::sm_count() * 16);
    k_span_copy<<<grid, 256, 0, gee::as_stream(stream)>>>(n_spans, src_first, src_len, dst_first, dst_len, targets, w,
                                                          sentinel, out_targets, w ? out_w : nullptr);
    return gee::check_launch("k_span_copy");
}

int gee_gather_tiles(const int32_t *targets, const int64_t *tile_start, int32_t n_tiles, int64_t region_start,
                     const int32_t *group_dst, const void *table, int64_t table_bytes, int64_t tile_slots, int32_t k,
                     uint8_t *cls, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs k <= 255");
    GEE_REQUIRE(n_tiles >= 0, GEE_ERR_INVALID, "n_tiles must be nonnegative");
    if (n_tiles == 0) return GEE_OK;
    GEE_REQUIRE(targets && tile_start && table && cls && group_dst, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(region_start >= 0 && region_start % 16 == 0, GEE_ERR_INVALID, "region_start must be a multiple of 16");
    GEE_REQUIRE(tile_slots >= 16 && tile_slots % 16 == 0 && tile_slots * n_tiles < ((int64_t)1 << 32), GEE_ERR_INVALID,
                "tile_slots must be a multiple of 16 (got %lld)", (long long)tile_slots);
    GEE_REQUIRE(((uintptr_t)targets & 63) == 0 && gee::aligned16(cls) && gee::aligned16(table), GEE_ERR_INVALID,
                "targets must be 64-byte aligned, cls/table 16-byte aligned");
    static int optin = 0;
    if (!optin) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
            optin = 48 * 1024;
    }
    GEE_REQUIRE(tile_slots <= optin, GEE_ERR_INVALID, "tile of %lld slots exceeds the %d bytes of shared memory",
                (long long)tile_slots, optin);
    GEE_CUDA(cudaFuncSetAttribute(k_gather_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_slots));
    k_gather_tiles<<<gee::sm_count(), TTHREADS, (size_t)tile_slots, gee::as_stream(stream)>>>(
        targets, tile_start, n_tiles, region_start, group_dst, static_cast<const uint8_t *>(table), table_bytes,
        (uint32_t)tile_slots, cls, k);
    return gee::check_launch("k_gather_tiles");
}

int gee_gather_scatter(const int32_t *targets, int64_t first, int64_t end, int64_t region_start,
                       const int32_t *group_dst, const void *table, int32_t k, uint8_t *cls, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs k <= 255");
    if (end <= first) return GEE_OK;
    GEE_REQUIRE(targets && table && cls && group_dst, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(region_start >= 0 && region_start % 16 == 0 && first >= region_start && first % 16 == 0 &&
                    end % 16 == 0,
                GEE_ERR_INVALID, "arc ranges must be multiples of 16");
    GEE_REQUIRE(((uintptr_t)targets & 63) == 0 && gee::aligned16(cls), GEE_ERR_INVALID,
                "targets must be 64-byte aligned, cls 16-byte aligned");
    const int64_t steps = (end - first + TSTEP - 1) / TSTEP;
    const int grid = (int)std::min<int64_t>((steps + TTHREADS / 32 - 1) / (TTHREADS / 32), (int64_t)gee::sm_count());
    k_gather_scatter<<<grid, TTHREADS, 0, gee::as_stream(stream)>>>(targets, first, end, region_start, group_dst,
                                                                  static_cast<const uint8_t *>(table), cls, k);
    return gee::check_launch("k_gather_scatter");
}

}  // extern "C"
