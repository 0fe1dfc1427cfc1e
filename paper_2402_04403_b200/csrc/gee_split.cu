// Two-region pull layout and the tiled gather of the heavy rows.
//
// The label gather of the pull (cls[e] = Y[target e], gee_gather.cu) is bound
// by the L2 request rate of its random 1-byte lookups: on C4 (R-MAT scale 27,
// K = 50) 2.25e9 of the 3.9e9 lookups miss the shared-memory head and each
// costs one 32-byte sector request.  Half of those misses come from the heavy
// rows (> 2048 arcs: 0.3% of the rows, 48% of the arcs).  A heavy row's arcs
// are sorted by label-table slot, so the arcs that fall into one slot range
// ("tile") of the hot tier form a contiguous run -- 43 arcs on average for
// C4 with 245 760-slot tiles.  This file makes those runs the unit of work:
//
//   * graph preparation relocates every heavy row's arcs behind the light
//     rows ([light rows in row order | heavy rows in row order]), so the
//     light gather streams the light region alone and the block reducer
//     reads light-only offsets (heavy rows marked in a bitmap);
//   * per hot tile, the list of (start, length) runs of heavy rows that fall
//     in it (long runs split at SEG_MAX arcs);
//   * per call, one CTA per (tile, split) packs the tile's labels into shared
//     memory (6-bit labels 5 per word for K <= 63, bytes up to K = 255) and
//     streams the tile's runs: coalesced target loads, shared-memory lookups,
//     coalesced class-byte stores -- the L2 sees the targets and classes
//     stream once instead of one sector request per lookup;
//   * each heavy row's cold tail (slots past the hot tier, and the row
//     padding) is looked up through L2 as before.
//
// Reference semantics are unchanged: the class stream is the same bytes the
// plain gather writes (cls[e] = table[targets[e]]), so every reducer sees the
// same input (reference arc rule _kernels.py:192-199).
#include <algorithm>

#include "gee_common.cuh"

namespace {

constexpr int TT = 1024;       // threads per tiled-gather CTA
constexpr int TU = 4;          // lookups in flight per lane per iteration
constexpr int64_t SEG_MAX = 2048;  // longest run one warp takes

__device__ __forceinline__ uint32_t ld_nc_na(const int32_t *p)
{
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Copy each row's arcs to its new position (warp per row).
__global__ void k_relocate_rows(const int64_t *__restrict__ offsets, const int64_t *__restrict__ newpos, int64_t n,
                                const int32_t *__restrict__ t_in, const float *__restrict__ w_in,
                                int32_t *__restrict__ t_out, float *__restrict__ w_out)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t GW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = gw; r < n; r += GW) {
        const int64_t a = offsets[r], len = offsets[r + 1] - a, d = newpos[r];
        for (int64_t j = lane; j < len; j += 32) {
            t_out[d + j] = t_in[a + j];
            if (w_in) w_out[d + j] = w_in[a + j];
        }
    }
}

// First arc index in [lo, hi) whose target slot is >= key (targets sorted
// within the row).
__device__ __forceinline__ int64_t lower_bound_slot(const int32_t *__restrict__ t, int64_t lo, int64_t hi, int64_t key)
{
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)t[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Runs of heavy row h in tile t: [lower_bound(t T), lower_bound(min((t+1) T,
// n_hot))), split into pieces of <= SEG_MAX arcs.  Pass 1 (out_start NULL)
// counts the pieces into cnt[t * n_heavy + h]; pass 2 writes them from
// base[t * n_heavy + h] (exclusive scan of cnt, tile-major).  Tile n_tiles
// holds the row's cold tail [lower_bound(n_hot), row end) as one piece.
__global__ void k_heavy_runs(const int64_t *__restrict__ hoff, int64_t n_heavy, const int32_t *__restrict__ targets,
                             int64_t n_hot, int64_t tile, int32_t n_tiles, int32_t *__restrict__ cnt,
                             const int64_t *__restrict__ base, int64_t *__restrict__ out_start,
                             int32_t *__restrict__ out_len)
{
    const int64_t total = (int64_t)(n_tiles + 1) * n_heavy;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t = (int32_t)(q / n_heavy);
        const int64_t h = q - (int64_t)t * n_heavy;
        const int64_t a = hoff[h], b = hoff[h + 1];
        int64_t lo, hi;
        if (t < n_tiles) {
            const int64_t k0 = (int64_t)t * tile, k1 = min((int64_t)(t + 1) * tile, n_hot);
            lo = k0 < k1 ? lower_bound_slot(targets, a, b, k0) : a;
            hi = k0 < k1 ? lower_bound_slot(targets, lo, b, k1) : a;
        } else {
            lo = lower_bound_slot(targets, a, b, n_hot);
            hi = b;
        }
        const int64_t len = hi - lo;
        const int32_t pieces = t < n_tiles ? (int32_t)((len + SEG_MAX - 1) / SEG_MAX) : (len > 0 ? 1 : 0);
        if (!out_start) {
            cnt[q] = pieces;
            continue;
        }
        int64_t o = base[q];
        for (int32_t p = 0; p < pieces; p++, o++) {
            const int64_t s = lo + (t < n_tiles ? (int64_t)p * SEG_MAX : 0);
            out_start[o] = s;
            out_len[o] = (int32_t)(t < n_tiles ? min(SEG_MAX, hi - s) : len);
        }
    }
}

// Per call: persistent CTAs, one per SM.  CTA c takes the runs
// [piece[c], piece[c+1]) of the tile-major run list (pieces balanced by arc
// count at preparation: the hottest tile alone holds ~40% of the arcs), and
// for every tile its range touches packs that tile's labels into shared
// memory (PER labels per u32 word: 5 x 6 bits for K <= 63, 4 bytes up to
// K = 255), then its warps stream the runs: coalesced target loads that skip
// L1, shared-memory lookups, coalesced class-byte stores.
template <int PER>
__global__ void __launch_bounds__(TT, 1)
k_gather_tiles(const int32_t *__restrict__ targets, const uint8_t *__restrict__ table, int64_t tile, int64_t n_hot,
               int32_t n_tiles, const int64_t *__restrict__ seg_off, const int64_t *__restrict__ seg_start,
               const int32_t *__restrict__ seg_len, const int64_t *__restrict__ piece, uint8_t *__restrict__ cls)
{
    constexpr uint32_t BITS = 32 / PER;
    constexpr uint32_t MASK = (1u << BITS) - 1u;
    extern __shared__ __align__(16) uint32_t tw[];
    int64_t sa = piece[blockIdx.x];
    const int64_t sb = piece[blockIdx.x + 1];
    if (sa >= sb) return;
    // tile of run sa: last t with seg_off[t] <= sa
    int lo = 0, hi = n_tiles - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (seg_off[mid] <= sa) lo = mid;
        else hi = mid - 1;
    }
    const int lane = threadIdx.x & 31;
    const int64_t nw = blockDim.x >> 5, wid = threadIdx.x >> 5;
    for (int t = lo; t < n_tiles && sa < sb; t++) {
        const int64_t te = min(sb, seg_off[t + 1]);
        if (sa >= te) continue;
        const int64_t k0 = (int64_t)t * tile;
        const int64_t span = min(tile, n_hot - k0);
        const int64_t words = (span + PER - 1) / PER;
        __syncthreads();  // the previous tile's lookups are done
        for (int64_t i = threadIdx.x; i < words; i += blockDim.x) {
            uint32_t v = 0;
#pragma unroll
            for (int q = 0; q < PER; q++) {
                const int64_t sl = i * PER + q;
                if (sl < span) v |= (uint32_t)__ldg(table + k0 + sl) << (BITS * q);
            }
            tw[i] = v;
        }
        __syncthreads();
        for (int64_t s = sa + wid; s < te; s += nw) {
            const int64_t p0 = seg_start[s];
            const int32_t len = seg_len[s];
            const int32_t *tp = targets + p0;
            uint8_t *cp = cls + p0;
            for (int32_t j0 = 0; j0 < len; j0 += 32 * TU) {
                uint32_t tv[TU];
#pragma unroll
                for (int u = 0; u < TU; u++) {
                    const int32_t j = j0 + u * 32 + lane;
                    tv[u] = j < len ? ld_nc_na(tp + j) : (uint32_t)k0;
                }
#pragma unroll
                for (int u = 0; u < TU; u++) {
                    const int32_t j = j0 + u * 32 + lane;
                    const uint32_t x = tv[u] - (uint32_t)k0;  // slot within the tile
                    const uint32_t wi = x / PER;
                    const uint32_t lab = (tw[wi] >> (BITS * (x - wi * PER))) & MASK;
                    if (j < len) cp[j] = (uint8_t)lab;
                }
            }
        }
        sa = te;
    }
}

// The heavy rows' cold tails (slots past the hot tier, row padding): one
// warp per tail, labels through L2 (evict_last, like the plain gather).
__global__ void k_gather_tails(const int32_t *__restrict__ targets, const uint8_t *__restrict__ table,
                               const int64_t *__restrict__ seg_start, const int32_t *__restrict__ seg_len, int64_t nseg,
                               uint8_t *__restrict__ cls)
{
    const uint64_t pol = gee::policy_evict_last();
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t GW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = gw; s < nseg; s += GW) {
        const int64_t p0 = seg_start[s];
        const int32_t len = seg_len[s];
        for (int32_t j0 = 0; j0 < len; j0 += 32 * TU) {
            uint32_t tv[TU], lv[TU];
#pragma unroll
            for (int u = 0; u < TU; u++) {
                const int32_t j = j0 + u * 32 + lane;
                tv[u] = j < len ? ld_nc_na(targets + p0 + j) : 0u;
            }
#pragma unroll
            for (int u = 0; u < TU; u++) {
                const int32_t j = j0 + u * 32 + lane;
                lv[u] = j < len ? gee::ld_label<uint8_t>(table + tv[u], pol) : 0u;
            }
#pragma unroll
            for (int u = 0; u < TU; u++) {
                const int32_t j = j0 + u * 32 + lane;
                if (j < len) cls[p0 + j] = (uint8_t)lv[u];
            }
        }
    }
}

int grid_for(int64_t items, int per_block, int waves)
{
    const int64_t want = (items + per_block - 1) / per_block;
    const int64_t cap = (int64_t)gee::sm_count() * waves;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" {

int gee_split_relocate(const int64_t *offsets, const int64_t *newpos, int64_t n, const int32_t *targets,
                       const float *weights, int32_t *out_targets, float *out_weights, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0, GEE_ERR_INVALID, "n must be nonnegative");
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && newpos && targets && out_targets, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(!weights == !out_weights, GEE_ERR_INVALID, "weights and out_weights go together");
    k_relocate_rows<<<grid_for(n * 32, 256, 16), 256, 0, gee::as_stream(stream)>>>(offsets, newpos, n, targets, weights,
                                                                                  out_targets, out_weights);
    return gee::check_launch("k_relocate_rows");
}

int gee_split_runs(const int64_t *hoff, int64_t n_heavy, const int32_t *targets, int64_t n_hot, int64_t tile,
                   int32_t n_tiles, int32_t *cnt, const int64_t *base, int64_t *out_start, int32_t *out_len,
                   void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n_heavy >= 0 && n_tiles >= 0 && tile >= 1, GEE_ERR_INVALID, "bad sizes");
    if (n_heavy == 0) return GEE_OK;
    GEE_REQUIRE(hoff && targets && (out_start ? (base && out_len) : cnt != nullptr), GEE_ERR_INVALID,
                "NULL array argument");
    const int64_t total = (int64_t)(n_tiles + 1) * n_heavy;
    k_heavy_runs<<<grid_for(total, 256, 16), 256, 0, gee::as_stream(stream)>>>(hoff, n_heavy, targets, n_hot, tile,
                                                                              n_tiles, cnt, base, out_start, out_len);
    return gee::check_launch("k_heavy_runs");
}

int64_t gee_tile_slots(int32_t k, int64_t smem_bytes)
{
    const int per = k <= 63 ? 5 : 4;
    return (smem_bytes / 4) * per;
}

int gee_gather_heavy_tiled(const int32_t *targets, const void *table, int64_t n_hot, int32_t k, int64_t tile,
                           int32_t n_tiles, const int64_t *seg_off, const int64_t *seg_start, const int32_t *seg_len,
                           const int64_t *piece, int32_t n_pieces, int64_t tail_first, int64_t n_tails, uint8_t *cls,
                           void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs k <= 255");
    GEE_REQUIRE(n_tiles >= 0 && n_pieces >= 0 && tile >= 1 && tail_first >= 0 && n_tails >= 0, GEE_ERR_INVALID,
                "bad sizes");
    GEE_REQUIRE(targets && table && cls && (n_tiles == 0 || (seg_off && seg_start && seg_len && piece)),
                GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(n_tiles == 0 || ((int64_t)n_tiles * tile >= n_hot && (int64_t)(n_tiles - 1) * tile < n_hot),
                GEE_ERR_INVALID, "tiles must cover the hot tier exactly");
    const int per = k <= 63 ? 5 : 4;
    GEE_REQUIRE(tile % per == 0, GEE_ERR_INVALID, "tile must hold whole words");
    const auto *tab = static_cast<const uint8_t *>(table);
    cudaStream_t st = gee::as_stream(stream);
    if (n_tiles > 0 && n_pieces > 0) {
        const size_t sh = (size_t)(tile / per) * 4;
        static int optin = 0;
        if (!optin) {
            int dev = 0;
            cudaGetDevice(&dev);
            if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
                optin <= 0)
                optin = 48 * 1024;
        }
        GEE_REQUIRE(sh <= (size_t)optin, GEE_ERR_INVALID,
                    "tile of %lld slots needs %zu bytes of shared memory (max %d)", (long long)tile, sh, optin);
        auto kern = per == 5 ? k_gather_tiles<5> : k_gather_tiles<4>;
        GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        kern<<<n_pieces, TT, sh, st>>>(targets, tab, tile, n_hot, n_tiles, seg_off, seg_start, seg_len, piece, cls);
        const int rc = gee::check_launch("k_gather_tiles");
        if (rc) return rc;
    }
    if (n_tails > 0) {
        k_gather_tails<<<grid_for(n_tails * 32, 256, 8), 256, 0, st>>>(targets, tab, seg_start + tail_first,
                                                                       seg_len + tail_first, n_tails, cls);
        return gee::check_launch("k_gather_tails");
    }
    return GEE_OK;
}

}  // extern "C"
