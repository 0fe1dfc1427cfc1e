// K4: pull (row-owner) edge map over a symmetric CSR, plus its plan and
// finalize kernels.
//
// For SOURCE_ONLY storage (reference encoder.py:37-55; build_csr's mirror
// arcs, graph.py:159-184) the reference's arc pass adds, for every arc
// x -> v, inv[Y[v]] * w into Z[x, Y[v]-1] (_kernels.py:192-199).  Grouped by
// row that is
//     Z[x, c] = inv[c+1] * sum_{arcs x->v, Y[v] = c+1} w,
// so inv factors out of the row sum and each row of Z is written exactly
// once: no zero wave (zero_worker, _kernels.py:124-135) and no global
// atomics on Z.
//
// Accumulation is exact integer arithmetic, which makes Z bit-stable run to
// run and independent of arc order:
//   unit weights -> u32 counts per (row, class) in shared memory;
//   weighted     -> w rounded to int64 fixed point q = rint(w * 2^e) with e
//                   chosen from the graph (gee_pull_scale_exp) so no row sum
//                   can overflow; the 64-bit sum is kept as two u32 shared
//                   planes with explicit carry (u32 ATOMS.ADD is native on
//                   sm_100a, 64-bit shared atomics are CAS loops).
//
// Work decomposition (balanced by arcs, hub rows split for free):
//   tile j = arcs [j*T, (j+1)*T), T = GEE_TILE_ARCS = 256 threads x 16 arcs;
//   tile j OWNS the rows whose first-arc position offsets[r] lies in it;
//   tile_row[j] = first owned row, chunk_row[c] = row of the first arc of
//   each 16-arc chunk relative to the tile's first row (gee_pull_plan).
//
// Pipeline.  One persistent CTA per SM runs GROUPS independent 256-thread
// groups (named barriers), each walking its own tiles.  While a group
// accumulates tile j it already has tile j+1's labels in flight (cp.async
// 4-byte gathers into shared memory; hot-tier labels copied from the
// shared-memory head) and tile j+2's arcs in flight (128-bit streaming loads
// into registers).  Measured on C4 (profiles/): label gathers dominate, and
// they only approach the L1TEX limit (~1 random gather/clk/SM) when their
// latency is hidden this way.
//
// Only nonempty rows are written here, from a compact window of their
// accumulators; k_zero_empty zero-fills the rows without arcs (55% of C4's
// rows).  Rows that run past their owner tile (hubs) are summed exactly
// through 64-bit global atomics into the owner tile's slot and written by
// k_pull_finalize over the planned list of cut tiles.
#include <cstdio>
#include <cstdlib>

#include "gee_common.cuh"

namespace {

constexpr int GT = 256;                  // threads per group (8 warps)
// independent tile pipelines per CTA: 2 when the kernel gathers labels
// itself (128 registers per thread), 4 in the gather-free class-stream mode
template <bool CLS>
__host__ __device__ constexpr int groups_for() { return CLS ? 2 : 2; }
constexpr int APT = 16;                  // arcs per thread (one chunk)
constexpr int TILE = GT * APT;           // 4096 arcs per tile
static_assert(TILE == GEE_TILE_ARCS, "tile size mismatch with header");
constexpr int SMEM_BYTES_MAX = 227 * 1024;  // opt-in maximum per CTA on sm_100a (queried at launch)
constexpr int WROWS = 2 * GT;            // rows per window (two per thread)
constexpr int OFF_MAX = WROWS + 1;       // staged offsets per buffer
constexpr int WIN_HOT_BYTES = 32 * 1024; // per-group window cap (the rest of smem is L1 or hot tier)
constexpr uint16_t CHUNK_FAR = 0xffff;   // chunk_row overflow: search instead

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t *__restrict__ a, int64_t lo,
                                                   int64_t hi, int64_t key)
{
    // first index in [lo, hi) with a[idx] >= key, or hi
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// tile_row[j] = first row r in [0, n] with offsets[r] >= j*T (j < n_tiles);
// tile_row[n_tiles] = first row with offsets[r] >= arcs (trailing rows have
// no arcs; k_zero_empty zero-fills them with the other empty rows).
__global__ void k_pull_plan(const int64_t *__restrict__ offsets, int64_t n, int64_t arcs,
                            int64_t n_tiles, int64_t *__restrict__ tile_row)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j > n_tiles) return;
    int64_t key = j < n_tiles ? j * (int64_t)TILE : arcs;
    tile_row[j] = lower_bound_i64(offsets, 0, n + 1, key);
}

// First row of tile j including a head row that started in an earlier tile.
__device__ __forceinline__ int64_t tile_base(const int64_t *__restrict__ offsets,
                                             const int64_t *__restrict__ tile_row, int64_t j)
{
    const int64_t r0 = tile_row[j];
    return offsets[r0] > j * (int64_t)TILE ? r0 - 1 : r0;
}

// chunk_row[c] = (row holding arc c*APT) - tile_base, or CHUNK_FAR.
__global__ void k_chunk_rows(const int64_t *__restrict__ offsets, const int64_t *__restrict__ tile_row,
                             int64_t arcs, uint16_t *__restrict__ chunk_row)
{
    const int64_t chunks = (arcs + APT - 1) / APT;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = c * APT, j = e / TILE;
        const int64_t base = tile_base(offsets, tile_row, j);
        // last row r in [base, tile_row[j+1]] with offsets[r] <= e
        const int64_t row = lower_bound_i64(offsets, base, tile_row[j + 1] + 1, e + 1) - 1;
        const int64_t rel = row - base;
        chunk_row[c] = (rel >= 0 && rel < CHUNK_FAR) ? (uint16_t)rel : CHUNK_FAR;
    }
}

// Tiles whose last owned row continues into later tiles (finalize list).
__global__ void k_cut_tiles(const int64_t *__restrict__ offsets, const int64_t *__restrict__ tile_row,
                            int64_t arcs, int64_t n_tiles, int32_t *__restrict__ cut,
                            unsigned long long *__restrict__ count)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_tiles;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r0 = tile_row[j], r1 = tile_row[j + 1];
        const int64_t a1 = min((j + 1) * (int64_t)TILE, arcs);
        if (r1 > r0 && offsets[r1] > a1) cut[atomicAdd(count, 1ull)] = (int32_t)j;
    }
}

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, uint64_t pol)
{
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem)
{
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void group_sync(int g) { asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(GT)); }

struct GroupSmem {  // per-group shared state (carved from dynamic smem)
    int64_t *off64;   // 2 x OFF_MAX staged offsets (cp.async double buffer)
    uint32_t *lab;    // 2 x TILE label words (cp.async double buffer)
    int32_t *ol;      // OFF_MAX + 3 tile-local clamped offsets of the window
    uint16_t *nzr;    // WROWS: rank of each nonempty row, 0xffff for empty rows
    uint16_t *rrow;   // WROWS: window row of each rank
    int32_t *wtot;    // 8 warp totals (+ 8 scratch)
    uint32_t *lo;     // wnz * k
    uint32_t *hi;     // wnz * k (weighted)
};

struct Arcs {  // one tile's arcs for this thread (registers)
    int32_t t[APT];
    float w[APT];
    int32_t r0, r1;  // tile_row[j], tile_row[j+1]
    int32_t crow;    // chunk_row of this thread's chunk
};

template <bool WEIGHTED, bool CLS>
__device__ __forceinline__ void load_arcs(Arcs &A, int64_t j, int gt, const int32_t *__restrict__ targets,
                                          const float *__restrict__ wts, const int64_t *__restrict__ tile_row,
                                          const uint16_t *__restrict__ chunk_row, int64_t arcs, int32_t sentinel)
{
    const int64_t e0 = j * (int64_t)TILE + (int64_t)gt * APT;
    if (CLS) {  // class stream (gee_gather_labels): 16 class bytes per chunk, 0 past the end
        const uint8_t *cls = reinterpret_cast<const uint8_t *>(targets);
        if (e0 + APT <= arcs) {
            const uint4 c4 = __ldcs(reinterpret_cast<const uint4 *>(cls + e0));
            A.t[0] = (int32_t)c4.x; A.t[1] = (int32_t)c4.y; A.t[2] = (int32_t)c4.z; A.t[3] = (int32_t)c4.w;
        } else {
            uint32_t wd[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int i = 0; i < APT; i++)
                if (e0 + i < arcs) wd[i >> 2] |= (uint32_t)cls[e0 + i] << (8 * (i & 3));
            A.t[0] = (int32_t)wd[0]; A.t[1] = (int32_t)wd[1]; A.t[2] = (int32_t)wd[2]; A.t[3] = (int32_t)wd[3];
        }
        if (WEIGHTED) {
            if (e0 + APT <= arcs) {
#pragma unroll
                for (int v = 0; v < APT / 4; v++) {
                    const float4 w4 = __ldcs(reinterpret_cast<const float4 *>(wts + e0) + v);
                    A.w[4 * v] = w4.x; A.w[4 * v + 1] = w4.y; A.w[4 * v + 2] = w4.z; A.w[4 * v + 3] = w4.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < APT; i++) A.w[i] = e0 + i < arcs ? __ldcs(wts + e0 + i) : 0.f;
            }
        }
        A.crow = e0 < arcs ? (int32_t)__ldcs(chunk_row + e0 / APT) : 0;
        A.r0 = (int32_t)tile_row[j];
        A.r1 = (int32_t)tile_row[j + 1];
        return;
    }
    if (e0 + APT <= arcs) {
#pragma unroll
        for (int v = 0; v < APT / 4; v++) {
            const int4 t4 = __ldcs(reinterpret_cast<const int4 *>(targets + e0) + v);
            A.t[4 * v] = t4.x; A.t[4 * v + 1] = t4.y; A.t[4 * v + 2] = t4.z; A.t[4 * v + 3] = t4.w;
            if (WEIGHTED) {
                const float4 w4 = __ldcs(reinterpret_cast<const float4 *>(wts + e0) + v);
                A.w[4 * v] = w4.x; A.w[4 * v + 1] = w4.y; A.w[4 * v + 2] = w4.z; A.w[4 * v + 3] = w4.w;
            }
        }
    } else {  // last tile: padding arcs read the sentinel slot (label 0)
#pragma unroll
        for (int i = 0; i < APT; i++) {
            const bool ok = e0 + i < arcs;
            A.t[i] = ok ? __ldcs(targets + e0 + i) : sentinel;
            if (WEIGHTED) A.w[i] = ok ? __ldcs(wts + e0 + i) : 0.f;
        }
    }
    A.crow = e0 < arcs ? (int32_t)__ldcs(chunk_row + e0 / APT) : 0;
    A.r0 = (int32_t)tile_row[j];
    A.r1 = (int32_t)tile_row[j + 1];
}

// Issue this thread's label fetches for a tile: hot-tier head labels are
// copied from shared memory now, everything else lands via cp.async as the
// containing aligned 4-byte word; returns the position of each label in its
// word (2 bits per arc).
template <typename LT>
__device__ __forceinline__ uint32_t fetch_labels(uint32_t *buf, const Arcs &A, const LT *__restrict__ table,
                                                 const LT *__restrict__ hot_s, uint32_t hot0, uint64_t pol)
{
    uint32_t pos = 0;
#pragma unroll
    for (int i = 0; i < APT; i++) {
        const uint32_t t = (uint32_t)A.t[i];
        if (t < hot0) {
            buf[i] = (uint32_t)hot_s[t];
        } else {
            const uintptr_t addr = reinterpret_cast<uintptr_t>(table + t);
            cp_async4(buf + i, reinterpret_cast<const void *>(addr & ~(uintptr_t)3), pol);
            pos |= (uint32_t)((addr & 3) / sizeof(LT)) << (2 * i);
        }
    }
    return pos;
}

template <typename LT>
__device__ __forceinline__ uint32_t extract_label(uint32_t word, uint32_t pos, int i)
{
    const uint32_t p = (pos >> (2 * i)) & 3u;
    if (sizeof(LT) == 1) return (word >> (8 * p)) & 0xffu;
    if (sizeof(LT) == 2) return (word >> (16 * p)) & 0xffffu;
    return word;
}

// Stage offsets[start .. start+cnt) into smem with cp.async (8 B per copy).
__device__ __forceinline__ void stage_offsets(int64_t *buf, const int64_t *__restrict__ offsets, int32_t r0,
                                              int32_t r1, int gt)
{
    const int32_t start = r0 > 0 ? r0 - 1 : 0;
    const int32_t cnt = min(r1 - start + 1, OFF_MAX);
    for (int i = gt; i < cnt; i += GT) cp_async8(buf + i, offsets + start + i);
}

template <bool WEIGHTED, typename LT, bool CLS>
__global__ void __launch_bounds__(groups_for<CLS>() * GT, 1)
k_pull(const int64_t *__restrict__ offsets, const int32_t *__restrict__ targets,
       const float *__restrict__ wts, int64_t arcs, const int64_t *__restrict__ tile_row,
       const uint16_t *__restrict__ chunk_row, int64_t n_tiles, float qscale, double dscale,
       const LT *__restrict__ table, int32_t sentinel, int32_t hot0, const double *__restrict__ inv, int32_t k,
       float *__restrict__ z, unsigned long long *__restrict__ slots, int wnz, int skip)
{
    // skip: experiment mask (GEE_PULL_SKIP; results are wrong when set):
    // 1 no label gathers, 2 no accumulation, 4 no Z write-out, 16 no partials
    constexpr int GROUPS = groups_for<CLS>();
    constexpr int PT = GROUPS * GT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int g = tid / GT, gt = tid % GT;
    const int lane = tid & 31, gw = gt >> 5;  // warp within the group
    const int kk = k;
    // ---- carve shared memory
    unsigned char *p = smem_raw;
    float *sc = reinterpret_cast<float *>(p);
    p += ((size_t)(kk + 4) & ~(size_t)3) * sizeof(float);
    const size_t plane = ((size_t)wnz * kk + 3) & ~(size_t)3;
    GroupSmem G;
    for (int q = 0; q < GROUPS; q++) {
        GroupSmem s;
        s.off64 = reinterpret_cast<int64_t *>(p);
        p += 2 * ((OFF_MAX + 1) & ~1) * sizeof(int64_t);
        s.lab = reinterpret_cast<uint32_t *>(p);
        if (!CLS) p += 2 * TILE * sizeof(uint32_t);
        s.ol = reinterpret_cast<int32_t *>(p);
        p += ((OFF_MAX + 3 + 3) & ~3) * sizeof(int32_t);
        s.nzr = reinterpret_cast<uint16_t *>(p);
        p += WROWS * sizeof(uint16_t);
        s.rrow = reinterpret_cast<uint16_t *>(p);
        p += WROWS * sizeof(uint16_t);
        s.wtot = reinterpret_cast<int32_t *>(p);
        p += 16 * sizeof(int32_t);
        s.lo = reinterpret_cast<uint32_t *>(p);
        p += plane * sizeof(uint32_t);
        s.hi = reinterpret_cast<uint32_t *>(p);
        if (WEIGHTED) p += plane * sizeof(uint32_t);
        if (q == g) G = s;
    }
    LT *hot_s = reinterpret_cast<LT *>(p);

    const uint64_t pol = gee::policy_evict_last();
    // Z[x, c] = sum * sc[c+1]: inv folded with the fixed-point scale, fp32.
    for (int c = tid; c <= kk; c += PT) sc[c] = (float)(inv[c] * dscale);
    {  // stage the head of the label table (hot tier) with 16 B copies
        const int vec = (int)(((size_t)hot0 * sizeof(LT) + 15) / 16);
        const uint4 *src = reinterpret_cast<const uint4 *>(table);
        uint4 *dst = reinterpret_cast<uint4 *>(hot_s);
        for (int i = tid; i < vec; i += PT) dst[i] = __ldg(src + i);
    }
    {  // windows start zeroed; the write-out clears every entry it reads
        uint4 *a4 = reinterpret_cast<uint4 *>(G.lo);
        const int w4 = (int)(plane * (WEIGHTED ? 2 : 1) / 4);
        for (int i = gt; i < w4; i += GT) a4[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();  // the only CTA-wide barrier: groups run independently after this

    const int64_t stride = (int64_t)gridDim.x * GROUPS;
    int64_t j = (int64_t)blockIdx.x * GROUPS + g;
    if (j >= n_tiles) return;
    const uint32_t uhot0 = (uint32_t)hot0;

    // ---- prologue: tile j's labels + offsets in flight, tile j+stride's arcs loading
    Arcs A;  // arcs two tiles ahead of the one being accumulated
    load_arcs<WEIGHTED, CLS>(A, j, gt, targets, wts, tile_row, chunk_row, arcs, sentinel);
    float wcur[APT], wnext[APT];
    uint32_t cw[4] = {0u, 0u, 0u, 0u};  // class words (CLS mode)
    int32_t R0 = A.r0, R1 = A.r1, crow = A.crow;
    uint32_t pos = 0, npos = 0;
    int32_t nR0 = 0, nR1 = 0, ncrow = 0;
    if (CLS) {
#pragma unroll
        for (int v = 0; v < 4; v++) cw[v] = (uint32_t)A.t[v];
    } else if (!(skip & 1)) {
        pos = fetch_labels<LT>(G.lab + gt * APT, A, table, hot_s, uhot0, pol);
    }
#pragma unroll
    for (int i = 0; i < APT; i++) wcur[i] = A.w[i];
    stage_offsets(G.off64, offsets, R0, R1, gt);
    cp_async_commit();
    if (j + stride < n_tiles)
        load_arcs<WEIGHTED, CLS>(A, j + stride, gt, targets, wts, tile_row, chunk_row, arcs, sentinel);
    int buf = 0;

    for (; j < n_tiles; j += stride) {
        const int64_t jn = j + stride;
        // ---- advance the pipeline: tile jn's labels + offsets, tile jn+stride's arcs
        if constexpr (CLS) {
            // class-stream mode keeps one register stage: A holds tile jn
            // (classes, weights) and is rotated into the current stage at the
            // end of this iteration, when tile jn+stride's load is issued
            if (jn < n_tiles) stage_offsets(G.off64 + (buf ^ 1) * ((OFF_MAX + 1) & ~1), offsets, A.r0, A.r1, gt);
            cp_async_commit();
        } else {
            if (jn < n_tiles) {
                if (!(skip & 1))
                    npos = fetch_labels<LT>(G.lab + (buf ^ 1) * TILE + gt * APT, A, table, hot_s, uhot0, pol);
                nR0 = A.r0;
                nR1 = A.r1;
                ncrow = A.crow;
#pragma unroll
                for (int i = 0; i < APT; i++) wnext[i] = A.w[i];
                stage_offsets(G.off64 + (buf ^ 1) * ((OFF_MAX + 1) & ~1), offsets, nR0, nR1, gt);
            }
            cp_async_commit();
            if (jn + stride < n_tiles)
                load_arcs<WEIGHTED, CLS>(A, jn + stride, gt, targets, wts, tile_row, chunk_row, arcs, sentinel);
        }
        cp_async_wait<1>();  // tile j's labels and offsets have landed

        const int64_t a0 = j * (int64_t)TILE;
        const int tlen = (int)min((int64_t)TILE, arcs - a0);
        const int el0 = gt * APT;  // this thread's first arc, tile-local
        const int64_t *off_s = G.off64 + buf * ((OFF_MAX + 1) & ~1);
        const uint32_t *labw = G.lab + buf * TILE + gt * APT;
        const int32_t st0 = R0 > 0 ? R0 - 1 : 0;  // first staged row
        const int32_t scnt = min(R1 - st0 + 1, OFF_MAX);
        group_sync(g);  // staged data visible; this group's previous tile fully written out
        const bool has_head = off_s[GEE_IDX(R0 - st0, OFF_MAX, 1)] > a0;  // also when R0 == n
        const int64_t offR1 = (R1 - st0 < scnt) ? off_s[GEE_IDX(R1 - st0, OFF_MAX, 2)] : __ldcs(offsets + R1);
        const bool tail_cut = (R1 > R0) && (offR1 > a0 + tlen);
        const int32_t base = has_head ? R0 - 1 : R0;

        int32_t wrow0 = base;
        bool first = true;
        while (wrow0 < R1) {
            // ---- window rows [wrow0, wrow0 + nr): tile-local int32 offsets and
            // nonempty flags (2 rows per thread), ranks by warp + group scan
            int nr = min(WROWS, R1 - wrow0);
            int f0 = 0, f1 = 0;
            {
                const int r = 2 * gt;
                int64_t o0 = 0, o1 = 0, o2 = 0;
                if (first && wrow0 - st0 + nr < scnt) {
                    const int sh = wrow0 - st0;
                    if (r <= nr) o0 = off_s[GEE_IDX(sh + r, OFF_MAX, 3)];
                    if (r + 1 <= nr) o1 = off_s[GEE_IDX(sh + r + 1, OFF_MAX, 3)];
                    if (r + 2 <= nr) o2 = off_s[GEE_IDX(sh + r + 2, OFF_MAX, 3)];
                } else {
                    if (!first) group_sync(g);  // previous window fully consumed
                    if (r <= nr) o0 = __ldcs(offsets + wrow0 + r);
                    if (r + 1 <= nr) o1 = __ldcs(offsets + wrow0 + r + 1);
                    if (r + 2 <= nr) o2 = __ldcs(offsets + wrow0 + r + 2);
                }
                auto loc = [&](int64_t o) {
                    const int64_t v = o - a0;
                    return (int32_t)(v < 0 ? 0 : (v > TILE + 1 ? TILE + 1 : v));
                };
                if (r <= nr) G.ol[r] = loc(o0);
                if (r + 1 <= nr) G.ol[r + 1] = loc(o1);
                if (r + 2 == nr) G.ol[nr] = loc(o2);  // nr == WROWS: no thread starts there
                if (r < nr) f0 = o1 > o0;
                if (r + 1 < nr) f1 = o2 > o1;
            }
            int incl = f0 + f1;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            if (lane == 31) G.wtot[gw] = incl;
            group_sync(g);
            int wpre = 0, nnz = 0;
#pragma unroll
            for (int q = 0; q < GT / 32; q++) {
                const int v = G.wtot[q];
                wpre += q < gw ? v : 0;
                nnz += v;
            }
            {
                const int r = 2 * gt;
                const int rk0 = wpre + incl - f0 - f1, rk1 = rk0 + f0;
                if (r < nr) {
                    G.nzr[r] = f0 ? (uint16_t)rk0 : (uint16_t)0xffff;
                    if (f0 && rk0 < wnz) G.rrow[rk0] = (uint16_t)r;
                    if (f0 && rk0 == wnz) G.wtot[8] = r;  // first row past a full window
                }
                if (r + 1 < nr) {
                    G.nzr[r + 1] = f1 ? (uint16_t)rk1 : (uint16_t)0xffff;
                    if (f1 && rk1 < wnz) G.rrow[rk1] = (uint16_t)(r + 1);
                    if (f1 && rk1 == wnz) G.wtot[8] = r + 1;
                }
            }
            group_sync(g);
            if (nnz > wnz) {
                nr = G.wtot[8];  // rows [0, nr) hold exactly wnz nonempty rows
                nnz = wnz;
            }
            // ---- accumulate this thread's arcs of the window
            const int32_t *ow = G.ol;
            const int wa0 = ow[0], wa1 = min(ow[GEE_IDX(nr, OFF_MAX, 15)], tlen);
            const int m0 = max(el0, wa0), m1 = min(el0 + APT, wa1);
            if (m0 < m1) {
                // row of m0: start from the planned chunk row, walk forward
                int r = 0;
                if (crow != CHUNK_FAR) {
                    r = crow - (wrow0 - base);
                    r = r < 0 ? 0 : (r >= nr ? nr - 1 : r);
                }
                if (ow[GEE_IDX(r, OFF_MAX, 16)] > m0) {  // planned row beyond m0: search (rare)
                    int lo = 0, hi = r;
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (ow[mid] <= m0) lo = mid;
                        else hi = mid;
                    }
                    r = lo;
                }
                int next = ow[GEE_IDX(r + 1, nr + 1, 4)];
                while (m0 >= next) next = ow[GEE_IDX(++r + 1, nr + 1, 6)];
                int slot = G.nzr[GEE_IDX(r, nr, 5)];
#pragma unroll
                for (int i = 0; i < APT; i++) {
                    const int e = el0 + i;
                    if (e < m0 || e >= m1) continue;
                    if (e >= next) {
                        do next = ow[GEE_IDX(++r + 1, nr + 1, 6)];
                        while (e >= next);
                        slot = G.nzr[GEE_IDX(r, nr, 7)];
                    }
                    const uint32_t c = CLS ? ((cw[i >> 2] >> (8 * (i & 3))) & 0xffu)
                                           : ((skip & 1) ? 1u + (i & 1) : extract_label<LT>(labw[i], pos, i));
                    if (c == 0u || c > (uint32_t)kk || (skip & 2)) continue;  // unlabeled / out-of-range raw label
                    const int idx = GEE_IDX(slot * kk + (int)c - 1, wnz * kk, 8);
                    if (WEIGHTED) {
                        const unsigned long long q = (unsigned long long)__float2ll_rn(wcur[i] * qscale);
                        const uint32_t lo32 = (uint32_t)q;
                        uint32_t hi32 = (uint32_t)(q >> 32);
                        const uint32_t old = atomicAdd(&G.lo[idx], lo32);
                        hi32 += (old + lo32 < old) ? 1u : 0u;  // carry out of the low plane
                        if (hi32) atomicAdd(&G.hi[idx], hi32);
                    } else {
                        atomicAdd(&G.lo[idx], 1u);
                    }
                }
            }
            group_sync(g);

            // ---- write out the window's complete nonempty rows (empty rows are
            // zeroed by k_zero_empty); flat over nnz x k, clearing what it reads
            {
                const int32_t lr_lo = max(wrow0, R0) - wrow0;                           // a head row is partial
                const int32_t lr_hi = min(wrow0 + nr, tail_cut ? R1 - 1 : R1) - wrow0;  // so is a cut tail
                const int total = (skip & 4) ? 0 : nnz * kk;
                int c = gt % kk, s = gt / kk;
                const int dc = GT % kk, ds = GT / kk;
                for (int e = gt; e < total; e += GT) {
                    const int lr = G.rrow[GEE_IDX(s, wnz, 9)];
                    if (lr >= lr_lo && lr < lr_hi) {
                        const int idx = GEE_IDX(s * kk + c, wnz * kk, 10);
                        float v;
                        if (WEIGHTED) {
                            v = (float)(long long)(((unsigned long long)G.hi[idx] << 32) | G.lo[idx]);
                            G.hi[idx] = 0u;
                        } else {
                            v = (float)G.lo[idx];
                        }
                        G.lo[idx] = 0u;
                        __stcs(z + (int64_t)(wrow0 + lr) * kk + c, v * sc[c + 1]);
                    }
                    c += dc;
                    s += ds;
                    if (c >= kk) {
                        c -= kk;
                        s++;
                    }
                }
            }
            // partial rows: the head (owned by an earlier tile) and a cut tail
            for (int part = 0; part < 2; part++) {
                int32_t row;
                if (part == 0) {
                    if (!(has_head && first)) continue;
                    row = base;
                } else {
                    if (!tail_cut) continue;
                    row = R1 - 1;
                    if (row < wrow0 || row >= wrow0 + nr) continue;
                }
                if (skip & 16) continue;
                const int64_t owner = part == 0 ? __ldg(offsets + row) / TILE : j;
                const int slot = G.nzr[GEE_IDX(row - wrow0, nr, 13)];
                for (int c = gt; c < kk; c += GT) {
                    const int idx = GEE_IDX(slot * kk + c, wnz * kk, 14);
                    const unsigned long long v =
                        WEIGHTED ? (((unsigned long long)G.hi[idx] << 32) | G.lo[idx]) : (unsigned long long)G.lo[idx];
                    G.lo[idx] = 0u;
                    if (WEIGHTED) G.hi[idx] = 0u;
                    if (v) atomicAdd(&slots[owner * kk + c], v);
                }
            }
            wrow0 += nr;
            first = false;
        }
        // rotate the pipeline registers
        if constexpr (CLS) {
            if (jn < n_tiles) {
                R0 = A.r0;
                R1 = A.r1;
                crow = A.crow;
#pragma unroll
                for (int v = 0; v < 4; v++) cw[v] = (uint32_t)A.t[v];
#pragma unroll
                for (int i = 0; i < APT; i++) wcur[i] = A.w[i];
                if (jn + stride < n_tiles)
                    load_arcs<WEIGHTED, CLS>(A, jn + stride, gt, targets, wts, tile_row, chunk_row, arcs, sentinel);
            }
        } else {
            R0 = nR0;
            R1 = nR1;
            crow = ncrow;
            pos = npos;
#pragma unroll
            for (int i = 0; i < APT; i++) wcur[i] = wnext[i];
        }
        buf ^= 1;
    }
    cp_async_wait<0>();
}

// Write the rows that spanned tiles from their owner's slot; re-zero slots.
template <bool WEIGHTED>
__global__ void k_pull_finalize(const int32_t *__restrict__ cut, int64_t n_cut, const int64_t *__restrict__ tile_row,
                                unsigned long long *__restrict__ slots, const double *__restrict__ inv, int32_t k,
                                double dscale, float *__restrict__ z)
{
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t i = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; i < n_cut; i += warps) {
        const int64_t j = cut[i];
        const int64_t row = tile_row[j + 1] - 1;
        for (int c = lane; c < k; c += 32) {
            const unsigned long long v = slots[j * k + c];
            slots[j * k + c] = 0ull;
            const float f = WEIGHTED ? (float)(long long)v : (float)v;
            z[row * (int64_t)k + c] = f * (float)(inv[c + 1] * dscale);
        }
    }
}

// Zero the Z rows with no arcs (the pull kernel writes only nonempty rows).
// One warp per 32 consecutive rows: a ballot marks the empty ones, then the
// warp writes their k floats as one coalesced flat range.
__global__ void k_zero_empty(const int64_t *__restrict__ offsets, int64_t n, int32_t k, float *__restrict__ z)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int c0 = lane % k, r0l = lane / k;
    const int dc = 32 % k, dr = 32 / k;
    for (int64_t r0 = ((((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5) * 32; r0 < n; r0 += warps * 32) {
        const int64_t r = r0 + lane;
        const bool empty = r < n && __ldcs(offsets + r + 1) == __ldcs(offsets + r);
        const unsigned mask = __ballot_sync(0xffffffffu, empty);
        if (!mask) continue;
        const int rows = (int)min((int64_t)32, n - r0);
        const int total = rows * k;
        float *zo = z + r0 * (int64_t)k;
        int c = c0, rr = r0l;
        for (int e = lane; e < total; e += 32) {
            if ((mask >> rr) & 1u) __stcs(zo + e, 0.f);
            c += dc;
            rr += dr;
            if (c >= k) {
                c -= k;
                rr++;
            }
        }
    }
}

size_t group_fixed_smem(bool cls)
{
    return 2 * ((OFF_MAX + 1) & ~1) * sizeof(int64_t) + (cls ? 0 : 2 * TILE * sizeof(uint32_t)) +
           ((OFF_MAX + 3 + 3) & ~3) * sizeof(int32_t) + 2 * WROWS * sizeof(uint16_t) + 16 * sizeof(int32_t);
}

struct PullShape {
    int wnz;  // nonempty rows per window
    int hot0;
    size_t smem;
};

PullShape pull_shape(int32_t k, bool weighted, int64_t n_hot, int label_bytes, size_t budget, bool cls)
{
    PullShape p{0, 0, 0};
    const int GROUPS = cls ? groups_for<true>() : groups_for<false>();
    const size_t sc = ((size_t)(k + 4) & ~(size_t)3) * sizeof(float);
    const size_t per_row = (size_t)k * sizeof(uint32_t) * (weighted ? 2 : 1);
    const size_t fixed = sc + GROUPS * group_fixed_smem(cls) + 64;
    if (fixed + GROUPS * (per_row + 16) > budget) return p;
    size_t win_bytes = (budget - fixed) / GROUPS;
    // windows hold a tile's nonempty rows; beyond ~WIN_HOT_BYTES per group the
    // smem is worth more as L1 (the gathers go through it)
    if (win_bytes > WIN_HOT_BYTES) win_bytes = WIN_HOT_BYTES > per_row ? WIN_HOT_BYTES : per_row;
    int wnz = (int)(win_bytes / per_row);
    if (wnz > WROWS) wnz = WROWS;
    const size_t plane = ((((size_t)wnz * k + 3) & ~(size_t)3) * sizeof(uint32_t));
    const size_t used = fixed + GROUPS * plane * (weighted ? 2 : 1);
    size_t hot_cap = used + 32 < budget ? (budget - used - 32) / (size_t)label_bytes : 0;
    hot_cap &= ~(size_t)15;
    p.wnz = wnz;
    p.hot0 = (int)(n_hot < (int64_t)hot_cap ? n_hot : (int64_t)hot_cap);
    p.hot0 &= ~15;  // whole 16 B vectors; the rest of the hot tier is read through L2
    p.smem = used + (((size_t)p.hot0 * label_bytes + 16 + 15) & ~(size_t)15);  // >= 16 B: slot 0 always readable
    return p;
}

template <bool WEIGHTED, typename LT, bool CLS>
int launch_pull(const int64_t *offsets, const int32_t *targets, const float *w, int64_t n, int64_t arcs,
                const int64_t *tile_row, const uint16_t *chunk_row, const int32_t *cut, int64_t n_cut,
                int32_t scale_exp, const LT *table, int64_t n_hot, const double *inv, int32_t k, float *z,
                unsigned long long *slots, cudaStream_t st)
{
    const int64_t n_tiles = gee_pull_tiles(arcs);
    static int optin = 0;
    if (!optin) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
            optin = 48 * 1024;
    }
    const size_t budget = (size_t)(optin < SMEM_BYTES_MAX ? optin : SMEM_BYTES_MAX);
    // The hot tier is read through L1/L2: staging its head in shared memory
    // measured 3x slower on C4 (skewed LDS bank conflicts, and the carve-out
    // starves L1); GEE_PULL_SMEM_HOT=1 re-enables it for experiments.
    static const bool smem_hot = getenv("GEE_PULL_SMEM_HOT") != nullptr;
    const PullShape ps = pull_shape(k, WEIGHTED, (CLS || !smem_hot) ? 0 : n_hot, (int)sizeof(LT), budget, CLS);
    constexpr int GROUPS = groups_for<CLS>();
    constexpr int PT = GROUPS * GT;
    GEE_REQUIRE(ps.wnz >= 1, GEE_ERR_INVALID, "k=%d too large for the pull window", k);
    auto kern = k_pull<WEIGHTED, LT, CLS>;
    {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps.smem);
        GEE_REQUIRE(e == cudaSuccess, GEE_ERR_CUDA, "k_pull: %zu B dynamic smem (opt-in max %d, window %d rows, hot %d): %s",
                    ps.smem, optin, ps.wnz, ps.hot0, cudaGetErrorString(e));
    }
    const int64_t ctas = (n_tiles + GROUPS - 1) / GROUPS;
    const int64_t cap = (int64_t)gee::sm_count();
    const int grid = (int)(ctas < cap ? ctas : cap);
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = WEIGHTED ? ldexp(1.0, -scale_exp) : 1.0;
    const int32_t sentinel = (int32_t)(n_hot + n);
    static const int skip = getenv("GEE_PULL_SKIP") ? atoi(getenv("GEE_PULL_SKIP")) : 0;
    if (getenv("GEE_PULL_VERBOSE"))
        fprintf(stderr, "k_pull grid %d x %d smem %zu wnz %d hot0 %d tiles %lld cut %lld skip %d\n", grid, PT, ps.smem,
                ps.wnz, ps.hot0, (long long)n_tiles, (long long)n_cut, skip);
    kern<<<grid, PT, ps.smem, st>>>(offsets, targets, w, arcs, tile_row, chunk_row, n_tiles, qscale, dscale, table,
                                    sentinel, ps.hot0, inv, k, z, slots, ps.wnz, skip);
    int rc = gee::check_launch("k_pull");
    if (rc) return rc;
    if (n_cut > 0) {
        const int64_t want = (n_cut * 32 + 255) / 256;
        const int64_t fcap = (int64_t)gee::sm_count() * 16;
        const int fgrid = (int)(want < 1 ? 1 : (want > fcap ? fcap : want));
        k_pull_finalize<WEIGHTED><<<fgrid, 256, 0, st>>>(cut, n_cut, tile_row, slots, inv, k, dscale, z);
        rc = gee::check_launch("k_pull_finalize");
    }
    return rc;
}

int grid_for(int64_t items)
{
    int64_t want = (items + 255) / 256;
    int64_t cap = (int64_t)gee::sm_count() * 16;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" {

/* Debug builds: first recorded bounds violation in the pull kernels. */
int gee_debug_word(unsigned int *out4)
{
#ifdef GEE_DEBUG
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out4, g_gee_dbg, sizeof(unsigned int) * 4) != cudaSuccess) return GEE_ERR_CUDA;
    unsigned int zero[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_gee_dbg, zero, sizeof(zero));
#else
    out4[0] = out4[1] = out4[2] = out4[3] = 0;
#endif
    return GEE_OK;
}

int64_t gee_pull_tiles(int64_t arcs) { return arcs <= 0 ? 0 : (arcs + TILE - 1) / TILE; }

int64_t gee_pull_chunks(int64_t arcs) { return arcs <= 0 ? 0 : (arcs + APT - 1) / APT; }

size_t gee_pull_slots_bytes(int64_t arcs, int32_t k)
{
    int64_t t = gee_pull_tiles(arcs);
    return (size_t)(t ? t : 1) * (size_t)(k > 0 ? k : 1) * sizeof(unsigned long long);
}

int gee_pull_plan(const int64_t *offsets, int64_t n, int64_t arcs, int64_t *tile_row, uint16_t *chunk_row,
                  int32_t *cut_tiles, int64_t *n_cut, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && arcs >= 0, GEE_ERR_INVALID, "n and arcs must be nonnegative");
    GEE_REQUIRE(n_cut != nullptr, GEE_ERR_INVALID, "n_cut must not be NULL");
    const int64_t n_tiles = gee_pull_tiles(arcs);
    cudaStream_t st = gee::as_stream(stream);
    *n_cut = 0;
    k_pull_plan<<<(unsigned)((n_tiles + 1 + 255) / 256), 256, 0, st>>>(offsets, n, arcs, n_tiles, tile_row);
    int rc = gee::check_launch("k_pull_plan");
    if (rc || n_tiles == 0) return rc;
    GEE_REQUIRE(chunk_row && cut_tiles, GEE_ERR_INVALID, "chunk_row / cut_tiles must not be NULL");
    k_chunk_rows<<<grid_for(gee_pull_chunks(arcs)), 256, 0, st>>>(offsets, tile_row, arcs, chunk_row);
    if ((rc = gee::check_launch("k_chunk_rows"))) return rc;
    unsigned long long *cnt = nullptr;
    unsigned long long h = 0;
    GEE_CUDA(cudaMallocAsync((void **)&cnt, sizeof(unsigned long long), st));
    GEE_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    k_cut_tiles<<<grid_for(n_tiles), 256, 0, st>>>(offsets, tile_row, arcs, n_tiles, cut_tiles, cnt);
    rc = gee::check_launch("k_cut_tiles");
    cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(cnt, st);
    GEE_CUDA(cudaStreamSynchronize(st));
    *n_cut = (int64_t)h;
    return rc;
}

int gee_pull_scale_exp(double max_row_abs, double min_abs_nz, int32_t *scale_exp, double *rel_err)
{
    gee::clear_error();
    GEE_REQUIRE(scale_exp != nullptr, GEE_ERR_INVALID, "scale_exp must not be NULL");
    int e = 0;
    if (max_row_abs > 0) {
        // largest e with max_row_abs * 2^e < 2^62 (one bit of headroom below int64)
        int ex;
        frexp(max_row_abs, &ex);  // max_row_abs < 2^ex
        e = 62 - ex;
        if (e > 126) e = 126;     // 2^e must be a finite float
        if (e < -126) e = -126;
    }
    *scale_exp = e;
    if (rel_err) *rel_err = min_abs_nz > 0 ? ldexp(1.0, -(e + 1)) / min_abs_nz : 0.0;
    return GEE_OK;
}

int gee_embed_csr_pull(const int64_t *offsets, const int32_t *targets, const float *w, int64_t n, int64_t arcs,
                       const int64_t *tile_row, const uint16_t *chunk_row, const int32_t *cut_tiles, int64_t n_cut,
                       int32_t scale_exp, const void *table, int64_t n_hot, const double *inv, int32_t k, float *z,
                       void *slots, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && arcs >= 0 && n_hot >= 0 && n_cut >= 0, GEE_ERR_INVALID,
                "n, arcs, n_hot and n_cut must be nonnegative");
    GEE_REQUIRE(n + n_hot < INT32_MAX, GEE_ERR_INVALID, "label table exceeds int32 slots");
    cudaStream_t st = gee::as_stream(stream);
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && tile_row && z, GEE_ERR_INVALID, "NULL array argument");
    if (arcs == 0) {
        GEE_CUDA(cudaMemsetAsync(z, 0, sizeof(float) * (size_t)n * k, st));
        return GEE_OK;
    }
    GEE_REQUIRE(targets && chunk_row && table && inv && slots && (n_cut == 0 || cut_tiles), GEE_ERR_INVALID,
                "NULL array argument");
    GEE_REQUIRE(gee::aligned16(targets) && (!w || gee::aligned16(w)) && gee::aligned16(table), GEE_ERR_INVALID,
                "targets/weights/table must be 16-byte aligned");
    {
        // Rows with no arcs (isolated vertices, trailing rows) are zeroed
        // here; the pull kernel writes exactly the nonempty rows.
        const int64_t warps = (n + 31) / 32;
        const int64_t want = (warps * 32 + 255) / 256;
        const int64_t cap = (int64_t)gee::sm_count() * 8;
        k_zero_empty<<<(int)(want < cap ? (want < 1 ? 1 : want) : cap), 256, 0, st>>>(offsets, n, k, z);
        int rc = gee::check_launch("k_zero_empty");
        if (rc) return rc;
    }
    auto *sl = reinterpret_cast<unsigned long long *>(slots);
    switch (gee_label_bytes(k)) {
    case 1: {
        const auto *t = static_cast<const uint8_t *>(table);
        return w ? launch_pull<true, uint8_t, false>(offsets, targets, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut,
                                              scale_exp, t, n_hot, inv, k, z, sl, st)
                 : launch_pull<false, uint8_t, false>(offsets, targets, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut,
                                               scale_exp, t, n_hot, inv, k, z, sl, st);
    }
    case 2: {
        const auto *t = static_cast<const uint16_t *>(table);
        return w ? launch_pull<true, uint16_t, false>(offsets, targets, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut,
                                               scale_exp, t, n_hot, inv, k, z, sl, st)
                 : launch_pull<false, uint16_t, false>(offsets, targets, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut,
                                                scale_exp, t, n_hot, inv, k, z, sl, st);
    }
    default: {
        const auto *t = static_cast<const int32_t *>(table);
        return w ? launch_pull<true, int32_t, false>(offsets, targets, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut,
                                              scale_exp, t, n_hot, inv, k, z, sl, st)
                 : launch_pull<false, int32_t, false>(offsets, targets, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut,
                                               scale_exp, t, n_hot, inv, k, z, sl, st);
    }
    }
}

int gee_embed_csr_pull_cls(const int64_t *offsets, const uint8_t *cls, const float *w, int64_t n, int64_t arcs,
                           const int64_t *tile_row, const uint16_t *chunk_row, const int32_t *cut_tiles,
                           int64_t n_cut, int32_t scale_exp, const double *inv, int32_t k, float *z, void *slots,
                           void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs 1 <= k <= 255 (got %d)", k);
    GEE_REQUIRE(n >= 0 && arcs >= 0 && n_cut >= 0, GEE_ERR_INVALID, "n, arcs and n_cut must be nonnegative");
    cudaStream_t st = gee::as_stream(stream);
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && tile_row && z, GEE_ERR_INVALID, "NULL array argument");
    if (arcs == 0) {
        GEE_CUDA(cudaMemsetAsync(z, 0, sizeof(float) * (size_t)n * k, st));
        return GEE_OK;
    }
    GEE_REQUIRE(cls && chunk_row && inv && slots && (n_cut == 0 || cut_tiles), GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(gee::aligned16(cls) && (!w || gee::aligned16(w)), GEE_ERR_INVALID, "cls/weights must be 16-byte aligned");
    {
        const int64_t warps = (n + 31) / 32;
        const int64_t want = (warps * 32 + 255) / 256;
        const int64_t cap = (int64_t)gee::sm_count() * 8;
        k_zero_empty<<<(int)(want < cap ? (want < 1 ? 1 : want) : cap), 256, 0, st>>>(offsets, n, k, z);
        int rc = gee::check_launch("k_zero_empty");
        if (rc) return rc;
    }
    auto *sl = reinterpret_cast<unsigned long long *>(slots);
    const auto *tg = reinterpret_cast<const int32_t *>(cls);
    const uint8_t *no_table = nullptr;
    return w ? launch_pull<true, uint8_t, true>(offsets, tg, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut, scale_exp,
                                                no_table, 0, inv, k, z, sl, st)
             : launch_pull<false, uint8_t, true>(offsets, tg, w, n, arcs, tile_row, chunk_row, cut_tiles, n_cut, scale_exp,
                                                 no_table, 0, inv, k, z, sl, st);
}

}  // extern "C"
