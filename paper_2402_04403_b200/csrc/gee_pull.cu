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
//   tile j = arcs [j*T, (j+1)*T), T = GEE_TILE_ARCS = 512 threads x 8 arcs;
//   tile j OWNS the rows whose first-arc position offsets[r] lies in it;
//   tile_row[j] = first owned row (gee_pull_plan, a lower_bound per tile).
//   The row of each arc comes from a block scan of row-start marks, so no
//   per-arc binary search is needed.  Rows that run past their owner tile
//   (hubs) are summed exactly through 64-bit global atomics into the owner
//   tile's slot and written by k_pull_finalize.
#include "gee_common.cuh"

namespace {

constexpr int PULL_THREADS = 512;
constexpr int PULL_APT = 8;                             // arcs per thread
constexpr int TILE = PULL_THREADS * PULL_APT;           // 4096
static_assert(TILE == GEE_TILE_ARCS, "tile size mismatch with header");
constexpr int PULL_SMEM_BYTES = 100 * 1024;             // 2 CTAs per SM
constexpr int MARK_WORDS = TILE + 4;
constexpr int SCAN_WORDS = 32;

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
// tile_row[n_tiles] = first row with offsets[r] >= arcs (trailing empty rows
// start there and are zero-filled by the host wrapper).
__global__ void k_pull_plan(const int64_t *__restrict__ offsets, int64_t n, int64_t arcs,
                            int64_t n_tiles, int64_t *__restrict__ tile_row)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j > n_tiles) return;
    int64_t key = j < n_tiles ? j * (int64_t)TILE : arcs;
    tile_row[j] = lower_bound_i64(offsets, 0, n + 1, key);
}

template <typename LB, bool WEIGHTED>
__global__ void __launch_bounds__(PULL_THREADS, 2)
k_pull(const int64_t *__restrict__ offsets, const int32_t *__restrict__ targets,
       const float *__restrict__ w, int64_t n, int64_t arcs,
       const int64_t *__restrict__ tile_row, float qscale, double dscale,
       const LB *__restrict__ labels, const double *__restrict__ inv, int32_t k,
       float *__restrict__ z, unsigned long long *__restrict__ slots, int win_rows)
{
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *marks = smem;                         // MARK_WORDS
    uint32_t *scan = smem + MARK_WORDS;             // SCAN_WORDS
    uint32_t *acc_lo = scan + SCAN_WORDS;           // win_rows * k
    uint32_t *acc_hi = acc_lo + (size_t)win_rows * k;  // weighted only

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int64_t j = blockIdx.x;
    const int64_t a0 = j * (int64_t)TILE;
    const int64_t a1 = min(a0 + (int64_t)TILE, arcs);
    const int64_t R0 = tile_row[j], R1 = tile_row[j + 1];
    // Head row: the row holding arc a0 started in an earlier tile.
    const bool has_head = (R0 >= n) || (offsets[R0] > a0);
    const int64_t base = has_head ? R0 - 1 : R0;
    // Tail row: the last owned row continues into later tiles.
    const bool tail_cut = (R1 > R0) && (offsets[R1] > a1);

    // 1-2. Row-start marks: marks[p] = number of owned rows whose first arc
    // position is a0 + p (empty rows share a position).
    for (int i = tid; i < MARK_WORDS; i += PULL_THREADS) marks[i] = 0;
    __syncthreads();
    for (int64_t r = R0 + tid; r < R1; r += PULL_THREADS)
        atomicAdd(&marks[offsets[r] - a0], 1u);
    __syncthreads();

    // 3. This thread's arcs, their marks, and the arc -> row mapping.
    const int64_t e0 = a0 + (int64_t)tid * PULL_APT;
    int32_t tgt[PULL_APT];
    float wt[PULL_APT];
    uint32_t cnt[PULL_APT];
    {
        const uint4 m0 = *reinterpret_cast<const uint4 *>(marks + tid * PULL_APT);
        const uint4 m1 = *reinterpret_cast<const uint4 *>(marks + tid * PULL_APT + 4);
        cnt[0] = m0.x; cnt[1] = m0.y; cnt[2] = m0.z; cnt[3] = m0.w;
        cnt[4] = m1.x; cnt[5] = m1.y; cnt[6] = m1.z; cnt[7] = m1.w;
    }
    if (e0 + PULL_APT <= a1) {
        const int4 t0 = __ldcs(reinterpret_cast<const int4 *>(targets + e0));
        const int4 t1 = __ldcs(reinterpret_cast<const int4 *>(targets + e0 + 4));
        tgt[0] = t0.x; tgt[1] = t0.y; tgt[2] = t0.z; tgt[3] = t0.w;
        tgt[4] = t1.x; tgt[5] = t1.y; tgt[6] = t1.z; tgt[7] = t1.w;
        if (WEIGHTED) {
            const float4 w0 = __ldcs(reinterpret_cast<const float4 *>(w + e0));
            const float4 w1 = __ldcs(reinterpret_cast<const float4 *>(w + e0 + 4));
            wt[0] = w0.x; wt[1] = w0.y; wt[2] = w0.z; wt[3] = w0.w;
            wt[4] = w1.x; wt[5] = w1.y; wt[6] = w1.z; wt[7] = w1.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < PULL_APT; i++) {
            bool ok = e0 + i < a1;
            tgt[i] = ok ? __ldcs(targets + e0 + i) : -1;
            if (WEIGHTED) wt[i] = ok ? __ldcs(w + e0 + i) : 0.f;
        }
    }
    // Gather labels early: these are the latency-bound loads.
    uint32_t lab[PULL_APT];
#pragma unroll
    for (int i = 0; i < PULL_APT; i++) {
        lab[i] = tgt[i] >= 0 ? (uint32_t)__ldg(labels + tgt[i]) : 0u;
        if (sizeof(LB) == 4 && lab[i] > (uint32_t)k) lab[i] = 0u;  // raw int32 labels: drop out-of-range
    }

#pragma unroll
    for (int i = 1; i < PULL_APT; i++) cnt[i] += cnt[i - 1];
    uint32_t tot = cnt[PULL_APT - 1];
    uint32_t incl = tot;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) scan[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < PULL_THREADS / 32 ? scan[lane] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += u;
        }
        scan[lane] = v;  // inclusive per-warp totals
    }
    __syncthreads();
    const uint32_t pre = (warp ? scan[warp - 1] : 0u) + incl - tot;
    // local row index (0 = base) of each arc
    int32_t lrow[PULL_APT];
#pragma unroll
    for (int i = 0; i < PULL_APT; i++) lrow[i] = (int32_t)(pre + cnt[i]) - 1 + (has_head ? 1 : 0);

    int64_t q[PULL_APT];
    if (WEIGHTED) {
#pragma unroll
        for (int i = 0; i < PULL_APT; i++) q[i] = __float2ll_rn(wt[i] * qscale);
    }

    // 4-5. Windows of win_rows rows: accumulate, then write out.
    const int64_t rows_total = R1 - base;
    const int kk = k;
    for (int64_t wo = 0; wo < rows_total; wo += win_rows) {
        const int nr = (int)min((int64_t)win_rows, rows_total - wo);
        const int words = nr * kk;
        for (int i = tid; i < words; i += PULL_THREADS) {
            acc_lo[i] = 0;
            if (WEIGHTED) acc_hi[i] = 0;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < PULL_APT; i++) {
            const int lr = lrow[i] - (int)wo;
            if (lab[i] != 0 && lr >= 0 && lr < nr) {
                const int idx = lr * kk + (int)lab[i] - 1;
                if (WEIGHTED) {
                    const uint32_t lo = (uint32_t)(unsigned long long)q[i];
                    uint32_t hi = (uint32_t)((unsigned long long)q[i] >> 32);
                    const uint32_t old = atomicAdd(&acc_lo[idx], lo);
                    hi += (old + lo < old) ? 1u : 0u;  // carry out of the low plane
                    if (hi) atomicAdd(&acc_hi[idx], hi);
                } else {
                    atomicAdd(&acc_lo[idx], 1u);
                }
            }
        }
        __syncthreads();

        // Rows of this window that are complete in this tile.
        const int64_t wrow0 = base + wo;                   // global row of local 0
        const int64_t fin_lo = max(wrow0, R0);             // head row is partial
        const int64_t fin_hi = min(wrow0 + nr, tail_cut ? R1 - 1 : R1);
        if (fin_hi > fin_lo) {
            const int off = (int)(fin_lo - wrow0) * kk;
            const int64_t total = (fin_hi - fin_lo) * kk;
            float *zo = z + fin_lo * (int64_t)kk;
            // flat coalesced walk; (row, class) tracked incrementally
            int c = tid % kk, rr = tid / kk;
            const int dc = PULL_THREADS % kk, dr = PULL_THREADS / kk;
            for (int64_t e = tid; e < total; e += PULL_THREADS) {
                const int idx = off + rr * kk + c;
                double v;
                if (WEIGHTED) {
                    const long long s64 = (long long)(((unsigned long long)acc_hi[idx] << 32) | acc_lo[idx]);
                    v = (double)s64 * dscale;
                } else {
                    v = (double)acc_lo[idx];
                }
                zo[e] = (float)(v * __ldg(inv + c + 1));
                c += dc;
                rr += dr;
                if (c >= kk) { c -= kk; rr++; }
            }
        }
        // Partial rows: the head (owned by an earlier tile) and a cut tail.
        for (int part = 0; part < 2; part++) {
            int64_t row;
            if (part == 0) {
                if (!(has_head && wo == 0)) continue;
                row = base;
            } else {
                if (!tail_cut) continue;
                row = R1 - 1;
                if (row < wrow0 || row >= wrow0 + nr) continue;
            }
            const int64_t owner = part == 0 ? offsets[row] / TILE : j;
            const int lr = (int)(row - wrow0);
            for (int c = tid; c < kk; c += PULL_THREADS) {
                const int idx = lr * kk + c;
                unsigned long long v = WEIGHTED ? (((unsigned long long)acc_hi[idx] << 32) | acc_lo[idx])
                                                : (unsigned long long)acc_lo[idx];
                if (v) atomicAdd(&slots[owner * kk + c], v);
            }
        }
        __syncthreads();
    }
}

// Write the rows that spanned tiles from their owner's slot; re-zero slots.
template <bool WEIGHTED>
__global__ void k_pull_finalize(const int64_t *__restrict__ offsets, const int64_t *__restrict__ tile_row,
                                int64_t arcs, int64_t n_tiles, unsigned long long *__restrict__ slots,
                                const double *__restrict__ inv, int32_t k, double dscale,
                                float *__restrict__ z)
{
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t j = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; j < n_tiles; j += warps) {
        const int64_t R0 = tile_row[j], R1 = tile_row[j + 1];
        const int64_t a1 = min((j + 1) * (int64_t)TILE, arcs);
        if (!(R1 > R0 && offsets[R1] > a1)) continue;
        const int64_t row = R1 - 1;
        for (int c = lane; c < k; c += 32) {
            unsigned long long v = slots[j * k + c];
            slots[j * k + c] = 0ull;
            double d = WEIGHTED ? (double)(long long)v * dscale : (double)v;
            z[row * (int64_t)k + c] = (float)(d * inv[c + 1]);
        }
    }
}

__global__ void k_zero_tail(const int64_t *__restrict__ first_row, int64_t n, int32_t k,
                            float *__restrict__ z)
{
    const int64_t r0 = *first_row;
    const int64_t total = (n - r0) * (int64_t)k;
    float *zo = z + r0 * (int64_t)k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        zo[i] = 0.f;
}

int pull_win_rows(int32_t k, bool weighted)
{
    size_t avail = PULL_SMEM_BYTES - (MARK_WORDS + SCAN_WORDS) * sizeof(uint32_t);
    size_t per_row = (size_t)k * sizeof(uint32_t) * (weighted ? 2 : 1);
    return (int)(avail / per_row);
}

template <typename LB, bool WEIGHTED>
int launch_pull(const int64_t *offsets, const int32_t *targets, const float *w, int64_t n,
                int64_t arcs, const int64_t *tile_row, int32_t scale_exp, const void *labels,
                const double *inv, int32_t k, float *z, unsigned long long *slots, cudaStream_t st)
{
    const int64_t n_tiles = gee_pull_tiles(arcs);
    int win = pull_win_rows(k, WEIGHTED);
    GEE_REQUIRE(win >= 1, GEE_ERR_INVALID, "k=%d too large for the pull window", k);
    size_t sh = (MARK_WORDS + SCAN_WORDS) * sizeof(uint32_t) +
                (size_t)win * k * sizeof(uint32_t) * (WEIGHTED ? 2 : 1);
    auto kern = k_pull<LB, WEIGHTED>;
    GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = ldexp(1.0, -scale_exp);
    kern<<<(unsigned)n_tiles, PULL_THREADS, sh, st>>>(offsets, targets, w, n, arcs, tile_row, qscale,
                                                      dscale, (const LB *)labels, inv, k, z, slots, win);
    int rc = gee::check_launch("k_pull");
    if (rc) return rc;
    int64_t want = (n_tiles * 32 + 255) / 256;
    int64_t cap = (int64_t)gee::sm_count() * 16;
    int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    k_pull_finalize<WEIGHTED><<<grid, 256, 0, st>>>(offsets, tile_row, arcs, n_tiles, slots, inv, k,
                                                     dscale, z);
    return gee::check_launch("k_pull_finalize");
}

}  // namespace

extern "C" {

int64_t gee_pull_tiles(int64_t arcs) { return arcs <= 0 ? 0 : (arcs + TILE - 1) / TILE; }

size_t gee_pull_slots_bytes(int64_t arcs, int32_t k)
{
    int64_t t = gee_pull_tiles(arcs);
    return (size_t)(t ? t : 1) * (size_t)(k > 0 ? k : 1) * sizeof(unsigned long long);
}

int gee_pull_plan(const int64_t *offsets, int64_t n, int64_t arcs, int64_t *tile_row, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && arcs >= 0, GEE_ERR_INVALID, "n and arcs must be nonnegative");
    const int64_t n_tiles = gee_pull_tiles(arcs);
    cudaStream_t st = gee::as_stream(stream);
    k_pull_plan<<<(unsigned)((n_tiles + 1 + 255) / 256), 256, 0, st>>>(offsets, n, arcs, n_tiles, tile_row);
    return gee::check_launch("k_pull_plan");
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

int gee_embed_csr_pull(const int64_t *offsets, const int32_t *targets, const float *w, int64_t n,
                       int64_t arcs, const int64_t *tile_row, int32_t scale_exp, const void *labels,
                       int32_t label_bytes, const double *inv, int32_t k, float *z, void *slots,
                       void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && arcs >= 0, GEE_ERR_INVALID, "n and arcs must be nonnegative");
    GEE_REQUIRE(n <= INT32_MAX, GEE_ERR_INVALID, "node count %lld exceeds int32 targets", (long long)n);
    GEE_REQUIRE(label_bytes == 1 || label_bytes == 2 || label_bytes == 4, GEE_ERR_INVALID,
                "label_bytes must be 1, 2 or 4 (got %d)", label_bytes);
    GEE_REQUIRE(label_bytes >= gee_label_bytes(k), GEE_ERR_INVALID,
                "label_bytes %d too narrow for k=%d", label_bytes, k);
    cudaStream_t st = gee::as_stream(stream);
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && tile_row && z, GEE_ERR_INVALID, "NULL array argument");
    // Trailing rows with no arcs belong to no tile: zero them (the first such
    // row is tile_row[n_tiles], read on the device; no host sync).
    if (arcs == 0) {
        GEE_CUDA(cudaMemsetAsync(z, 0, sizeof(float) * (size_t)n * k, st));
        return GEE_OK;
    }
    {
        const int64_t n_tiles = gee_pull_tiles(arcs);
        k_zero_tail<<<gee::sm_count() * 2, 256, 0, st>>>(tile_row + n_tiles, n, k, z);
        int rc = gee::check_launch("k_zero_tail");
        if (rc) return rc;
    }
    if (arcs == 0) return GEE_OK;
    GEE_REQUIRE(targets && labels && inv && slots, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(gee::aligned16(targets) && (!w || gee::aligned16(w)), GEE_ERR_INVALID,
                "targets/weights must be 16-byte aligned");
    auto *sl = reinterpret_cast<unsigned long long *>(slots);
    const bool weighted = w != nullptr;
    switch (label_bytes) {
    case 1:
        return weighted ? launch_pull<uint8_t, true>(offsets, targets, w, n, arcs, tile_row, scale_exp, labels, inv, k, z, sl, st)
                        : launch_pull<uint8_t, false>(offsets, targets, w, n, arcs, tile_row, scale_exp, labels, inv, k, z, sl, st);
    case 2:
        return weighted ? launch_pull<uint16_t, true>(offsets, targets, w, n, arcs, tile_row, scale_exp, labels, inv, k, z, sl, st)
                        : launch_pull<uint16_t, false>(offsets, targets, w, n, arcs, tile_row, scale_exp, labels, inv, k, z, sl, st);
    default:
        return weighted ? launch_pull<int32_t, true>(offsets, targets, w, n, arcs, tile_row, scale_exp, labels, inv, k, z, sl, st)
                        : launch_pull<int32_t, false>(offsets, targets, w, n, arcs, tile_row, scale_exp, labels, inv, k, z, sl, st);
    }
}

}  // extern "C"
