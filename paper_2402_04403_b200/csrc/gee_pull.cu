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
//   tile j = arcs [j*T, (j+1)*T), T = GEE_TILE_ARCS = 256 threads x 8 arcs;
//   tile j OWNS the rows whose first-arc position offsets[r] lies in it;
//   tile_row[j] = first owned row (gee_pull_plan, a lower_bound per tile).
//   Persistent CTAs (4 per SM) walk tiles j = blockIdx.x, += gridDim.x.
//   Per tile: arcs stream in (128-bit, L2 evict-first), labels are gathered
//   (packed words, L2 evict-last), the tile's row offsets are staged in
//   shared memory and each thread finds its arcs' rows by one binary search
//   plus a forward walk.  Rows that run past their owner tile (hubs) are
//   summed exactly through 64-bit global atomics into the owner tile's slot
//   and written by k_pull_finalize.
#include "gee_common.cuh"

namespace {

constexpr int PT = 256;                  // threads per CTA
constexpr int APT = 8;                   // arcs per thread
constexpr int TILE = PT * APT;           // 2048
static_assert(TILE == GEE_TILE_ARCS, "tile size mismatch with header");
constexpr int CTAS_PER_SM = 4;
constexpr int SMEM_BYTES = 54 * 1024;    // 4 CTAs per SM (228 KB)
constexpr int OFF_MAX = 513;             // staged offsets per window (<= 512 rows)

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
// start there and are zero-filled by k_zero_tail).
__global__ void k_pull_plan(const int64_t *__restrict__ offsets, int64_t n, int64_t arcs,
                            int64_t n_tiles, int64_t *__restrict__ tile_row)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j > n_tiles) return;
    int64_t key = j < n_tiles ? j * (int64_t)TILE : arcs;
    tile_row[j] = lower_bound_i64(offsets, 0, n + 1, key);
}

__device__ __forceinline__ int4 ld_stream4(const int32_t *p) { return __ldcs(reinterpret_cast<const int4 *>(p)); }
__device__ __forceinline__ float4 ld_stream4(const float *p) { return __ldcs(reinterpret_cast<const float4 *>(p)); }

template <bool WEIGHTED>
__global__ void __launch_bounds__(PT, CTAS_PER_SM)
k_pull(const int64_t *__restrict__ offsets, const int32_t *__restrict__ targets,
       const float *__restrict__ w, int64_t arcs, const int64_t *__restrict__ tile_row, int64_t n_tiles,
       float qscale, double dscale, const uint32_t *__restrict__ labels, gee::LabelFmt lf,
       const double *__restrict__ inv, int32_t k, float *__restrict__ z,
       unsigned long long *__restrict__ slots, int win_rows)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int64_t *off_s = reinterpret_cast<int64_t *>(smem_raw);          // OFF_MAX
    float *sc = reinterpret_cast<float *>(off_s + OFF_MAX + 1);      // k+1 output scales
    uint32_t *acc_lo = reinterpret_cast<uint32_t *>(sc + ((k + 4) & ~3));
    uint32_t *acc_hi = acc_lo + (size_t)win_rows * k;                // weighted only

    const int tid = threadIdx.x;
    const int kk = k;
    const uint64_t pol = gee::policy_evict_last();
    // Z[x, c] = sum * sc[c+1]: inv folded with the fixed-point scale, fp32.
    for (int c = tid; c <= kk; c += PT) sc[c] = (float)(inv[c] * dscale);

    for (int64_t j = blockIdx.x; j < n_tiles; j += gridDim.x) {
        const int64_t a0 = j * (int64_t)TILE;
        const int64_t a1 = min(a0 + (int64_t)TILE, arcs);
        const int64_t e0 = a0 + (int64_t)tid * APT;
        // --- issue this thread's arc loads first (independent of the plan)
        int32_t tgt[APT];
        float wt[APT];
        if (e0 + APT <= a1) {
            const int4 t0 = ld_stream4(targets + e0), t1 = ld_stream4(targets + e0 + 4);
            tgt[0] = t0.x; tgt[1] = t0.y; tgt[2] = t0.z; tgt[3] = t0.w;
            tgt[4] = t1.x; tgt[5] = t1.y; tgt[6] = t1.z; tgt[7] = t1.w;
            if (WEIGHTED) {
                const float4 w0 = ld_stream4(w + e0), w1 = ld_stream4(w + e0 + 4);
                wt[0] = w0.x; wt[1] = w0.y; wt[2] = w0.z; wt[3] = w0.w;
                wt[4] = w1.x; wt[5] = w1.y; wt[6] = w1.z; wt[7] = w1.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < APT; i++) {
                const bool ok = e0 + i < a1;
                tgt[i] = ok ? __ldcs(targets + e0 + i) : -1;
                if (WEIGHTED) wt[i] = ok ? __ldcs(w + e0 + i) : 0.f;
            }
        }
        const int64_t R0 = tile_row[j], R1 = tile_row[j + 1];
        const int64_t offR0 = offsets[R0], offR1 = offsets[R1];
        // --- label gathers (latency-bound; all APT in flight)
        uint32_t lab[APT];
#pragma unroll
        for (int i = 0; i < APT; i++) {
            lab[i] = tgt[i] >= 0 ? gee::gather_label(labels, (uint32_t)tgt[i], lf, pol) : 0u;
            if (lab[i] > (uint32_t)kk) lab[i] = 0u;  // raw int32 labels: drop out-of-range
        }
        int64_t q[APT];
        if (WEIGHTED) {
#pragma unroll
            for (int i = 0; i < APT; i++) q[i] = __float2ll_rn(wt[i] * qscale);
        }
        // Head row: the row holding arc a0 started in an earlier tile.
        const bool has_head = offR0 > a0;  // also true when R0 == n (offsets[n] = arcs > a0)
        const int64_t base = has_head ? R0 - 1 : R0;
        // Tail row: the last owned row continues into later tiles.
        const bool tail_cut = (R1 > R0) && (offR1 > a1);
        const int64_t rows_total = R1 - base;

        for (int64_t wo = 0; wo < rows_total; wo += win_rows) {
            const int nr = (int)min((int64_t)win_rows, rows_total - wo);
            const int64_t wrow0 = base + wo;
            // stage offsets[wrow0 .. wrow0+nr] and zero the window
            for (int i = tid; i <= nr; i += PT) off_s[i] = __ldcs(offsets + wrow0 + i);
            const int words = nr * kk;
            for (int i = tid; i < words; i += PT) {
                acc_lo[i] = 0u;
                if (WEIGHTED) acc_hi[i] = 0u;
            }
            __syncthreads();
            // my arcs inside this window's arc range
            const int64_t wa0 = max(off_s[0], a0), wa1 = min(off_s[nr], a1);
            const int64_t m0 = max(e0, wa0), m1 = min(e0 + APT, wa1);
            if (m0 < m1) {
                // row of m0: last r in [0, nr) with off_s[r] <= m0
                int lo = 0, hi = nr;  // off_s[lo] <= m0 < off_s[hi]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (off_s[mid] <= m0) lo = mid;
                    else hi = mid;
                }
                int r = lo;
                int64_t next = off_s[r + 1];
#pragma unroll
                for (int i = 0; i < APT; i++) {
                    const int64_t e = e0 + i;
                    if (e < m0 || e >= m1) continue;
                    while (e >= next) next = off_s[++r + 1];
                    if (lab[i] == 0u) continue;
                    const int idx = r * kk + (int)lab[i] - 1;
                    if (WEIGHTED) {
                        const uint32_t lo32 = (uint32_t)(unsigned long long)q[i];
                        uint32_t hi32 = (uint32_t)((unsigned long long)q[i] >> 32);
                        const uint32_t old = atomicAdd(&acc_lo[idx], lo32);
                        hi32 += (old + lo32 < old) ? 1u : 0u;  // carry out of the low plane
                        if (hi32) atomicAdd(&acc_hi[idx], hi32);
                    } else {
                        atomicAdd(&acc_lo[idx], 1u);
                    }
                }
            }
            __syncthreads();

            // complete rows of this window -> Z (flat, coalesced, streaming stores)
            const int64_t fin_lo = max(wrow0, R0);  // a head row is partial
            const int64_t fin_hi = min(wrow0 + nr, tail_cut ? R1 - 1 : R1);
            if (fin_hi > fin_lo) {
                const int off = (int)(fin_lo - wrow0) * kk;
                const int total = (int)(fin_hi - fin_lo) * kk;
                float *zo = z + fin_lo * (int64_t)kk;
                int c = tid % kk, rr = tid / kk;
                const int dc = PT % kk, dr = PT / kk;
                for (int e = tid; e < total; e += PT) {
                    const int idx = off + rr * kk + c;
                    float v;
                    if (WEIGHTED) {
                        const long long s64 = (long long)(((unsigned long long)acc_hi[idx] << 32) | acc_lo[idx]);
                        v = (float)s64;
                    } else {
                        v = (float)acc_lo[idx];
                    }
                    __stcs(zo + e, v * sc[c + 1]);
                    c += dc;
                    rr += dr;
                    if (c >= kk) {
                        c -= kk;
                        rr++;
                    }
                }
            }
            // partial rows: the head (owned by an earlier tile) and a cut tail
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
                const int64_t owner = part == 0 ? off_s[0] / TILE : j;
                const int lr = (int)(row - wrow0);
                for (int c = tid; c < kk; c += PT) {
                    const int idx = lr * kk + c;
                    const unsigned long long v =
                        WEIGHTED ? (((unsigned long long)acc_hi[idx] << 32) | acc_lo[idx]) : (unsigned long long)acc_lo[idx];
                    if (v) atomicAdd(&slots[owner * kk + c], v);
                }
            }
            __syncthreads();
        }
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
            const unsigned long long v = slots[j * k + c];
            slots[j * k + c] = 0ull;
            const float f = WEIGHTED ? (float)(long long)v : (float)v;
            z[row * (int64_t)k + c] = f * (float)(inv[c + 1] * dscale);
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
        __stcs(zo + i, 0.f);
}

size_t pull_fixed_smem(int32_t k)
{
    return (OFF_MAX + 1) * sizeof(int64_t) + (size_t)((k + 4) & ~3) * sizeof(float);
}

int pull_win_rows(int32_t k, bool weighted)
{
    const size_t fixed = pull_fixed_smem(k);
    if (fixed >= SMEM_BYTES) return 0;
    const size_t per_row = (size_t)k * sizeof(uint32_t) * (weighted ? 2 : 1);
    int rows = (int)((SMEM_BYTES - fixed) / per_row);
    return rows > OFF_MAX - 1 ? OFF_MAX - 1 : rows;
}

template <bool WEIGHTED>
int launch_pull(const int64_t *offsets, const int32_t *targets, const float *w, int64_t arcs,
                const int64_t *tile_row, int32_t scale_exp, const uint32_t *labels, gee::LabelFmt lf,
                const double *inv, int32_t k, float *z, unsigned long long *slots, cudaStream_t st)
{
    const int64_t n_tiles = gee_pull_tiles(arcs);
    const int win = pull_win_rows(k, WEIGHTED);
    GEE_REQUIRE(win >= 1, GEE_ERR_INVALID, "k=%d too large for the pull window", k);
    const size_t sh = pull_fixed_smem(k) + (size_t)win * k * sizeof(uint32_t) * (WEIGHTED ? 2 : 1);
    auto kern = k_pull<WEIGHTED>;
    GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    int per_sm = 0;
    GEE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PT, sh));
    if (per_sm < 1) per_sm = 1;
    const int64_t cap = (int64_t)gee::sm_count() * per_sm;
    const int grid = (int)(n_tiles < cap ? n_tiles : cap);
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = WEIGHTED ? ldexp(1.0, -scale_exp) : 1.0;
    kern<<<grid, PT, sh, st>>>(offsets, targets, w, arcs, tile_row, n_tiles, qscale, dscale, labels, lf, inv, k, z,
                               slots, win);
    int rc = gee::check_launch("k_pull");
    if (rc) return rc;
    const int64_t want = (n_tiles * 32 + 255) / 256;
    const int64_t fcap = (int64_t)gee::sm_count() * 16;
    const int fgrid = (int)(want < 1 ? 1 : (want > fcap ? fcap : want));
    k_pull_finalize<WEIGHTED><<<fgrid, 256, 0, st>>>(offsets, tile_row, arcs, n_tiles, slots, inv, k, dscale, z);
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
                       int64_t arcs, const int64_t *tile_row, int32_t scale_exp, const uint32_t *labels,
                       int32_t label_bits, const double *inv, int32_t k, float *z, void *slots,
                       void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && arcs >= 0, GEE_ERR_INVALID, "n and arcs must be nonnegative");
    GEE_REQUIRE(n <= INT32_MAX, GEE_ERR_INVALID, "node count %lld exceeds int32 targets", (long long)n);
    GEE_REQUIRE(label_bits == 32 || label_bits == gee_label_bits(k), GEE_ERR_INVALID,
                "label_bits must be 32 (raw int32) or gee_label_bits(k)=%d (got %d)", gee_label_bits(k), label_bits);
    cudaStream_t st = gee::as_stream(stream);
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && tile_row && z, GEE_ERR_INVALID, "NULL array argument");
    // Trailing rows with no arcs belong to no tile: zero them (the first such
    // row is tile_row[n_tiles], read on the device; no host sync).
    if (arcs == 0) {
        GEE_CUDA(cudaMemsetAsync(z, 0, sizeof(float) * (size_t)n * k, st));
        return GEE_OK;
    }
    GEE_REQUIRE(targets && labels && inv && slots, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(gee::aligned16(targets) && (!w || gee::aligned16(w)), GEE_ERR_INVALID,
                "targets/weights must be 16-byte aligned");
    {
        const int64_t n_tiles = gee_pull_tiles(arcs);
        k_zero_tail<<<gee::sm_count() * 2, 256, 0, st>>>(tile_row + n_tiles, n, k, z);
        int rc = gee::check_launch("k_zero_tail");
        if (rc) return rc;
    }
    const gee::LabelFmt lf = gee::label_fmt(label_bits);
    auto *sl = reinterpret_cast<unsigned long long *>(slots);
    return w ? launch_pull<true>(offsets, targets, w, arcs, tile_row, scale_exp, labels, lf, inv, k, z, sl, st)
             : launch_pull<false>(offsets, targets, w, arcs, tile_row, scale_exp, labels, lf, inv, k, z, sl, st);
}

}  // extern "C"
