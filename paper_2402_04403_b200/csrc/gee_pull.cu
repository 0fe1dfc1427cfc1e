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
//   One persistent 512-thread CTA per SM walks tiles j = blockIdx.x,
//   += gridDim.x through a two-stage software pipeline: while tile j is
//   accumulated, tile j+G's labels are being gathered and its row offsets
//   staged (cp.async), and tile j+2G's arcs stream in (128-bit, L2
//   evict-first).  Targets are label-table slots (gee_common.cuh): the hot
//   tier's head is staged in shared memory, the rest of the table is read
//   through L2 (evict-last).  Rows use 32-bit tile-local offsets; a warp
//   brackets its first arc with two 32-way ballots and each lane gallops to
//   its own.  Rows that run past their owner tile (hubs) are
//   summed exactly through 64-bit global atomics into the owner tile's slot
//   and written by k_pull_finalize.
#include "gee_common.cuh"

namespace {

constexpr int PT = 512;                  // threads per CTA (one persistent CTA per SM)
constexpr int APT = 8;                   // arcs per thread
constexpr int TILE = PT * APT;           // 4096
static_assert(TILE == GEE_TILE_ARCS, "tile size mismatch with header");
constexpr int SMEM_BYTES_MAX = 227 * 1024;  // opt-in maximum per CTA on sm_100a (queried at launch)
constexpr int OFF_MAX = 513;             // staged offsets per buffer (<= 512 rows)
constexpr int WIN_BYTES_MAX = 120 * 1024;

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

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem)
{
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

struct TileArcs {  // stage A: streamed arcs of a tile
    int32_t t[APT];
    float w[APT];
    int32_t r0, r1;  // tile_row[j], tile_row[j+1]
};
struct TileLabs {  // stage B: gathered labels of a tile
    uint32_t l[APT];
    float w[APT];
    int32_t r0, r1;
};

template <bool WEIGHTED>
__device__ __forceinline__ void load_arcs(TileArcs &A, int64_t j, int tid, const int32_t *__restrict__ targets,
                                          const float *__restrict__ w, int64_t arcs,
                                          const int64_t *__restrict__ tile_row, int32_t sentinel)
{
    const int64_t e0 = j * (int64_t)TILE + (int64_t)tid * APT;
    if (e0 + APT <= arcs) {
        const int4 t0 = __ldcs(reinterpret_cast<const int4 *>(targets + e0));
        const int4 t1 = __ldcs(reinterpret_cast<const int4 *>(targets + e0 + 4));
        A.t[0] = t0.x; A.t[1] = t0.y; A.t[2] = t0.z; A.t[3] = t0.w;
        A.t[4] = t1.x; A.t[5] = t1.y; A.t[6] = t1.z; A.t[7] = t1.w;
        if (WEIGHTED) {
            const float4 w0 = __ldcs(reinterpret_cast<const float4 *>(w + e0));
            const float4 w1 = __ldcs(reinterpret_cast<const float4 *>(w + e0 + 4));
            A.w[0] = w0.x; A.w[1] = w0.y; A.w[2] = w0.z; A.w[3] = w0.w;
            A.w[4] = w1.x; A.w[5] = w1.y; A.w[6] = w1.z; A.w[7] = w1.w;
        }
    } else {  // last tile: padding arcs read the sentinel slot (label 0)
#pragma unroll
        for (int i = 0; i < APT; i++) {
            const bool ok = e0 + i < arcs;
            A.t[i] = ok ? __ldcs(targets + e0 + i) : sentinel;
            if (WEIGHTED) A.w[i] = ok ? __ldcs(w + e0 + i) : 0.f;
        }
    }
    A.r0 = (int32_t)tile_row[j];
    A.r1 = (int32_t)tile_row[j + 1];
}

// Labels of this thread's arcs: slots below hot0 from shared memory, the
// rest through L2 (one predicated load each; all APT in flight).
template <bool WEIGHTED, typename LT>
__device__ __forceinline__ void gather_labs(TileLabs &B, const TileArcs &A, const LT *__restrict__ table,
                                            const LT *__restrict__ hot_s, uint32_t hot0, uint64_t pol)
{
#pragma unroll
    for (int i = 0; i < APT; i++) {
        const uint32_t t = (uint32_t)A.t[i];
        const bool in_smem = t < hot0;
        uint32_t lab = (uint32_t)hot_s[in_smem ? t : 0u];
        if (!in_smem) lab = gee::ld_label<LT>(table + t, pol);
        B.l[i] = lab;
        if (WEIGHTED) B.w[i] = A.w[i];
    }
    B.r0 = A.r0;
    B.r1 = A.r1;
}

// Stage offsets[start .. start+cnt) into smem with cp.async (one 8 B copy per thread).
__device__ __forceinline__ void stage_offsets(int64_t *buf, const int64_t *__restrict__ offsets, int32_t r0,
                                              int32_t r1, int tid)
{
    const int32_t start = r0 > 0 ? r0 - 1 : 0;
    const int32_t cnt = min(r1 - start + 1, OFF_MAX);
    for (int i = tid; i < cnt; i += PT) cp_async8(buf + i, offsets + start + i);
}

template <bool WEIGHTED, typename LT>
__global__ void __launch_bounds__(PT, 1)
k_pull(const int64_t *__restrict__ offsets, const int32_t *__restrict__ targets,
       const float *__restrict__ w, int64_t arcs, const int64_t *__restrict__ tile_row, int64_t n_tiles,
       float qscale, double dscale, const LT *__restrict__ table, int32_t sentinel, int32_t hot0,
       const double *__restrict__ inv, int32_t k, float *__restrict__ z, unsigned long long *__restrict__ slots,
       int win_rows)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int64_t *off_buf = reinterpret_cast<int64_t *>(smem_raw);          // 2 x OFF_MAX int64
    int32_t *ol = reinterpret_cast<int32_t *>(off_buf + 2 * OFF_MAX);  // OFF_MAX (+3) tile-local int32
    float *sc = reinterpret_cast<float *>(ol + OFF_MAX + 3);           // k+1 output scales
    uint32_t *acc_lo = reinterpret_cast<uint32_t *>(sc + ((k + 4) & ~3));
    const size_t plane = ((size_t)win_rows * k + 3) & ~(size_t)3;      // 16 B aligned planes
    uint32_t *acc_hi = acc_lo + plane;                                 // weighted only
    LT *hot_s = reinterpret_cast<LT *>(acc_lo + plane * (WEIGHTED ? 2 : 1));

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int kk = k;
    const uint64_t pol = gee::policy_evict_last();
    // Z[x, c] = sum * sc[c+1]: inv folded with the fixed-point scale, fp32.
    for (int c = tid; c <= kk; c += PT) sc[c] = (float)(inv[c] * dscale);
    {  // stage the head of the label table (hot tier) with 16 B copies
        const int vec = (int)(((size_t)hot0 * sizeof(LT) + 15) / 16);
        const uint4 *src = reinterpret_cast<const uint4 *>(table);
        uint4 *dst = reinterpret_cast<uint4 *>(hot_s);
        for (int i = tid; i < vec; i += PT) dst[i] = __ldg(src + i);
    }
    __syncthreads();

    const int64_t G = gridDim.x;
    int64_t jA = blockIdx.x;
    if (jA >= n_tiles) return;
    TileArcs A;
    TileLabs B;
    // prologue: tile j0 gathered + offsets staged, tile j0+G arcs in flight
    load_arcs<WEIGHTED>(A, jA, tid, targets, w, arcs, tile_row, sentinel);
    gather_labs<WEIGHTED, LT>(B, A, table, hot_s, (uint32_t)hot0, pol);
    stage_offsets(off_buf, offsets, B.r0, B.r1, tid);
    cp_async_commit();
    jA += G;
    if (jA < n_tiles) load_arcs<WEIGHTED>(A, jA, tid, targets, w, arcs, tile_row, sentinel);
    int buf = 0;
    const int el0 = tid * APT;  // this thread's first arc, tile-local

    for (int64_t j = blockIdx.x; j < n_tiles; j += G) {
        uint32_t lab[APT];
        float wcur[APT];
#pragma unroll
        for (int i = 0; i < APT; i++) {
            lab[i] = B.l[i];
            if (WEIGHTED) wcur[i] = B.w[i];
        }
        const int32_t R0 = B.r0, R1 = B.r1;
        // advance the pipeline: gather tile j+G, stage its offsets, load tile j+2G
        if (jA < n_tiles) {
            gather_labs<WEIGHTED, LT>(B, A, table, hot_s, (uint32_t)hot0, pol);
            stage_offsets(off_buf + (buf ^ 1) * OFF_MAX, offsets, B.r0, B.r1, tid);
        }
        cp_async_commit();
        jA += G;
        if (jA < n_tiles) load_arcs<WEIGHTED>(A, jA, tid, targets, w, arcs, tile_row, sentinel);
        cp_async_wait<1>();  // tile j's staged offsets have landed (tile j+G's may be in flight)

        // ---- process tile j
        const int64_t a0 = j * (int64_t)TILE;
        const int tlen = (int)min((int64_t)TILE, arcs - a0);
        const int64_t *off_s = off_buf + buf * OFF_MAX;
        const int32_t st0 = R0 > 0 ? R0 - 1 : 0;  // first staged row
        int32_t scnt = min(R1 - st0 + 1, OFF_MAX);
        __syncthreads();  // staged offsets visible; previous tile's smem reads done
        // has_head: offsets[R0] > a0; tail_cut: offsets[R1] > a1 (read before ol is rewritten)
        const bool has_head = off_s[R0 - st0] > a0;  // also when R0 == n (offsets[n] = arcs > a0)
        const int64_t offR1 = (R1 - st0 < scnt) ? off_s[R1 - st0] : __ldcs(offsets + R1);
        const bool tail_cut = (R1 > R0) && (offR1 > a0 + tlen);
        const int32_t base = has_head ? R0 - 1 : R0;
        const int32_t rows_total = R1 - base;
        int32_t ost = st0;  // row of ol[0]

        for (int32_t wo = 0; wo < rows_total; wo += win_rows) {
            const int nr = min(win_rows, rows_total - wo);
            const int32_t wrow0 = base + wo;
            const int words = nr * kk;
            if (wo > 0) __syncthreads();  // previous window's write-out done
            if (wrow0 - ost + nr < scnt && wo == 0) {
                // tile-local int32 offsets, clamped to [0, TILE+1]
                for (int i = tid; i < scnt; i += PT) {
                    const int64_t v = off_s[i] - a0;
                    ol[i] = (int32_t)(v < 0 ? 0 : (v > TILE + 1 ? TILE + 1 : v));
                }
            } else {
                // window not fully staged (large tiles): load it directly
                for (int i = tid; i <= nr; i += PT) {
                    const int64_t v = __ldcs(offsets + wrow0 + i) - a0;
                    ol[i] = (int32_t)(v < 0 ? 0 : (v > TILE + 1 ? TILE + 1 : v));
                }
                ost = wrow0;
                scnt = nr + 1;
            }
            {  // zero the window
                uint4 *a4 = reinterpret_cast<uint4 *>(acc_lo);
                const int w4 = (words + 3) >> 2;
                const uint4 zero4 = make_uint4(0u, 0u, 0u, 0u);
                for (int i = tid; i < w4; i += PT) a4[i] = zero4;
                if (WEIGHTED) {
                    uint4 *h4 = reinterpret_cast<uint4 *>(acc_hi);
                    for (int i = tid; i < w4; i += PT) h4[i] = zero4;
                }
            }
            __syncthreads();
            const int32_t *ow = ol + (wrow0 - ost);  // ow[r] = offsets[wrow0 + r] - a0 (clamped)
            const int wa0 = ow[0], wa1 = min(ow[nr], tlen);
            const int m0 = max(el0, wa0), m1 = min(el0 + APT, wa1);
            // Row of the warp's first arc: two 32-way ballots.
            const int ew = max(el0 - lane * APT, wa0);
            int rw = 0;
            if (ew < wa1) {  // warp-uniform
                const int step = (nr + 31) >> 5;  // <= 16
                int cand = min(lane * step, nr);
                unsigned bal = __ballot_sync(0xffffffffu, ow[cand] <= ew);
                const int b = (31 - __clz(bal)) * step;  // ow[b] <= ew
                cand = min(b + lane, nr);
                bal = __ballot_sync(0xffffffffu, lane < step && ow[cand] <= ew);
                rw = b + (31 - __clz(bal));
            }
            if (m0 < m1) {
                // gallop from rw to the last r with ow[r] <= m0, then walk arcs
                int lo = rw, g = 1;
                while (lo + g < nr && ow[lo + g] <= m0) {
                    lo += g;
                    g <<= 1;
                }
                int hi = min(lo + g, nr);  // ow[lo] <= m0 < ow[hi]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (ow[mid] <= m0) lo = mid;
                    else hi = mid;
                }
                int r = lo;
                int next = ow[r + 1];
#pragma unroll
                for (int i = 0; i < APT; i++) {
                    const int e = el0 + i;
                    if (e < m0 || e >= m1) continue;
                    while (e >= next) next = ow[++r + 1];
                    const uint32_t c = lab[i];
                    if (c == 0u || c > (uint32_t)kk) continue;  // unlabeled (or out-of-range raw label)
                    const int idx = r * kk + (int)c - 1;
                    if (WEIGHTED) {
                        const unsigned long long q = (unsigned long long)__float2ll_rn(wcur[i] * qscale);
                        const uint32_t lo32 = (uint32_t)q;
                        uint32_t hi32 = (uint32_t)(q >> 32);
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
            const int32_t fin_lo = max(wrow0, R0);  // a head row is partial
            const int32_t fin_hi = min(wrow0 + nr, tail_cut ? R1 - 1 : R1);
            if (fin_hi > fin_lo) {
                const int off = (fin_lo - wrow0) * kk;
                const int total = (fin_hi - fin_lo) * kk;
                float *zo = z + (int64_t)fin_lo * kk;
                const uint32_t *plo = acc_lo + off;
                const uint32_t *phi = acc_hi + off;
                int c = tid % kk;
                const int dc = PT % kk;
                for (int e = tid; e < total; e += PT) {
                    float v;
                    if (WEIGHTED) v = (float)(long long)(((unsigned long long)phi[e] << 32) | plo[e]);
                    else v = (float)plo[e];
                    __stcs(zo + e, v * sc[c + 1]);
                    c += dc;
                    if (c >= kk) c -= kk;
                }
            }
            // partial rows: the head (owned by an earlier tile) and a cut tail
            for (int part = 0; part < 2; part++) {
                int32_t row;
                if (part == 0) {
                    if (!(has_head && wo == 0)) continue;
                    row = base;
                } else {
                    if (!tail_cut) continue;
                    row = R1 - 1;
                    if (row < wrow0 || row >= wrow0 + nr) continue;
                }
                const int64_t owner = part == 0 ? __ldg(offsets + row) / TILE : j;
                const int lr = row - wrow0;
                for (int c = tid; c < kk; c += PT) {
                    const int idx = lr * kk + c;
                    const unsigned long long v =
                        WEIGHTED ? (((unsigned long long)acc_hi[idx] << 32) | acc_lo[idx]) : (unsigned long long)acc_lo[idx];
                    if (v) atomicAdd(&slots[owner * kk + c], v);
                }
            }
        }
        buf ^= 1;
    }
    cp_async_wait<0>();
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
    return 2 * OFF_MAX * sizeof(int64_t) + (OFF_MAX + 3) * sizeof(int32_t) + (size_t)((k + 4) & ~3) * sizeof(float);
}

struct PullShape {
    int win_rows;
    int hot0;
    size_t smem;
};

PullShape pull_shape(int32_t k, bool weighted, int64_t n_hot, int label_bytes, size_t SMEM_BYTES)
{
    PullShape p{0, 0, 0};
    const size_t fixed = pull_fixed_smem(k);
    const size_t per_row = (size_t)k * sizeof(uint32_t) * (weighted ? 2 : 1);
    if (fixed + per_row + 16 > SMEM_BYTES) return p;
    size_t win_bytes = per_row * (OFF_MAX - 1);
    if (win_bytes > WIN_BYTES_MAX) win_bytes = WIN_BYTES_MAX > per_row ? WIN_BYTES_MAX : per_row;
    if (fixed + win_bytes + 16 > SMEM_BYTES) win_bytes = SMEM_BYTES - fixed - 16;
    p.win_rows = (int)(win_bytes / per_row);
    if (p.win_rows > OFF_MAX - 1) p.win_rows = OFF_MAX - 1;
    const size_t plane = (((size_t)p.win_rows * k + 3) & ~(size_t)3) * sizeof(uint32_t);
    const size_t used = fixed + plane * (weighted ? 2 : 1);
    size_t hot_cap = (SMEM_BYTES - used - 32) / (size_t)label_bytes;  // 32 B: rounding + the always-readable slot 0
    hot_cap &= ~(size_t)15;
    p.hot0 = (int)(n_hot < (int64_t)hot_cap ? n_hot : (int64_t)hot_cap);
    p.hot0 &= ~15;  // whole 16 B vectors; the rest of the hot tier is read through L2
    p.smem = used + (((size_t)p.hot0 * label_bytes + 16 + 15) & ~(size_t)15);  // >= 16 B: slot 0 always readable
    return p;
}

template <bool WEIGHTED, typename LT>
int launch_pull(const int64_t *offsets, const int32_t *targets, const float *w, int64_t n, int64_t arcs,
                const int64_t *tile_row, int32_t scale_exp, const LT *table, int64_t n_hot, const double *inv,
                int32_t k, float *z, unsigned long long *slots, cudaStream_t st)
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
    const PullShape ps = pull_shape(k, WEIGHTED, n_hot, (int)sizeof(LT), budget);
    GEE_REQUIRE(ps.win_rows >= 1, GEE_ERR_INVALID, "k=%d too large for the pull window", k);
    auto kern = k_pull<WEIGHTED, LT>;
    {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps.smem);
        GEE_REQUIRE(e == cudaSuccess, GEE_ERR_CUDA, "k_pull: %zu B dynamic smem (opt-in max %d, window %d rows, hot %d): %s",
                    ps.smem, optin, ps.win_rows, ps.hot0, cudaGetErrorString(e));
    }
    const int64_t cap = (int64_t)gee::sm_count();
    const int grid = (int)(n_tiles < cap ? n_tiles : cap);
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = WEIGHTED ? ldexp(1.0, -scale_exp) : 1.0;
    const int32_t sentinel = (int32_t)(n_hot + n);
    kern<<<grid, PT, ps.smem, st>>>(offsets, targets, w, arcs, tile_row, n_tiles, qscale, dscale, table, sentinel,
                                    ps.hot0, inv, k, z, slots, ps.win_rows);
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

int gee_embed_csr_pull(const int64_t *offsets, const int32_t *targets, const float *w, int64_t n, int64_t arcs,
                       const int64_t *tile_row, int32_t scale_exp, const void *table, int64_t n_hot,
                       const double *inv, int32_t k, float *z, void *slots, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && arcs >= 0 && n_hot >= 0, GEE_ERR_INVALID, "n, arcs and n_hot must be nonnegative");
    GEE_REQUIRE(n + n_hot < INT32_MAX, GEE_ERR_INVALID, "label table exceeds int32 slots");
    cudaStream_t st = gee::as_stream(stream);
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && tile_row && z, GEE_ERR_INVALID, "NULL array argument");
    // Trailing rows with no arcs belong to no tile: zero them (the first such
    // row is tile_row[n_tiles], read on the device; no host sync).
    if (arcs == 0) {
        GEE_CUDA(cudaMemsetAsync(z, 0, sizeof(float) * (size_t)n * k, st));
        return GEE_OK;
    }
    GEE_REQUIRE(targets && table && inv && slots, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(gee::aligned16(targets) && (!w || gee::aligned16(w)) && gee::aligned16(table), GEE_ERR_INVALID,
                "targets/weights/table must be 16-byte aligned");
    {
        const int64_t n_tiles = gee_pull_tiles(arcs);
        k_zero_tail<<<gee::sm_count() * 2, 256, 0, st>>>(tile_row + n_tiles, n, k, z);
        int rc = gee::check_launch("k_zero_tail");
        if (rc) return rc;
    }
    auto *sl = reinterpret_cast<unsigned long long *>(slots);
    switch (gee_label_bytes(k)) {
    case 1: {
        const auto *t = static_cast<const uint8_t *>(table);
        return w ? launch_pull<true, uint8_t>(offsets, targets, w, n, arcs, tile_row, scale_exp, t, n_hot, inv, k, z, sl, st)
                 : launch_pull<false, uint8_t>(offsets, targets, w, n, arcs, tile_row, scale_exp, t, n_hot, inv, k, z, sl, st);
    }
    case 2: {
        const auto *t = static_cast<const uint16_t *>(table);
        return w ? launch_pull<true, uint16_t>(offsets, targets, w, n, arcs, tile_row, scale_exp, t, n_hot, inv, k, z, sl, st)
                 : launch_pull<false, uint16_t>(offsets, targets, w, n, arcs, tile_row, scale_exp, t, n_hot, inv, k, z, sl, st);
    }
    default: {
        const auto *t = static_cast<const int32_t *>(table);
        return w ? launch_pull<true, int32_t>(offsets, targets, w, n, arcs, tile_row, scale_exp, t, n_hot, inv, k, z, sl, st)
                 : launch_pull<false, int32_t>(offsets, targets, w, n, arcs, tile_row, scale_exp, t, n_hot, inv, k, z, sl, st);
    }
    }
}

}  // extern "C"
