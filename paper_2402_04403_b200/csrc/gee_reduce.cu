// K4b: row-per-warp segmented reduction over the class stream (split pull).
//
// After gee_gather_labels has turned every arc x -> v of the symmetric CSR
// into its class byte cls[e] = Y[v], the pull pass is a gather-free
// segmented histogram per row (reference arc rule, _kernels.py:192-199):
//     Z[x, c] = inv[c+1] * sum_{e in row x, cls[e] = c+1} w[e].
//
// One warp per row, rows strided over all warps: no block barriers, so
// latency is hidden by occupancy and by a software pipeline across a warp's
// rows (offsets two rows ahead, the first 128 arcs one row ahead).  Each warp
// accumulates its row exactly in integers (u32 counts, or int64 fixed point
// as two u32 planes with carry) in a warp-private shared-memory vector, then
// writes the whole Z row (zeros for empty rows: no separate zero fill) and
// clears the vector as it reads it.  Rows heavier than GEE_HEAVY_ARCS are
// skipped here: gee_reduce_heavy splits them into chunks whose exact int64
// partials meet in a global accumulator, written by gee_reduce_heavy's
// finalize.  Z therefore is bit-stable and independent of arc order, like
// the tiled pull kernel (gee_pull.cu).
#include "gee_common.cuh"

namespace {

constexpr int RT = 256;       // threads per CTA
constexpr int RW = RT / 32;   // warps per CTA
constexpr int UNR = 4;        // arcs per lane per round (128 arcs per warp round)

template <bool WEIGHTED>
struct Acc {
    static constexpr int planes = WEIGHTED ? 2 : 1;
};

// Add arc (class c, weight wt) into a warp vector (lo plane at v, hi at v + k).
template <bool WEIGHTED>
__device__ __forceinline__ void acc_add(uint32_t *v, int k, uint32_t c, float wt, float qscale)
{
    if (WEIGHTED) {
        const unsigned long long q = (unsigned long long)__float2ll_rn(wt * qscale);
        const uint32_t lo32 = (uint32_t)q;
        uint32_t hi32 = (uint32_t)(q >> 32);
        const uint32_t old = atomicAdd(&v[c - 1], lo32);
        hi32 += (old + lo32 < old) ? 1u : 0u;  // carry out of the low plane
        if (hi32) atomicAdd(&v[k + c - 1], hi32);
    } else {
        atomicAdd(&v[c - 1], 1u);
    }
}

template <bool WEIGHTED>
__device__ __forceinline__ long long acc_take(uint32_t *v, int k, int c)
{
    const uint32_t lo = v[c];
    v[c] = 0u;
    if (!WEIGHTED) return (long long)lo;
    const uint32_t hi = v[k + c];
    v[k + c] = 0u;
    return (long long)(((unsigned long long)hi << 32) | lo);
}

template <bool WEIGHTED>
__global__ void __launch_bounds__(RT)
k_reduce_rows(const int64_t *__restrict__ offsets, int64_t n, const uint8_t *__restrict__ cls,
              const float *__restrict__ w, float qscale, double dscale, const double *__restrict__ inv, int32_t k,
              int64_t heavy_arcs, float *__restrict__ z)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *sc = reinterpret_cast<float *>(smem_raw);
    const int kk = k;
    const int vecw = ((kk + 3) & ~3) * Acc<WEIGHTED>::planes;  // words per warp vector
    uint32_t *vbase = reinterpret_cast<uint32_t *>(sc + ((kk + 4) & ~3));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *v = vbase + wid * vecw;
    for (int c = threadIdx.x; c <= kk; c += RT) sc[c] = (float)(inv[c] * dscale);
    for (int i = threadIdx.x; i < RW * vecw; i += RT) vbase[i] = 0u;
    __syncthreads();

    const int64_t gw = (int64_t)blockIdx.x * RW + wid, GW = (int64_t)gridDim.x * RW;
    const bool even = (kk & 1) == 0;
    // pipeline: offsets of rows r+GW (o_n) and r+2GW (o_nn in flight);
    // the current row's first round of arcs (c0/w0) loaded during the previous row
    int64_t r = gw;
    int64_t ob = 0, oe = 0;
    if (r < n) {
        ob = __ldcs(offsets + r);
        oe = __ldcs(offsets + r + 1);
    }
    int64_t obn = 0, oen = 0;
    if (r + GW < n) {
        obn = __ldcs(offsets + r + GW);
        oen = __ldcs(offsets + r + GW + 1);
    }
    uint32_t c0[UNR];
    float w0[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
        const int64_t e = ob + lane + 32 * u;
        const bool ok = e < oe && oe - ob <= heavy_arcs;
        c0[u] = ok ? __ldcs(cls + e) : 0u;
        w0[u] = (WEIGHTED && ok) ? __ldcs(w + e) : 0.f;
    }

    for (; r < n; r += GW) {
        const int64_t d = oe - ob;
        // ---- prefetch: next row's first round, the row after's offsets
        const int64_t rn = r + GW;
        uint32_t c1[UNR];
        float w1[UNR];
#pragma unroll
        for (int u = 0; u < UNR; u++) {
            const int64_t e = obn + lane + 32 * u;
            const bool ok = rn < n && e < oen && oen - obn <= heavy_arcs;
            c1[u] = ok ? __ldcs(cls + e) : 0u;
            w1[u] = (WEIGHTED && ok) ? __ldcs(w + e) : 0.f;
        }
        int64_t obnn = 0, oenn = 0;
        if (rn + GW < n) {
            obnn = __ldcs(offsets + rn + GW);
            oenn = __ldcs(offsets + rn + GW + 1);
        }

        float *zr = z + r * (int64_t)kk;
        if (d > heavy_arcs) {
            // heavy row: written by gee_reduce_heavy
        } else if (d == 0) {
            if (even) {
                float2 *z2 = reinterpret_cast<float2 *>(zr);
                for (int c = lane; c < (kk >> 1); c += 32) __stcs(z2 + c, make_float2(0.f, 0.f));
            } else {
                for (int c = lane; c < kk; c += 32) __stcs(zr + c, 0.f);
            }
        } else {
#pragma unroll
            for (int u = 0; u < UNR; u++)
                if (c0[u] != 0u && c0[u] <= (uint32_t)kk) acc_add<WEIGHTED>(v, vecw / Acc<WEIGHTED>::planes, c0[u], w0[u], qscale);
            for (int64_t e0 = ob + 32 * UNR; e0 < oe; e0 += 32 * UNR) {  // rows longer than one round
                uint32_t cc[UNR];
                float ww[UNR];
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    const int64_t e = e0 + lane + 32 * u;
                    cc[u] = e < oe ? __ldcs(cls + e) : 0u;
                    ww[u] = (WEIGHTED && e < oe) ? __ldcs(w + e) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < UNR; u++)
                    if (cc[u] != 0u && cc[u] <= (uint32_t)kk) acc_add<WEIGHTED>(v, vecw / Acc<WEIGHTED>::planes, cc[u], ww[u], qscale);
            }
            __syncwarp();
            const int pk = vecw / Acc<WEIGHTED>::planes;  // plane stride (k rounded up to 4)
            if (even) {
                float2 *z2 = reinterpret_cast<float2 *>(zr);
                for (int c2 = lane; c2 < (kk >> 1); c2 += 32) {
                    const float a = (float)acc_take<WEIGHTED>(v, pk, 2 * c2) * sc[2 * c2 + 1];
                    const float b = (float)acc_take<WEIGHTED>(v, pk, 2 * c2 + 1) * sc[2 * c2 + 2];
                    __stcs(z2 + c2, make_float2(a, b));
                }
            } else {
                for (int c = lane; c < kk; c += 32) __stcs(zr + c, (float)acc_take<WEIGHTED>(v, pk, c) * sc[c + 1]);
            }
            __syncwarp();
        }
        // rotate the pipeline
        ob = obn;
        oe = oen;
        obn = obnn;
        oen = oenn;
#pragma unroll
        for (int u = 0; u < UNR; u++) {
            c0[u] = c1[u];
            w0[u] = w1[u];
        }
    }
}

// Degree-binned variant: rows come from a prepared list (gee_reduce_bins);
// groups of GS lanes each own one row at a time (GS = 8 for rows of <= 32
// arcs, so a warp has 4 rows in flight; GS = 32 for medium rows, with the
// next 32*UNR-arc round loaded while the current one accumulates).  Each
// group prefetches its next row's offsets and first round.
template <bool WEIGHTED, int GS>
__global__ void __launch_bounds__(RT)
k_reduce_list(const int64_t *__restrict__ offsets, const int32_t *__restrict__ rows, int64_t n_rows,
              const uint8_t *__restrict__ cls, const float *__restrict__ w, float qscale, double dscale,
              const double *__restrict__ inv, int32_t k, float *__restrict__ z)
{
    constexpr int GPW = 32 / GS;  // groups per warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *sc = reinterpret_cast<float *>(smem_raw);
    const int kk = k;
    const int pk = (kk + 3) & ~3;
    const int vecw = pk * Acc<WEIGHTED>::planes;
    uint32_t *vbase = reinterpret_cast<uint32_t *>(sc + ((kk + 4) & ~3));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gid = lane / GS, gl = lane % GS;
    const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1u) << (gid * GS));
    uint32_t *v = vbase + (wid * GPW + gid) * vecw;
    for (int c = threadIdx.x; c <= kk; c += RT) sc[c] = (float)(inv[c] * dscale);
    for (int i = threadIdx.x; i < RW * GPW * vecw; i += RT) vbase[i] = 0u;
    __syncthreads();
    const bool even = (kk & 1) == 0;
    const int64_t G0 = ((int64_t)blockIdx.x * RW + wid) * GPW + gid;
    const int64_t GG = (int64_t)gridDim.x * RW * GPW;
    constexpr int ROUND = GS * UNR;

    int64_t i = G0;
    int64_t ob = 0, oe = 0, r = 0;
    if (i < n_rows) {
        r = rows[i];
        ob = __ldcs(offsets + r);
        oe = __ldcs(offsets + r + 1);
    }
    uint32_t c0[UNR];
    float w0[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
        const int64_t e = ob + gl + GS * u;
        c0[u] = (i < n_rows && e < oe) ? __ldcs(cls + e) : 0u;
        w0[u] = (WEIGHTED && i < n_rows && e < oe) ? __ldcs(w + e) : 0.f;
    }
    int64_t rn = 0, obn = 0, oen = 0;
    if (i + GG < n_rows) {
        rn = rows[i + GG];
        obn = __ldcs(offsets + rn);
        oen = __ldcs(offsets + rn + 1);
    }
    for (; i < n_rows; i += GG) {
        // prefetch the next row's first round and the row after's offsets
        uint32_t c1[UNR];
        float w1[UNR];
        const bool has_next = i + GG < n_rows;
#pragma unroll
        for (int u = 0; u < UNR; u++) {
            const int64_t e = obn + gl + GS * u;
            c1[u] = (has_next && e < oen) ? __ldcs(cls + e) : 0u;
            w1[u] = (WEIGHTED && has_next && e < oen) ? __ldcs(w + e) : 0.f;
        }
        int64_t rnn = 0, obnn = 0, oenn = 0;
        if (i + 2 * GG < n_rows) {
            rnn = rows[i + 2 * GG];
            obnn = __ldcs(offsets + rnn);
            oenn = __ldcs(offsets + rnn + 1);
        }
        float *zr = z + r * (int64_t)kk;
        if (oe == ob) {
            if (even) {
                float2 *z2 = reinterpret_cast<float2 *>(zr);
                for (int c = gl; c < (kk >> 1); c += GS) __stcs(z2 + c, make_float2(0.f, 0.f));
            } else {
                for (int c = gl; c < kk; c += GS) __stcs(zr + c, 0.f);
            }
        } else {
#pragma unroll
            for (int u = 0; u < UNR; u++)
                if (c0[u] != 0u && c0[u] <= (uint32_t)kk) acc_add<WEIGHTED>(v, pk, c0[u], w0[u], qscale);
            if (oe - ob > ROUND) {  // longer rows: rounds with the next one in flight
                uint32_t ca[UNR];
                float wa[UNR];
                int64_t e0 = ob + ROUND;
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    const int64_t e = e0 + gl + GS * u;
                    ca[u] = e < oe ? __ldcs(cls + e) : 0u;
                    wa[u] = (WEIGHTED && e < oe) ? __ldcs(w + e) : 0.f;
                }
                for (; e0 < oe; e0 += ROUND) {
                    uint32_t cb[UNR];
                    float wb[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; u++) {
                        const int64_t e = e0 + ROUND + gl + GS * u;
                        cb[u] = e < oe ? __ldcs(cls + e) : 0u;
                        wb[u] = (WEIGHTED && e < oe) ? __ldcs(w + e) : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < UNR; u++)
                        if (ca[u] != 0u && ca[u] <= (uint32_t)kk) acc_add<WEIGHTED>(v, pk, ca[u], wa[u], qscale);
#pragma unroll
                    for (int u = 0; u < UNR; u++) {
                        ca[u] = cb[u];
                        wa[u] = wb[u];
                    }
                }
            }
            __syncwarp(gmask);
            if (even) {
                float2 *z2 = reinterpret_cast<float2 *>(zr);
                for (int c2 = gl; c2 < (kk >> 1); c2 += GS) {
                    const float a = (float)acc_take<WEIGHTED>(v, pk, 2 * c2) * sc[2 * c2 + 1];
                    const float b = (float)acc_take<WEIGHTED>(v, pk, 2 * c2 + 1) * sc[2 * c2 + 2];
                    __stcs(z2 + c2, make_float2(a, b));
                }
            } else {
                for (int c = gl; c < kk; c += GS) __stcs(zr + c, (float)acc_take<WEIGHTED>(v, pk, c) * sc[c + 1]);
            }
            __syncwarp(gmask);
        }
        r = rn;
        ob = obn;
        oe = oen;
        rn = rnn;
        obn = obnn;
        oen = oenn;
#pragma unroll
        for (int u = 0; u < UNR; u++) {
            c0[u] = c1[u];
            w0[u] = w1[u];
        }
    }
}

// Bin rows by degree: small (<= small_arcs, incl. empty) and medium
// (<= heavy_arcs); heavier rows are left to the chunked path.
__global__ void k_bin_rows(const int64_t *__restrict__ offsets, int64_t n, int64_t small_arcs, int64_t heavy_arcs,
                           int32_t *__restrict__ small_rows, int32_t *__restrict__ medium_rows,
                           unsigned long long *__restrict__ counts)
{
    const int lane = threadIdx.x & 31;
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = base + lane;
        int64_t d = -1;
        if (r < n) d = offsets[r + 1] - offsets[r];
        const bool sm = r < n && d <= small_arcs, md = r < n && d > small_arcs && d <= heavy_arcs;
        // warp-aggregated appends keep each warp's rows consecutive in the lists
        const unsigned bs = __ballot_sync(0xffffffffu, sm), bm = __ballot_sync(0xffffffffu, md);
        unsigned long long ps = 0, pm = 0;
        if (lane == 0) {
            if (bs) ps = atomicAdd(&counts[0], (unsigned long long)__popc(bs));
            if (bm) pm = atomicAdd(&counts[1], (unsigned long long)__popc(bm));
        }
        ps = __shfl_sync(0xffffffffu, ps, 0);
        pm = __shfl_sync(0xffffffffu, pm, 0);
        const unsigned below = (1u << lane) - 1u;
        if (sm) small_rows[ps + __popc(bs & below)] = (int32_t)r;
        if (md) medium_rows[pm + __popc(bm & below)] = (int32_t)r;
    }
}

// Heavy rows: one warp per chunk of GEE_HEAVY_ARCS arcs; exact int64 partial
// sums meet in acc[h][c] through 64-bit global atomics.
template <bool WEIGHTED>
__global__ void __launch_bounds__(RT)
k_reduce_heavy(const int64_t *__restrict__ offsets, const int32_t *__restrict__ heavy_rows,
               const int64_t *__restrict__ chunk_first, const int32_t *__restrict__ chunk_heavy, int64_t n_chunks,
               int64_t chunk_arcs, const uint8_t *__restrict__ cls, const float *__restrict__ w, float qscale,
               int32_t k, unsigned long long *__restrict__ acc)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int kk = k;
    const int pk = (kk + 3) & ~3;
    const int vecw = pk * Acc<WEIGHTED>::planes;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *v = reinterpret_cast<uint32_t *>(smem_raw) + wid * vecw;
    for (int i = lane; i < vecw; i += 32) v[i] = 0u;
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * RW + wid, GW = (int64_t)gridDim.x * RW;
    for (int64_t q = gw; q < n_chunks; q += GW) {
        const int32_t h = chunk_heavy[q];
        const int64_t e1 = min(chunk_first[q] + chunk_arcs, offsets[(int64_t)heavy_rows[h] + 1]);
        for (int64_t e0 = chunk_first[q]; e0 < e1; e0 += 32 * UNR) {
            uint32_t cc[UNR];
            float ww[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                const int64_t e = e0 + lane + 32 * u;
                cc[u] = e < e1 ? __ldcs(cls + e) : 0u;
                ww[u] = (WEIGHTED && e < e1) ? __ldcs(w + e) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < UNR; u++)
                if (cc[u] != 0u && cc[u] <= (uint32_t)kk) acc_add<WEIGHTED>(v, pk, cc[u], ww[u], qscale);
        }
        __syncwarp();
        for (int c = lane; c < kk; c += 32) {
            const long long s = acc_take<WEIGHTED>(v, pk, c);
            if (s) atomicAdd(&acc[(int64_t)h * kk + c], (unsigned long long)s);
        }
        __syncwarp();
    }
}

template <bool WEIGHTED>
__global__ void k_heavy_finalize(const int32_t *__restrict__ heavy_rows, int64_t n_heavy, int32_t k,
                                 unsigned long long *__restrict__ acc, const double *__restrict__ inv, double dscale,
                                 float *__restrict__ z)
{
    const int64_t total = n_heavy * k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = i / k;
        const int c = (int)(i - h * k);
        const unsigned long long s = acc[i];
        acc[i] = 0ull;
        const float f = WEIGHTED ? (float)(long long)s : (float)s;
        z[(int64_t)heavy_rows[h] * k + c] = f * (float)(inv[c + 1] * dscale);
    }
}

__global__ void k_mark_heavy(const int64_t *__restrict__ offsets, int64_t n, int64_t thr, int32_t *__restrict__ rows,
                             unsigned long long *__restrict__ count)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        if (offsets[r + 1] - offsets[r] > thr) rows[atomicAdd(count, 1ull)] = (int32_t)r;
}

int grid_for(int64_t items, int per_block, int waves)
{
    int64_t want = (items + per_block - 1) / per_block;
    int64_t cap = (int64_t)gee::sm_count() * waves;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

size_t rows_smem(int32_t k, bool weighted)
{
    return ((size_t)(k + 4) & ~(size_t)3) * sizeof(float) +
           (size_t)RW * (((size_t)k + 3) & ~(size_t)3) * (weighted ? 2 : 1) * sizeof(uint32_t);
}

}  // namespace

extern "C" {

int gee_reduce_heavy_plan(const int64_t *offsets, int64_t n, int64_t heavy_arcs, int32_t *heavy_rows,
                          int64_t *n_heavy, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && heavy_arcs >= 1, GEE_ERR_INVALID, "n must be >= 0 and heavy_arcs >= 1");
    GEE_REQUIRE(n_heavy && (n == 0 || (offsets && heavy_rows)), GEE_ERR_INVALID, "NULL array argument");
    *n_heavy = 0;
    if (n == 0) return GEE_OK;
    cudaStream_t st = gee::as_stream(stream);
    unsigned long long *cnt = nullptr, h = 0;
    GEE_CUDA(cudaMallocAsync((void **)&cnt, sizeof(unsigned long long), st));
    GEE_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    k_mark_heavy<<<grid_for(n, 256, 16), 256, 0, st>>>(offsets, n, heavy_arcs, heavy_rows, cnt);
    int rc = gee::check_launch("k_mark_heavy");
    cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(cnt, st);
    GEE_CUDA(cudaStreamSynchronize(st));
    *n_heavy = (int64_t)h;
    return rc;
}

int gee_reduce_rows(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                    const double *inv, int32_t k, int64_t heavy_arcs, const int32_t *heavy_rows, int64_t n_heavy,
                    const int64_t *chunk_first, const int32_t *chunk_heavy, int64_t n_chunks, void *heavy_acc, float *z,
                    void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs 1 <= k <= 255 (got %d)", k);
    GEE_REQUIRE(n >= 0 && n_heavy >= 0 && n_chunks >= 0 && heavy_arcs >= 1, GEE_ERR_INVALID, "bad sizes");
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && z && inv && (cls || n_chunks == 0), GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(n_heavy == 0 || (heavy_rows && chunk_first && chunk_heavy && heavy_acc), GEE_ERR_INVALID,
                "heavy rows need their chunk list and accumulator");
    cudaStream_t st = gee::as_stream(stream);
    const bool weighted = w != nullptr;
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = weighted ? ldexp(1.0, -scale_exp) : 1.0;
    const size_t sh = rows_smem(k, weighted);
    const int64_t warps = n;  // one warp per row, strided
    const int grid = grid_for(warps * 32, RT, 8);
    auto *acc = static_cast<unsigned long long *>(heavy_acc);
    if (weighted) {
        GEE_CUDA(cudaFuncSetAttribute(k_reduce_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        k_reduce_rows<true><<<grid, RT, sh, st>>>(offsets, n, cls, w, qscale, dscale, inv, k, heavy_arcs, z);
    } else {
        GEE_CUDA(cudaFuncSetAttribute(k_reduce_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        k_reduce_rows<false><<<grid, RT, sh, st>>>(offsets, n, cls, w, qscale, dscale, inv, k, heavy_arcs, z);
    }
    int rc = gee::check_launch("k_reduce_rows");
    if (rc || n_heavy == 0) return rc;
    const size_t shh = (size_t)RW * (((size_t)k + 3) & ~(size_t)3) * (weighted ? 2 : 1) * sizeof(uint32_t);
    const int hgrid = grid_for(n_chunks * 32, RT, 8);
    if (weighted)
        k_reduce_heavy<true><<<hgrid, RT, shh, st>>>(offsets, heavy_rows, chunk_first, chunk_heavy, n_chunks, heavy_arcs,
                                                     cls, w, qscale, k, acc);
    else
        k_reduce_heavy<false><<<hgrid, RT, shh, st>>>(offsets, heavy_rows, chunk_first, chunk_heavy, n_chunks,
                                                      heavy_arcs, cls, w, qscale, k, acc);
    if ((rc = gee::check_launch("k_reduce_heavy"))) return rc;
    const int fgrid = grid_for(n_heavy * k, 256, 4);
    if (weighted)
        k_heavy_finalize<true><<<fgrid, 256, 0, st>>>(heavy_rows, n_heavy, k, acc, inv, dscale, z);
    else
        k_heavy_finalize<false><<<fgrid, 256, 0, st>>>(heavy_rows, n_heavy, k, acc, inv, dscale, z);
    return gee::check_launch("k_heavy_finalize");
}

int gee_reduce_bins(const int64_t *offsets, int64_t n, int64_t small_arcs, int64_t heavy_arcs, int32_t *small_rows,
                    int32_t *medium_rows, int64_t *n_small, int64_t *n_medium, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && small_arcs >= 0 && heavy_arcs >= small_arcs, GEE_ERR_INVALID, "bad bin sizes");
    GEE_REQUIRE(n_small && n_medium, GEE_ERR_INVALID, "NULL count argument");
    *n_small = *n_medium = 0;
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && small_rows && medium_rows, GEE_ERR_INVALID, "NULL array argument");
    cudaStream_t st = gee::as_stream(stream);
    unsigned long long *cnt = nullptr, h[2] = {0, 0};
    GEE_CUDA(cudaMallocAsync((void **)&cnt, 2 * sizeof(unsigned long long), st));
    GEE_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), st));
    k_bin_rows<<<grid_for(n, 256, 16), 256, 0, st>>>(offsets, n, small_arcs, heavy_arcs, small_rows, medium_rows, cnt);
    int rc = gee::check_launch("k_bin_rows");
    cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(cnt, st);
    GEE_CUDA(cudaStreamSynchronize(st));
    *n_small = (int64_t)h[0];
    *n_medium = (int64_t)h[1];
    return rc;
}

int gee_reduce_lists(const int64_t *offsets, const int32_t *small_rows, int64_t n_small, const int32_t *medium_rows,
                     int64_t n_medium, const uint8_t *cls, const float *w, int32_t scale_exp, const double *inv,
                     int32_t k, int64_t heavy_arcs, const int32_t *heavy_rows, int64_t n_heavy,
                     const int64_t *chunk_first, const int32_t *chunk_heavy, int64_t n_chunks, void *heavy_acc, float *z,
                     void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs 1 <= k <= 255 (got %d)", k);
    GEE_REQUIRE(n_small >= 0 && n_medium >= 0 && n_heavy >= 0 && n_chunks >= 0, GEE_ERR_INVALID, "bad sizes");
    GEE_REQUIRE(offsets && z && inv, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(n_heavy == 0 || (heavy_rows && chunk_first && chunk_heavy && heavy_acc), GEE_ERR_INVALID,
                "heavy rows need their chunk list and accumulator");
    cudaStream_t st = gee::as_stream(stream);
    const bool weighted = w != nullptr;
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = weighted ? ldexp(1.0, -scale_exp) : 1.0;
    const size_t vec = (((size_t)k + 3) & ~(size_t)3) * (weighted ? 2 : 1) * sizeof(uint32_t);
    const size_t scb = ((size_t)(k + 4) & ~(size_t)3) * sizeof(float);
    int rc = GEE_OK;
    if (n_small > 0) {
        const size_t sh = scb + (size_t)RW * 4 * vec;
        const int grid = grid_for((n_small + 3) / 4 * 32, RT, 8);
        if (weighted) {
            GEE_CUDA(cudaFuncSetAttribute(k_reduce_list<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
            k_reduce_list<true, 8><<<grid, RT, sh, st>>>(offsets, small_rows, n_small, cls, w, qscale, dscale, inv, k, z);
        } else {
            GEE_CUDA(cudaFuncSetAttribute(k_reduce_list<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
            k_reduce_list<false, 8><<<grid, RT, sh, st>>>(offsets, small_rows, n_small, cls, w, qscale, dscale, inv, k, z);
        }
        if ((rc = gee::check_launch("k_reduce_list<8>"))) return rc;
    }
    if (n_medium > 0) {
        const size_t sh = scb + (size_t)RW * vec;
        const int grid = grid_for(n_medium * 32, RT, 8);
        if (weighted) {
            GEE_CUDA(cudaFuncSetAttribute(k_reduce_list<true, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
            k_reduce_list<true, 32><<<grid, RT, sh, st>>>(offsets, medium_rows, n_medium, cls, w, qscale, dscale, inv, k, z);
        } else {
            GEE_CUDA(cudaFuncSetAttribute(k_reduce_list<false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
            k_reduce_list<false, 32><<<grid, RT, sh, st>>>(offsets, medium_rows, n_medium, cls, w, qscale, dscale, inv, k, z);
        }
        if ((rc = gee::check_launch("k_reduce_list<32>"))) return rc;
    }
    if (n_heavy == 0) return GEE_OK;
    const size_t shh = (size_t)RW * vec;
    auto *acc = static_cast<unsigned long long *>(heavy_acc);
    const int hgrid = grid_for(n_chunks * 32, RT, 8);
    if (weighted)
        k_reduce_heavy<true><<<hgrid, RT, shh, st>>>(offsets, heavy_rows, chunk_first, chunk_heavy, n_chunks, heavy_arcs,
                                                     cls, w, qscale, k, acc);
    else
        k_reduce_heavy<false><<<hgrid, RT, shh, st>>>(offsets, heavy_rows, chunk_first, chunk_heavy, n_chunks,
                                                      heavy_arcs, cls, w, qscale, k, acc);
    if ((rc = gee::check_launch("k_reduce_heavy"))) return rc;
    const int fgrid = grid_for(n_heavy * k, 256, 4);
    if (weighted)
        k_heavy_finalize<true><<<fgrid, 256, 0, st>>>(heavy_rows, n_heavy, k, acc, inv, dscale, z);
    else
        k_heavy_finalize<false><<<fgrid, 256, 0, st>>>(heavy_rows, n_heavy, k, acc, inv, dscale, z);
    return gee::check_launch("k_heavy_finalize");
}

}  // extern "C"
