// Wide-embedding pull (K > 255): label gather fused with a per-row class
// window, one warp per light row, one CTA per heavy row.
//
// The reference's arc rule (_kernels.py:192-199, SOURCE_ONLY storage) over
// the symmetric CSR:   Z[x, c] = inv[c] * sum_{e in row x, Y[target e] = c} w[e].
// For K = 1000 (BASELINE C5) a Z row is 4 KB and most of it is zero, so the
// kernel is bound by writing Z once (16 GB of C5's 18 GB compulsory bytes):
//   * a warp owns a row: lanes stream its targets (coalesced int32), look up
//     u16/int32 labels through L1/L2 (the table is small and stays in L2) and
//     add the arc into a warp-private K-bin window in shared memory with
//     fire-and-forget shared atomics (u32 counts; weighted arcs as the
//     signed split fixed point of the block reducer: q = rint(w 2^e) =
//     A 2^21 + B, two u32 planes, rows <= 2048 arcs so neither plane
//     overflows, the A plane decoded with sign extension);
//   * the warp then writes the WHOLE Z row with 16-byte streaming stores
//     (zeros included: no separate zero fill), reading each 4-class group of
//     the window once and clearing only the groups that were touched.
// Rows longer than 2048 arcs are skipped and written by k_wide_heavy (one
// CTA per row, u64 window).  Values are (float)sum * (float)(inv[c] 2^-e),
// the formula every pull reducer uses, so all pull paths agree bit for bit.
#include <cstdlib>

#include "gee_common.cuh"

namespace {

constexpr int WT = 256;        // threads per CTA (8 warps)
constexpr int WW = WT / 32;
constexpr int SPLIT = 21;      // == BLOCK_SPLIT of gee_reduce.cu (gee_block_scale_exp bounds |q| < 2^41)
constexpr int LIGHT_MAX = 2048;
constexpr int UNR = 8;         // 32-arc rounds in flight per warp (256 arcs)
#ifndef GEE_WIDE_MINB
#define GEE_WIDE_MINB 5
#endif
#ifndef GEE_WIDE_ST
#define GEE_WIDE_ST 0  // Z row stores: 0 streaming (.cs), 1 default write-back
#endif
#ifndef GEE_WIDE_CONTIG
#define GEE_WIDE_CONTIG 0
#endif

__device__ __forceinline__ void st_z4(float4 *p, float4 v)
{
    if (GEE_WIDE_ST == 0) __stcs(p, v);
    else *p = v;
}

// Signed split decode (see gee_reduce.cu): the high plane holds the two's
// complement of a sum in [-2^31, 2^31).
__device__ __forceinline__ long long plane_sum(uint32_t lo, uint32_t hi)
{
    return (long long)(int32_t)hi * (1ll << SPLIT) + (long long)lo;
}

template <typename LT>
__device__ __forceinline__ uint32_t ld_lab(const LT *t, uint32_t slot)
{
    return (uint32_t)__ldg(t + slot);
}

// Labels of a loaded segment (predicated gathers; 0 for lanes past the row).
template <typename LT>
__device__ __forceinline__ void wide_labels(const int32_t (&t)[UNR], const LT *__restrict__ table, uint32_t (&lab)[UNR])
{
#pragma unroll
    for (int u = 0; u < UNR; u++) lab[u] = t[u] >= 0 ? ld_lab(table, (uint32_t)t[u]) : 0u;
}

// Add a segment's arcs (labels + weights) into the window.
template <bool WEIGHTED>
__device__ __forceinline__ void wide_add(const uint32_t (&lab)[UNR], const float (&wt)[UNR], uint32_t *win,
                                         int32_t kp, float qscale)
{
#pragma unroll
    for (int u = 0; u < UNR; u++) {
        if (lab[u] == 0u) continue;
        GEE_DCHECK(lab[u] - 1u < (uint32_t)kp);
        uint32_t *p = win + (lab[u] - 1);
        if (WEIGHTED) {
            const unsigned long long q = (unsigned long long)__float2ll_rn(wt[u] * qscale);
            atomicAdd(p, (uint32_t)q & ((1u << SPLIT) - 1u));
            atomicAdd(p + kp, (uint32_t)(q >> SPLIT));
        } else {
            atomicAdd(p, 1u);
        }
    }
}

template <bool WEIGHTED>
__device__ __forceinline__ void wide_load(const int32_t *__restrict__ targets, const float *__restrict__ w, int64_t e0,
                                          int64_t e1, int lane, int32_t (&t)[UNR], float (&wt)[UNR])
{
#pragma unroll
    for (int u = 0; u < UNR; u++) {
        const int64_t e = e0 + 32 * u + lane;
        t[u] = e < e1 ? __ldcs(targets + e) : -1;
        if (WEIGHTED) wt[u] = e < e1 ? __ldcs(w + e) : 0.f;
    }
}

// window layout per warp: planes x kp u32 (kp = k rounded up to 4).
// Software pipeline per warp (rows r, r+GW, r+2GW, ...): while row i's Z row
// is written out, row i+1's labels and row i+2's targets (+ weights) and
// offsets are in flight, so the write-out hides both dependent latencies.
// Only a row's first 32 * UNR arcs are pipelined; longer rows finish their
// remaining segments in place.
template <typename LT, bool WEIGHTED, bool VEC>
__global__ void __launch_bounds__(WT, WEIGHTED ? 3 : GEE_WIDE_MINB)
k_wide_rows(const int64_t *__restrict__ offsets, int64_t n, const int32_t *__restrict__ targets,
            const float *__restrict__ w, const LT *__restrict__ table, float qscale, double dscale,
            const double *__restrict__ inv, int32_t k, int32_t kp, float *__restrict__ z)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *sc = reinterpret_cast<float *>(smem_raw);  // sc[c] = inv[c+1] * dscale, c < kp
    constexpr int planes = WEIGHTED ? 2 : 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *win = reinterpret_cast<uint32_t *>(sc + kp) + (size_t)wid * planes * kp;
    for (int c = threadIdx.x; c < kp; c += WT) sc[c] = c < k ? (float)(inv[c + 1] * dscale) : 0.f;
    for (int i = lane; i < planes * kp; i += 32) win[i] = 0u;
    __syncthreads();
#if GEE_WIDE_CONTIG
    // each CTA owns a contiguous run of rows (its warps interleave in it), so
    // the SM's Z rows go out as one sequential stream
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r_beg = (int64_t)blockIdx.x * per;
    const int64_t r_end = min(n, r_beg + per);
    const int64_t GW = WW;
    int64_t r = r_beg + wid;
    n = r_end;  // the pipeline below stops at the end of the CTA's run
#else
    const int64_t GW = (int64_t)gridDim.x * WW;
    int64_t r = (int64_t)blockIdx.x * WW + wid;
#endif
    if (r >= n) return;
    auto seg_end = [](int64_t b0, int64_t b1) { return b1 - b0 <= LIGHT_MAX ? (b1 < b0 + 32 * UNR ? b1 : b0 + 32 * UNR) : b0; };
    // stage 0 (row r): labels in flight; stage 1 (row r+GW): targets in flight
    int64_t a0 = offsets[r], a1 = offsets[r + 1];
    int32_t t[UNR];
    float wt[UNR], wt1[UNR];
    uint32_t lab[UNR];
    wide_load<WEIGHTED>(targets, w, a0, seg_end(a0, a1), lane, t, wt);
    wide_labels<LT>(t, table, lab);
    int64_t b0 = 0, b1 = 0;
    if (r + GW < n) {
        b0 = offsets[r + GW], b1 = offsets[r + GW + 1];
        wide_load<WEIGHTED>(targets, w, b0, seg_end(b0, b1), lane, t, wt1);
    }
    while (true) {
        const bool light = a1 - a0 <= LIGHT_MAX;  // heavy rows: k_wide_heavy writes them
        if (light) {
            wide_add<WEIGHTED>(lab, wt, win, kp, qscale);
            for (int64_t e0 = a0 + 32 * UNR; e0 < a1; e0 += 32 * UNR) {  // rows longer than one segment
                int32_t tx[UNR];
                uint32_t lx[UNR];
                wide_load<WEIGHTED>(targets, w, e0, a1, lane, tx, wt);
                wide_labels<LT>(tx, table, lx);
                wide_add<WEIGHTED>(lx, wt, win, kp, qscale);
            }
        }
        const int64_t rn = r + GW;
        // advance the pipeline: labels of rn, targets (+ offsets) of rn + GW
        int64_t c0 = 0, c1 = 0;
        if (rn < n) {
            wide_labels<LT>(t, table, lab);
#pragma unroll
            for (int u = 0; u < UNR; u++) wt[u] = wt1[u];
            const int64_t rnn = rn + GW;
            if (rnn < n) {
                c0 = offsets[rnn], c1 = offsets[rnn + 1];
                wide_load<WEIGHTED>(targets, w, c0, seg_end(c0, c1), lane, t, wt1);
            }
        }
        if (light) {
            __syncwarp();
            float *zr = z + r * (int64_t)k;
            if (VEC) {  // k % 4 == 0 and z 16-byte aligned: whole row in 16-byte streaming stores
                // (a TMA bulk store of the converted row measured slower: 4.99 vs 4.58 ms on C5)
                const int groups = kp >> 2;
                uint4 *w4 = reinterpret_cast<uint4 *>(win);
                float4 *z4 = reinterpret_cast<float4 *>(zr);
#pragma unroll 4
                for (int g = lane; g < groups; g += 32) {
                    const uint4 lo = w4[g];
                    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                    uint4 hi = make_uint4(0u, 0u, 0u, 0u);
                    if (WEIGHTED) hi = w4[g + (kp >> 2)];
                    if ((lo.x | lo.y | lo.z | lo.w | hi.x | hi.y | hi.z | hi.w) != 0u) {
                        const float4 s4 = reinterpret_cast<const float4 *>(sc)[g];
                        if (WEIGHTED) {
                            o.x = (float)plane_sum(lo.x, hi.x) * s4.x;
                            o.y = (float)plane_sum(lo.y, hi.y) * s4.y;
                            o.z = (float)plane_sum(lo.z, hi.z) * s4.z;
                            o.w = (float)plane_sum(lo.w, hi.w) * s4.w;
                            w4[g + (kp >> 2)] = make_uint4(0u, 0u, 0u, 0u);
                        } else {
                            o.x = (float)lo.x * s4.x, o.y = (float)lo.y * s4.y;
                            o.z = (float)lo.z * s4.z, o.w = (float)lo.w * s4.w;
                        }
                        w4[g] = make_uint4(0u, 0u, 0u, 0u);
                    }
                    st_z4(z4 + g, o);
                }
            } else {
                for (int c = lane; c < k; c += 32) {
                    const uint32_t lo = win[c];
                    float o = 0.f;
                    if (WEIGHTED) {
                        const uint32_t hi = win[c + kp];
                        if (lo | hi) {
                            o = (float)plane_sum(lo, hi) * sc[c];
                            win[c] = 0u, win[c + kp] = 0u;
                        }
                    } else if (lo) {
                        o = (float)lo * sc[c];
                        win[c] = 0u;
                    }
                    __stcs(zr + c, o);
                }
            }
            __syncwarp();
        }
        if (rn >= n) break;
        r = rn, a0 = b0, a1 = b1, b0 = c0, b1 = c1;
    }
}

// Heavy rows (> LIGHT_MAX arcs): one CTA per row, u64 window, any length.
template <typename LT, bool WEIGHTED>
__global__ void __launch_bounds__(1024)
k_wide_heavy(const int64_t *__restrict__ offsets, const int32_t *__restrict__ heavy_rows, int64_t n_heavy,
             const int32_t *__restrict__ targets, const float *__restrict__ w, const LT *__restrict__ table,
             float qscale, double dscale, const double *__restrict__ inv, int32_t k, float *__restrict__ z)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long *win = reinterpret_cast<unsigned long long *>(smem_raw);
    float *sc = reinterpret_cast<float *>(win + k);
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        win[c] = 0ull;
        sc[c] = (float)(inv[c + 1] * dscale);
    }
    __syncthreads();
    for (int64_t h = blockIdx.x; h < n_heavy; h += gridDim.x) {
        const int64_t r = heavy_rows[h];
        const int64_t a0 = offsets[r], a1 = offsets[r + 1];
        for (int64_t e = a0 + threadIdx.x; e < a1; e += blockDim.x) {
            const uint32_t lab = ld_lab(table, (uint32_t)__ldcs(targets + e));
            if (lab == 0u) continue;
            if (WEIGHTED)
                atomicAdd(win + (lab - 1), (unsigned long long)__float2ll_rn(__ldcs(w + e) * qscale));
            else
                atomicAdd(win + (lab - 1), 1ull);
        }
        __syncthreads();
        float *zr = z + r * (int64_t)k;
        for (int c = threadIdx.x; c < k; c += blockDim.x) {
            const unsigned long long s = win[c];
            win[c] = 0ull;
            zr[c] = (WEIGHTED ? (float)(long long)s : (float)s) * sc[c];
        }
        __syncthreads();
    }
}

template <typename LT>
int launch_wide(const int64_t *offsets, int64_t n, const int32_t *targets, const float *w, const void *table,
                int32_t scale_exp, const double *inv, int32_t k, const int32_t *heavy_rows, int64_t n_heavy, float *z,
                cudaStream_t st)
{
    const bool weighted = w != nullptr;
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = weighted ? ldexp(1.0, -scale_exp) : 1.0;
    const int32_t kp = (k + 3) & ~3;
    const LT *tab = static_cast<const LT *>(table);
    if (n > 0) {
        const size_t smem = (size_t)kp * 4 + (size_t)WW * (weighted ? 2 : 1) * kp * 4;
        const bool vec = (k % 4 == 0) && gee::aligned16(z);
        auto kern = weighted ? (vec ? k_wide_rows<LT, true, true> : k_wide_rows<LT, true, false>)
                             : (vec ? k_wide_rows<LT, false, true> : k_wide_rows<LT, false, false>);
        GEE_REQUIRE(smem <= (size_t)227 * 1024, GEE_ERR_INVALID, "k = %d too wide for the shared-memory window", k);
        GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        GEE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WT, smem));
        if (per_sm < 1) per_sm = 1;
        int64_t want = (n + WW - 1) / WW;
        int64_t grid = (int64_t)gee::sm_count() * per_sm;
        if (grid > want) grid = want;
        kern<<<(int)grid, WT, smem, st>>>(offsets, n, targets, w, tab, qscale, dscale, inv, k, kp, z);
        if (int rc = gee::check_launch("k_wide_rows")) return rc;
    }
    if (n_heavy > 0) {
        const size_t smem = (size_t)k * 8 + (size_t)k * 4;
        GEE_REQUIRE(smem <= (size_t)227 * 1024, GEE_ERR_INVALID, "k = %d too wide for the heavy-row window", k);
        auto kern = weighted ? k_wide_heavy<LT, true> : k_wide_heavy<LT, false>;
        GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int64_t grid = n_heavy < 2LL * gee::sm_count() ? n_heavy : 2LL * gee::sm_count();
        kern<<<(int)grid, 1024, smem, st>>>(offsets, heavy_rows, n_heavy, targets, w, tab, qscale, dscale, inv, k, z);
        return gee::check_launch("k_wide_heavy");
    }
    return GEE_OK;
}

}  // namespace

extern "C" int gee_reduce_wide(const int64_t *offsets, int64_t n, const int32_t *targets, const float *w,
                               const void *table, int32_t k, int32_t scale_exp, const double *inv,
                               const int32_t *heavy_rows, int64_t n_heavy, float *z, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive");
    GEE_REQUIRE(n >= 0 && n_heavy >= 0, GEE_ERR_INVALID, "n and n_heavy must be nonnegative");
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && table && inv && z, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(n_heavy == 0 || heavy_rows, GEE_ERR_INVALID, "heavy_rows must not be NULL");
    cudaStream_t st = gee::as_stream(stream);
    switch (gee_label_bytes(k)) {
    case 1: return launch_wide<uint8_t>(offsets, n, targets, w, table, scale_exp, inv, k, heavy_rows, n_heavy, z, st);
    case 2: return launch_wide<uint16_t>(offsets, n, targets, w, table, scale_exp, inv, k, heavy_rows, n_heavy, z, st);
    default: return launch_wide<int32_t>(offsets, n, targets, w, table, scale_exp, inv, k, heavy_rows, n_heavy, z, st);
    }
}
