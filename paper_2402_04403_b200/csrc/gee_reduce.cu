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
#include <algorithm>
#include <cstdlib>

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

// Block variant: one warp per block of 32 consecutive rows.  Lane i loads
// offsets[r0+i] (one coalesced load per block).  The block's arcs stream in
// rounds of 32 x 8 contiguous arcs (one 8-byte class load and two 16-byte
// weight loads per lane; the next round, and the next block's first round,
// in flight).  Arc -> row mapping is branch-free: the lanes whose rows start
// inside the round set bits in a 256-bit start mask (shared memory, three
// rotating buffers so one __syncwarp per round suffices); a lane's arcs then
// take the owner rank "rows started at or before the round" + popcounts.
// Nonempty rows get compact slots in a warp-private window.  The block's Z
// range is zero-filled with 16-byte stores when it holds empty rows, then the
// nonempty rows are written from their slots in one flat loop; heavy rows are
// left to the chunked path (k_heavy_finalize runs after).  Blocks with more
// than `nslots` nonempty rows take several passes.
#ifndef BLOCKS_MINB
#define BLOCKS_MINB 3  // CTAs per SM the block reducer is register-capped for
#endif
constexpr int BU = 8;            // contiguous arcs per lane per round
constexpr int BLOCK_SPLIT = 21;  // weighted: low plane takes q's low 21 bits
constexpr int64_t BLOCK_ROW_MAX = 2048;  // longest row the block kernel takes (longer: heavy path)
constexpr int BROUND = 32 * BU;  // arcs per warp round
constexpr int BMETA = 96;        // per-warp ints: 3 x 8 mask words, 33 slot offsets, 32 rows (+pad)

template <bool WEIGHTED>
__device__ __forceinline__ void block_round(const uint8_t *__restrict__ cls, const float *__restrict__ w, int64_t e,
                                            int64_t arcs, bool vec, uint2 &c, float (&wt)[BU])
{
    if (vec && e + BU <= arcs) {
        c = __ldcs(reinterpret_cast<const uint2 *>(cls + e));
        if (WEIGHTED) {
            const float4 a = __ldcs(reinterpret_cast<const float4 *>(w + e));
            const float4 b = __ldcs(reinterpret_cast<const float4 *>(w + e + 4));
            wt[0] = a.x, wt[1] = a.y, wt[2] = a.z, wt[3] = a.w;
            wt[4] = b.x, wt[5] = b.y, wt[6] = b.z, wt[7] = b.w;
        }
    } else {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int u = 0; u < BU; u++) {
            const bool ok = e + u < arcs;
            const uint32_t cv = ok ? (uint32_t)cls[e + u] : 0u;
            if (u < 4)
                lo |= cv << (8 * u);
            else
                hi |= cv << (8 * (u - 4));
            if (WEIGHTED) wt[u] = ok ? w[e + u] : 0.f;
        }
        c = make_uint2(lo, hi);
    }
}

// Window of one warp: per plane [nslots x vector | 32 trash words]; a slot's
// vector is [3 pad | unused | bin 1 .. bin k | pad] so that bin pairs
// (2j+1, 2j+2) are 8-byte aligned for the write-out.  Masked arcs (class 0,
// past the block, rows outside this pass) add into the lane's own trash
// word: no branch, and no two lanes on one address.
__host__ __device__ constexpr int block_vec_words(int k) { return 4 + ((k + 3) & ~3); }

// One round of arcs already in registers: start mask -> owner ranks -> slots.
template <bool WEIGHTED>
__device__ __forceinline__ void block_round_acc(uint32_t *__restrict__ vw, const int32_t *__restrict__ s_soff,
                                                uint32_t *__restrict__ s_mask, int &rot, int lane, bool owner,
                                                int32_t ol, int32_t lr, int32_t lend, int hoff, int trash,
                                                float qscale, const uint2 &ca, const float (&wa)[BU])
{
    const unsigned startm = __ballot_sync(0xffffffffu, owner && ol <= lr);
    uint32_t *mk = s_mask + 8 * rot;
    const int32_t pos = ol - lr;
    if (owner && pos > 0 && pos < BROUND) atomicOr(mk + (pos >> 5), 1u << (pos & 31));
    __syncwarp();
    const uint32_t mb = (mk[lane >> 2] >> (8 * (lane & 3))) & 0xffu;
    if (lane < 8) s_mask[8 * (rot == 0 ? 2 : rot - 1) + lane] = 0u;  // buffer read last round
    rot = rot == 2 ? 0 : rot + 1;
    const int pc = __popc(mb);
    int incl = pc;
#pragma unroll
    for (int st = 1; st < 32; st <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, st);
        incl += lane >= st ? t : 0;
    }
    int r = __popc(startm) + incl - pc;  // owner rank + 1 before this lane's first arc
    // arcs past the block end get class 0 (masked), once per round
    const int nvalid = lend - (lr + lane * BU);
    uint2 cm = ca;
    if (nvalid < BU) {
        const uint32_t nv = nvalid <= 0 ? 0u : (uint32_t)nvalid;
        cm.x &= nv >= 4 ? 0xffffffffu : ((1u << (8 * nv)) - 1u);
        cm.y &= nv >= 8 ? 0xffffffffu : (nv <= 4 ? 0u : ((1u << (8 * (nv - 4))) - 1u));
    }
#pragma unroll
    for (int u = 0; u < BU; u++) {
        r += (mb >> u) & 1u;
        const uint32_t c = __byte_perm(u < 4 ? cm.x : cm.y, 0u, 0x4440 + (u & 3));
        const int so = s_soff[r];
        const int idx = (c != 0u && so >= 0) ? so + (int)c : trash;
        if (WEIGHTED) {
            // carry-free split q = A * 2^21 + B: both plane sums stay below
            // 2^32 (rows <= BLOCK_ROW_MAX arcs, q < 2^42), so neither add
            // needs its return value
            const unsigned long long q = (unsigned long long)__float2ll_rn(wa[u] * qscale);
            atomicAdd(vw + idx, (uint32_t)q & ((1u << BLOCK_SPLIT) - 1u));
            atomicAdd(vw + hoff + idx, (uint32_t)(q >> BLOCK_SPLIT));
        } else {
            atomicAdd(vw + idx, 1u);
        }
    }
}

// One round over PADDED rows (every row's arc run is a multiple of BU, so
// each lane's 8 arcs belong to one row): the lane's owner rank is the count
// of rows started before the round plus the row starts at lane chunks <= its
// own -- one ballot, one OR-reduction, two popcounts, no shared masks.
template <bool WEIGHTED>
__device__ __forceinline__ void block_round_pad(uint32_t *__restrict__ vw, const int32_t *__restrict__ s_soff, int lane,
                                                bool owner, int32_t ol, int32_t lr, int32_t lend, int hoff, int trash,
                                                float qscale, const uint2 &ca, const float (&wa)[BU])
{
    const unsigned startm = __ballot_sync(0xffffffffu, owner && ol <= lr);
    const int32_t pos = ol - lr;
    const unsigned m = __reduce_or_sync(0xffffffffu, (owner && pos > 0 && pos < BROUND) ? 1u << (pos >> 3) : 0u);
    const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    const int r = __popc(startm) + __popc(m & upto);  // owner rank + 1 (0: before the block)
    const int so = s_soff[r];
    const bool ok = so >= 0 && lr + lane * BU < lend;
#pragma unroll
    for (int u = 0; u < BU; u++) {
        const uint32_t c = __byte_perm(u < 4 ? ca.x : ca.y, 0u, 0x4440 + (u & 3));
        // masked arcs (pads, unlabeled, other passes, past the block) add into
        // the lane's trash word: branch-free (predicating the atomics off
        // measured slower: 8.20 vs 8.01 ms on C4)
        const int idx = (ok && c != 0u) ? so + (int)c : trash;
        if (WEIGHTED) {
            const unsigned long long q = (unsigned long long)__float2ll_rn(wa[u] * qscale);
            atomicAdd(vw + idx, (uint32_t)q & ((1u << BLOCK_SPLIT) - 1u));
            atomicAdd(vw + hoff + idx, (uint32_t)(q >> BLOCK_SPLIT));
        } else {
            atomicAdd(vw + idx, 1u);
        }
    }
}

// A padded row of exactly one 8-arc chunk (<= 8 real arcs) is reduced by the
// lane that owns it, in registers: equal classes combine exactly (integer
// sums, as in the window), and only the nonzero entries are stored into the
// zero-filled Z row.
template <bool WEIGHTED>
__device__ __forceinline__ void single_row(const uint8_t *__restrict__ cls, const float *__restrict__ w, int64_t a,
                                           float qscale, const float *__restrict__ sc1, float *__restrict__ zr)
{
    const uint2 c8 = *reinterpret_cast<const uint2 *>(cls + a);
    uint32_t c[BU];
    unsigned long long q[BU];
    float wv[BU];
    if (WEIGHTED) {
        const float4 x0 = *reinterpret_cast<const float4 *>(w + a);
        const float4 x1 = *reinterpret_cast<const float4 *>(w + a + 4);
        wv[0] = x0.x, wv[1] = x0.y, wv[2] = x0.z, wv[3] = x0.w;
        wv[4] = x1.x, wv[5] = x1.y, wv[6] = x1.z, wv[7] = x1.w;
    }
#pragma unroll
    for (int u = 0; u < BU; u++) {
        c[u] = __byte_perm(u < 4 ? c8.x : c8.y, 0u, 0x4440 + (u & 3));
        q[u] = WEIGHTED ? (unsigned long long)__float2ll_rn(wv[u] * qscale) : 1ull;
    }
#pragma unroll
    for (int u = 0; u < BU; u++) {
        bool first = c[u] != 0u;
#pragma unroll
        for (int v = 0; v < u; v++) first = first && c[v] != c[u];
        if (first) {
            unsigned long long sum = q[u];
#pragma unroll
            for (int v = u + 1; v < BU; v++) sum += c[v] == c[u] ? q[v] : 0ull;
            zr[c[u] - 1] = (WEIGHTED ? (float)(long long)sum : (float)sum) * sc1[c[u] - 1];
        }
    }
}

template <bool WEIGHTED>
__global__ void __launch_bounds__(RT, BLOCKS_MINB)
k_reduce_blocks(const int64_t *__restrict__ offsets, int64_t n, const uint8_t *__restrict__ cls,
                const float *__restrict__ w, float qscale, double dscale, const double *__restrict__ inv, int32_t k,
                int64_t heavy_arcs, int nslots, bool vec, float *__restrict__ z)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int kk = k;
    const int pkb = block_vec_words(kk);
    const int hoff = nslots * pkb + 32;  // hi plane offset
    const int wwords = hoff * Acc<WEIGHTED>::planes;
    float *sc1 = reinterpret_cast<float *>(smem_raw);  // sc1[c] = inv[c+1] * dscale
    int32_t *meta = reinterpret_cast<int32_t *>(sc1 + pkb);
    uint32_t *vbase = reinterpret_cast<uint32_t *>(meta + RW * BMETA);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *s_mask = reinterpret_cast<uint32_t *>(meta + wid * BMETA);  // 3 x 8 words
    int32_t *s_soff = meta + wid * BMETA + 24;                              // [owner rank + 1] -> slot offset
    int32_t *s_row = s_soff + 36;                                           // [slot] -> row in block
    uint32_t *vw = vbase + wid * wwords;
    for (int c = threadIdx.x; c < pkb; c += RT) sc1[c] = c < kk ? (float)(inv[c + 1] * dscale) : 0.f;
    for (int i = threadIdx.x; i < RW * wwords; i += RT) vbase[i] = 0u;
    for (int i = threadIdx.x; i < RW * BMETA; i += RT) meta[i] = -1;
    __syncthreads();
    if (lane < 24) s_mask[lane] = 0u;
    __syncwarp();
    const int trash = nslots * pkb + lane;
    const unsigned below = (1u << lane) - 1u;
    const int64_t nblocks = (n + 31) / 32;
    const int64_t gw = (int64_t)blockIdx.x * RW + wid, GW = (int64_t)gridDim.x * RW;
    const int64_t arcs = offsets[n];
    const int half = kk >> 1;

    int64_t b = gw;
    int64_t o_lo = 0;
    uint2 ca = make_uint2(0u, 0u), cb = make_uint2(0u, 0u);
    float wa[BU], wb[BU];
#pragma unroll
    for (int u = 0; u < BU; u++) wa[u] = wb[u] = 0.f;
    if (b < nblocks) {
        o_lo = __ldcs(offsets + min(32 * b + lane, n));
        const int64_t b0 = __shfl_sync(0xffffffffu, o_lo, 0) & ~(int64_t)(BU - 1);
        block_round<WEIGHTED>(cls, w, b0 + lane * BU, arcs, vec, ca, wa);
    }
    int rot = 0;  // mask buffer rotation
    for (; b < nblocks; b += GW) {
        const int64_t r0 = 32 * b;
        int64_t o_hi = __shfl_down_sync(0xffffffffu, o_lo, 1);
        if (lane == 31) o_hi = r0 + 32 <= n ? __ldcs(offsets + r0 + 32) : arcs;
        const bool more = b + GW < nblocks;
        const int64_t o_nx = more ? __ldcs(offsets + min(32 * (b + GW) + lane, n)) : 0;
        const bool valid = r0 + lane < n;
        const int64_t d = valid ? o_hi - o_lo : 0;
        const bool heavy = d > heavy_arcs;
        const bool nz = d > 0 && !heavy;
        const unsigned nzm = __ballot_sync(0xffffffffu, nz), hvm = __ballot_sync(0xffffffffu, heavy);
        const unsigned anym = nzm | hvm;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        const int rank = __popc(nzm & below);    // slot order among light nonempty rows
        const int orank = __popc(anym & below);  // owner order among all nonempty rows
        const int nnz = __popc(nzm);
        const int64_t base = __shfl_sync(0xffffffffu, o_lo, 0);
        const int64_t abase = base & ~(int64_t)(BU - 1);
        const int32_t ol = (int32_t)(o_lo - base);  // local start of this lane's row
        const int32_t oh = (int32_t)(o_hi - base);
        const bool owner = (anym >> lane) & 1u;
        const int32_t lend = __shfl_sync(0xffffffffu, oh, 31);
        const int32_t lr0 = (int32_t)(abase - base);  // in [-(BU-1), 0]
        const int rows = (int)min((int64_t)32, n - r0);
        float *zb = z + r0 * (int64_t)kk;
        if (anym != vm) {  // the block holds empty rows: zero-fill its Z range
            const int total = rows * kk;
            const int q4 = total >> 2;
            float4 *z4 = reinterpret_cast<float4 *>(zb);
            for (int q = lane; q < q4; q += 32) z4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int e = 4 * q4 + lane; e < total; e += 32) zb[e] = 0.f;
        }
        for (int p0 = 0; p0 < nnz; p0 += nslots) {
            const bool mine = nz && rank >= p0 && rank < p0 + nslots;
            if (owner) s_soff[orank + 1] = mine ? (rank - p0) * pkb + 3 : -1;
            if (mine) s_row[rank - p0] = lane;
            const int npass = min(nslots, nnz - p0);
            __syncwarp();
            int32_t lr = lr0;
            if (p0 > 0) block_round<WEIGHTED>(cls, w, abase + lane * BU, arcs, vec, ca, wa);
            // rounds, ping-ponging between the (ca, wa) and (cb, wb) buffers
            while (lr < lend) {
                if (hvm) {  // skip a heavy row's arcs wholesale (warp-uniform)
                    const unsigned sm = __ballot_sync(0xffffffffu, owner && ol <= lr);
                    if (sm) {
                        const int jr = 31 - __clz(sm);
                        const int32_t hend = __shfl_sync(0xffffffffu, oh, jr);
                        if (((hvm >> jr) & 1u) && hend >= lr + BROUND) {
                            lr = ((hend - lr0) & ~(BU - 1)) + lr0;
                            block_round<WEIGHTED>(cls, w, abase + (lr - lr0) + lane * BU, arcs, vec, ca, wa);
                            continue;
                        }
                    }
                }
                int32_t l1 = lr + BROUND;
                if (l1 < lend) block_round<WEIGHTED>(cls, w, abase + (l1 - lr0) + lane * BU, arcs, vec, cb, wb);
                block_round_acc<WEIGHTED>(vw, s_soff, s_mask, rot, lane, owner, ol, lr, lend, hoff, trash, qscale,
                                          ca, wa);
                lr = l1;
                if (lr >= lend) break;
                if (hvm) {
                    const unsigned sm = __ballot_sync(0xffffffffu, owner && ol <= lr);
                    if (sm) {
                        const int jr = 31 - __clz(sm);
                        const int32_t hend = __shfl_sync(0xffffffffu, oh, jr);
                        if (((hvm >> jr) & 1u) && hend >= lr + BROUND) {
                            lr = ((hend - lr0) & ~(BU - 1)) + lr0;
                            block_round<WEIGHTED>(cls, w, abase + (lr - lr0) + lane * BU, arcs, vec, ca, wa);
                            continue;
                        }
                    }
                }
                l1 = lr + BROUND;
                if (l1 < lend) block_round<WEIGHTED>(cls, w, abase + (l1 - lr0) + lane * BU, arcs, vec, ca, wa);
                block_round_acc<WEIGHTED>(vw, s_soff, s_mask, rot, lane, owner, ol, lr, lend, hoff, trash, qscale,
                                          cb, wb);
                lr = l1;
            }
            __syncwarp();
            // write this pass's rows from their slots: flat over (row, column pair)
            if ((kk & 1) == 0) {
                const int total = npass * half;
                int sl = lane / half, c2 = lane - sl * half;
                const int dsl = 32 / half, dc2 = 32 - dsl * half;
                for (int q = lane; q < total; q += 32) {
                    uint32_t *vs = vw + sl * pkb + 4 + 2 * c2;
                    const uint2 lo = *reinterpret_cast<uint2 *>(vs);
                    *reinterpret_cast<uint2 *>(vs) = make_uint2(0u, 0u);
                    float s0, s1;
                    if (WEIGHTED) {
                        const uint2 hi = *reinterpret_cast<uint2 *>(vs + hoff);
                        *reinterpret_cast<uint2 *>(vs + hoff) = make_uint2(0u, 0u);
                        s0 = (float)(long long)(((unsigned long long)hi.x << BLOCK_SPLIT) + lo.x);
                        s1 = (float)(long long)(((unsigned long long)hi.y << BLOCK_SPLIT) + lo.y);
                    } else {
                        s0 = (float)lo.x;
                        s1 = (float)lo.y;
                    }
                    const float2 f = *reinterpret_cast<const float2 *>(sc1 + 2 * c2);
                    float2 *zr = reinterpret_cast<float2 *>(zb + s_row[sl] * kk);
                    __stcs(zr + c2, make_float2(s0 * f.x, s1 * f.y));
                    sl += dsl;
                    c2 += dc2;
                    if (c2 >= half) {
                        c2 -= half;
                        sl++;
                    }
                }
            } else {
                const int total = npass * kk;
                int sl = lane / kk, c = lane - sl * kk;
                const int dsl = 32 / kk, dc = 32 - dsl * kk;
                for (int q = lane; q < total; q += 32) {
                    uint32_t *vs = vw + sl * pkb + 4 + c;
                    const uint32_t lo = *vs;
                    *vs = 0u;
                    float s0;
                    if (WEIGHTED) {
                        const uint32_t hi = vs[hoff];
                        vs[hoff] = 0u;
                        s0 = (float)(long long)(((unsigned long long)hi << BLOCK_SPLIT) + lo);
                    } else {
                        s0 = (float)lo;
                    }
                    __stcs(zb + s_row[sl] * kk + c, s0 * sc1[c]);
                    sl += dsl;
                    c += dc;
                    if (c >= kk) {
                        c -= kk;
                        sl++;
                    }
                }
            }
            __syncwarp();
        }
        // next block: its first round in flight while this one finishes
        o_lo = o_nx;
        if (more) {
            const int64_t b0 = __shfl_sync(0xffffffffu, o_nx, 0) & ~(int64_t)(BU - 1);
            block_round<WEIGHTED>(cls, w, b0 + lane * BU, arcs, vec, ca, wa);
        }
    }
}

// ---------------------------------------------------------------------------
// Ring variant of the block reducer.  The same 32-row blocks, slot windows,
// start-mask row mapping and write-out, but the arc stream (classes and
// weights) is fetched by cp.async into a per-warp ring of RING rounds in
// shared memory: RING rounds per warp are in flight without holding
// registers (the register-fed kernel keeps one), and the ring is primed
// across passes and blocks so a block's first rounds arrive while the
// previous block is written out.  Each lane copies and consumes the same 8
// arcs of a round, so cp.async.wait_group alone orders them.
constexpr int RING = 4;
// Single-chunk rows reduced in registers after the block (single_row):
// measured slower on C4 (9.09 vs 8.01 ms: each block then waits on the L2
// reloads of its short rows), so off.
#ifndef BLOCK_SINGLE_ROWS
#define BLOCK_SINGLE_ROWS 0
#endif
constexpr int RING_CLS = BROUND;                        // bytes per round
constexpr int RING_W = BROUND * (int)sizeof(float);     // bytes per round (weighted)

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Per-block view shared by the warp (uniform fields) and per lane.
struct RingBlk {
    int64_t base, bend;      // arc range of the block
    unsigned nzm, hvm, anym, vm;
    int32_t ol, oh;          // this lane's row bounds, block-local
};

__device__ __forceinline__ RingBlk ring_open(int64_t r0, int64_t n, int64_t o_lo, int64_t o_hi31, int64_t heavy_arcs,
                                             int lane)
{
    RingBlk B;
    int64_t o_hi = __shfl_down_sync(0xffffffffu, o_lo, 1);
    if (lane == 31) o_hi = o_hi31;
    const bool valid = r0 + lane < n;
    const int64_t d = valid ? o_hi - o_lo : 0;
    const bool heavy = d > heavy_arcs;
    B.nzm = __ballot_sync(0xffffffffu, d > 0 && !heavy);
    B.hvm = __ballot_sync(0xffffffffu, heavy);
    B.vm = __ballot_sync(0xffffffffu, valid);
    B.anym = B.nzm | B.hvm;
    B.base = __shfl_sync(0xffffffffu, o_lo, 0);
    B.bend = __shfl_sync(0xffffffffu, o_hi, 31);
    B.ol = (int32_t)(o_lo - B.base);
    B.oh = (int32_t)(o_hi - B.base);
    return B;
}

// First round at or after arc e that is not entirely inside a heavy row
// (warp-uniform).
__device__ __forceinline__ int64_t ring_skip(const RingBlk &B, int64_t e, int lane)
{
    if (!B.hvm || e >= B.bend) return e;
    const int32_t lr = (int32_t)(e - B.base);
    const unsigned sm = __ballot_sync(0xffffffffu, ((B.anym >> lane) & 1u) && B.ol <= lr);
    if (!sm) return e;
    const int jr = 31 - __clz(sm);
    const int32_t hend = __shfl_sync(0xffffffffu, B.oh, jr);
    if (((B.hvm >> jr) & 1u) && B.base + hend >= e + BROUND) return (B.base + hend) & ~(int64_t)(BU - 1);
    return e;
}

// SPANS: the two weight copies of a round each move 512 contiguous bytes
// (lane l: arcs [4l, 4l + 4), then [128 + 4l, 128 + 4l + 4)), so every
// 32-byte sector is read once; otherwise lane l copies its own 8 arcs' 32
// bytes as two 16-byte halves, and each copy instruction reads every sector
// of the round half-used (2x the L2->SM bytes; blocks: 8.00 -> 7.81 ms with
// spans, the heavy kernel 2.52 vs 2.61 ms the other way round).
template <bool WEIGHTED, bool SPANS = true>
__device__ __forceinline__ void ring_issue(uint8_t *ring, int slot, int64_t e, int64_t bend, int64_t arcs,
                                           const uint8_t *__restrict__ cls, const float *__restrict__ w, int lane)
{
    if (e < bend) {
        const int64_t a = e + lane * BU;  // classes: lane l copies arcs [8l, 8l + 8)
        uint8_t *rs = ring + slot * (RING_CLS + (WEIGHTED ? RING_W : 0));
        const uint32_t dc = smem_u32(rs + lane * BU);
        const uint32_t dw = smem_u32(rs + RING_CLS + lane * (SPANS ? 16 : 32));
        const int64_t a0 = SPANS ? e + lane * 4 : a, a1 = SPANS ? e + 128 + lane * 4 : a + 4;
        const uint32_t d1 = SPANS ? 512u : 16u;
        if (e + BROUND <= arcs) {  // whole round inside the arrays (warp-uniform)
            cp_async8(dc, cls + a, BU);
            if (WEIGHTED) {
                cp_async16(dw, w + a0, 16u);
                cp_async16(dw + d1, w + a1, 16u);
            }
        } else {
            const int64_t left = arcs - a;
            const uint32_t nc = left <= 0 ? 0u : (left >= BU ? (uint32_t)BU : (uint32_t)left);
            cp_async8(dc, nc ? (const void *)(cls + a) : (const void *)cls, nc);
            if (WEIGHTED) {
                const int64_t l0 = arcs - a0, l1 = arcs - a1;
                const uint32_t n0 = l0 <= 0 ? 0u : (l0 >= 4 ? 16u : (uint32_t)l0 * 4u);
                const uint32_t n1 = l1 <= 0 ? 0u : (l1 >= 4 ? 16u : (uint32_t)l1 * 4u);
                cp_async16(dw, n0 ? (const void *)(w + a0) : (const void *)w, n0);
                cp_async16(dw + d1, n1 ? (const void *)(w + a1) : (const void *)w, n1);
            }
        }
    }
    cp_commit();
}

template <bool WEIGHTED, bool PAD>
__global__ void __launch_bounds__(RT, 2)
k_reduce_blocks_ring(const int64_t *__restrict__ offsets, int64_t n, const uint8_t *__restrict__ cls,
                     const float *__restrict__ w, float qscale, double dscale, const double *__restrict__ inv,
                     int32_t k, int64_t heavy_arcs, int nslots, float *__restrict__ z)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int kk = k;
    const int pkb = block_vec_words(kk);
    const int hoff = nslots * pkb + 32;
    const int wwords = hoff * Acc<WEIGHTED>::planes;
    constexpr int RSLOT = RING_CLS + (WEIGHTED ? RING_W : 0);
    uint8_t *ring_base = smem_raw;  // RW x RING x RSLOT (16-byte aligned)
    float *sc1 = reinterpret_cast<float *>(smem_raw + RW * RING * RSLOT);
    int32_t *meta = reinterpret_cast<int32_t *>(sc1 + pkb);
    uint32_t *vbase = reinterpret_cast<uint32_t *>(meta + RW * BMETA);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *ring = ring_base + wid * RING * RSLOT;
    uint32_t *s_mask = reinterpret_cast<uint32_t *>(meta + wid * BMETA);
    int32_t *s_soff = meta + wid * BMETA + 24;
    int32_t *s_row = s_soff + 36;
    uint32_t *vw = vbase + wid * wwords;
    for (int c = threadIdx.x; c < pkb; c += RT) sc1[c] = c < kk ? (float)(inv[c + 1] * dscale) : 0.f;
    for (int i = threadIdx.x; i < RW * wwords; i += RT) vbase[i] = 0u;
    for (int i = threadIdx.x; i < RW * BMETA; i += RT) meta[i] = -1;
    __syncthreads();
    if (lane < 24) s_mask[lane] = 0u;
    __syncwarp();
    const int trash = nslots * pkb + lane;
    const unsigned below = (1u << lane) - 1u;
    const int64_t nblocks = (n + 31) / 32;
    const int64_t gw = (int64_t)blockIdx.x * RW + wid, GW = (int64_t)gridDim.x * RW;
    const int64_t arcs = offsets[n];
    const int half = kk >> 1;
    int rot = 0;

    int64_t b = gw;
    if (b >= nblocks) return;
    // open the first block and prime its first rounds
    RingBlk B;
    {
        const int64_t r0 = 32 * b;
        const int64_t o_lo = __ldcs(offsets + min(r0 + lane, n));
        const int64_t o_31 = lane == 31 ? __ldcs(offsets + min(r0 + 32, n)) : 0;
        B = ring_open(r0, n, o_lo, o_31, heavy_arcs, lane);
    }
    int64_t ep = ring_skip(B, B.base & ~(int64_t)(BU - 1), lane);  // next round to issue
#pragma unroll
    for (int i = 0; i < RING; i++) {
        ring_issue<WEIGHTED>(ring, i, ep, B.bend, arcs, cls, w, lane);
        if (ep < B.bend) ep = ring_skip(B, ep + BROUND, lane);
    }
    int slot0 = 0;  // ring slot of the pass's first round
    for (; b < nblocks; b += GW) {
        const int64_t r0 = 32 * b;
        const bool more = b + GW < nblocks;
        // next block's offsets, in flight during this block
        const int64_t nr0 = 32 * (b + GW);
        const int64_t o_lo_n = more ? __ldcs(offsets + min(nr0 + lane, n)) : 0;
        const int64_t o_31_n = (more && lane == 31) ? __ldcs(offsets + min(nr0 + 32, n)) : 0;
        // PAD: single-chunk rows (padded length BU) go to single_row, not to
        // the window
        const unsigned singlem =
            (PAD && BLOCK_SINGLE_ROWS) ? __ballot_sync(0xffffffffu, ((B.nzm >> lane) & 1u) && B.oh - B.ol == BU) : 0u;
        const unsigned winm = B.nzm & ~singlem;
        const int rank = __popc(winm & below);
        const int orank = __popc(B.anym & below);
        const int nnz = __popc(winm);
        const bool owner = (B.anym >> lane) & 1u;
        const bool nz = (winm >> lane) & 1u;
        const int32_t lend = (int32_t)(B.bend - B.base);
        const int rows = (int)min((int64_t)32, n - r0);
        float *zb = z + r0 * (int64_t)kk;
        if ((winm | B.hvm) != B.vm) {  // empty or single rows: zero-fill the block's Z range
            const int total = rows * kk;
            const int q4 = total >> 2;
            float4 *z4 = reinterpret_cast<float4 *>(zb);
            for (int q = lane; q < q4; q += 32) z4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int e = 4 * q4 + lane; e < total; e += 32) zb[e] = 0.f;
        }
        RingBlk NB;
        bool opened = false;
        for (int p0 = 0; p0 < max(nnz, 1); p0 += nslots) {
            const bool mine = nz && rank >= p0 && rank < p0 + nslots;
            if (owner) s_soff[orank + 1] = mine ? (rank - p0) * pkb + 3 : -1;
            if (mine) s_row[rank - p0] = lane;
            const int npass = min(nslots, nnz - p0);
            __syncwarp();
            int64_t ec = ring_skip(B, B.base & ~(int64_t)(BU - 1), lane);  // next round to consume
            int slot = slot0;
            while (ec < B.bend) {
                cp_wait<RING - 1>();
                const uint8_t *rs = ring + slot * RSLOT;
                const uint2 ca = *reinterpret_cast<const uint2 *>(rs + lane * BU);
                float wa[BU];
                if (WEIGHTED) {
                    const float4 x0 = *reinterpret_cast<const float4 *>(rs + RING_CLS + lane * BU * 4);
                    const float4 x1 = *reinterpret_cast<const float4 *>(rs + RING_CLS + lane * BU * 4 + 16);
                    wa[0] = x0.x, wa[1] = x0.y, wa[2] = x0.z, wa[3] = x0.w;
                    wa[4] = x1.x, wa[5] = x1.y, wa[6] = x1.z, wa[7] = x1.w;
                } else {
#pragma unroll
                    for (int u = 0; u < BU; u++) wa[u] = 1.f;
                }
                if (nnz > 0) {
                    if (PAD)
                        block_round_pad<WEIGHTED>(vw, s_soff, lane, owner, B.ol, (int32_t)(ec - B.base), lend, hoff,
                                                  trash, qscale, ca, wa);
                    else
                        block_round_acc<WEIGHTED>(vw, s_soff, s_mask, rot, lane, owner, B.ol, (int32_t)(ec - B.base),
                                                  lend, hoff, trash, qscale, ca, wa);
                }
                __syncwarp();
                // refill the slot just consumed with the round RING ahead
                ring_issue<WEIGHTED>(ring, slot, ep, B.bend, arcs, cls, w, lane);
                if (ep < B.bend) ep = ring_skip(B, ep + BROUND, lane);
                slot = slot + 1 == RING ? 0 : slot + 1;
                ec = ring_skip(B, ec + BROUND, lane);
            }
            // prime the ring for what comes next: this block's next pass, or
            // the next block's first rounds (in flight during the write-out)
            const bool last = p0 + nslots >= nnz;
            if (!last) {
                ep = ring_skip(B, B.base & ~(int64_t)(BU - 1), lane);
            } else if (more) {
                NB = ring_open(nr0, n, o_lo_n, o_31_n, heavy_arcs, lane);
                opened = true;
                ep = ring_skip(NB, NB.base & ~(int64_t)(BU - 1), lane);
            }
            if (!last || more) {
                const RingBlk &P = last ? NB : B;
#pragma unroll
                for (int i = 0; i < RING; i++) {
                    ring_issue<WEIGHTED>(ring, (slot + i) % RING, ep, P.bend, arcs, cls, w, lane);
                    if (ep < P.bend) ep = ring_skip(P, ep + BROUND, lane);
                }
                slot0 = slot;
            }
            if (nnz == 0) break;
            // write this pass's rows from their slots: each lane owns column
            // pairs (scale factors hoisted), rows loop with uniform addresses
            if ((kk & 1) == 0) {
                for (int c2 = lane; c2 < half; c2 += 32) {
                    const float2 f = *reinterpret_cast<const float2 *>(sc1 + 2 * c2);
                    uint32_t *vs = vw + 4 + 2 * c2;
                    float *zc = zb + 2 * c2;
                    for (int sl = 0; sl < npass; sl++, vs += pkb) {
                        const uint2 lo = *reinterpret_cast<uint2 *>(vs);
                        *reinterpret_cast<uint2 *>(vs) = make_uint2(0u, 0u);
                        float s0, s1;
                        if (WEIGHTED) {
                            const uint2 hi = *reinterpret_cast<uint2 *>(vs + hoff);
                            *reinterpret_cast<uint2 *>(vs + hoff) = make_uint2(0u, 0u);
                            s0 = (float)(long long)(((unsigned long long)hi.x << BLOCK_SPLIT) + lo.x);
                            s1 = (float)(long long)(((unsigned long long)hi.y << BLOCK_SPLIT) + lo.y);
                        } else {
                            s0 = (float)lo.x;
                            s1 = (float)lo.y;
                        }
                        __stcs(reinterpret_cast<float2 *>(zc + s_row[sl] * kk), make_float2(s0 * f.x, s1 * f.y));
                    }
                }
            } else {
                for (int c = lane; c < kk; c += 32) {
                    const float f = sc1[c];
                    uint32_t *vs = vw + 4 + c;
                    for (int sl = 0; sl < npass; sl++, vs += pkb) {
                        const uint32_t lo = *vs;
                        *vs = 0u;
                        float s0;
                        if (WEIGHTED) {
                            const uint32_t hi = vs[hoff];
                            vs[hoff] = 0u;
                            s0 = (float)(long long)(((unsigned long long)hi << BLOCK_SPLIT) + lo);
                        } else {
                            s0 = (float)lo;
                        }
                        __stcs(zb + s_row[sl] * kk + c, s0 * f);
                    }
                }
            }
            __syncwarp();
        }
        if (PAD && singlem) {
            __syncwarp();  // the zero fill lands before the single rows' entries
            if ((singlem >> lane) & 1u)
                single_row<WEIGHTED>(cls, w, B.base + B.ol, qscale, sc1, zb + (int64_t)lane * kk);
        }
        if (!more) break;
        B = opened ? NB : ring_open(nr0, n, o_lo_n, o_31_n, heavy_arcs, lane);
    }
    cp_wait<0>();
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

// Heavy rows for gee_reduce_heavy, one warp per work item: an item is a
// run of up to HEAVY_ITEM_ARCS arcs of one heavy row.  Lanes take 8
// contiguous arcs per round (one 8-byte class load, two 16-byte weight
// loads; the next round in flight) into the carry-free split window of the
// block kernel; every BLOCK_ROW_MAX arcs the window is folded into per-lane
// 64-bit column sums in registers.  An item that is its row's only item
// writes the Z row itself; the items of longer (mega) rows meet in acc[m]
// through 64-bit atomics and a small finalize.
constexpr int HCOL = 8;   // columns per lane: k <= 256
constexpr int HCOPY = 4;  // private window copies per warp (heavy items)

template <bool WEIGHTED>
__global__ void __launch_bounds__(RT)
k_reduce_heavy_items(const int64_t *__restrict__ item_first, const int64_t *__restrict__ item_end,
                     const int32_t *__restrict__ item_row, const int32_t *__restrict__ item_slot, int64_t n_items,
                     const uint8_t *__restrict__ cls, const float *__restrict__ w, float qscale, double dscale,
                     const double *__restrict__ inv, int32_t k, int64_t arcs, unsigned long long *__restrict__ acc,
                     unsigned long long *__restrict__ counter, float *__restrict__ z)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int kk = k;
    const int pkb = block_vec_words(kk);  // [3 pad | trash | bins 1..k | pad]
    constexpr int RSLOT = RING_CLS + (WEIGHTED ? RING_W : 0);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *ring = smem_raw + wid * RING * RSLOT;
    float *sc1 = reinterpret_cast<float *>(smem_raw + RW * RING * RSLOT);  // sc1[c] = inv[c+1] * dscale
    // HCOPY private copies of the window per warp (lane groups of 32/HCOPY):
    // all lanes add into one row, so a single copy serialises on equal
    // classes; the copy stride (== 4 mod 32 words) puts copies on other banks
    const int cs = pkb * Acc<WEIGHTED>::planes + 4;
    uint32_t *vw = reinterpret_cast<uint32_t *>(sc1 + pkb) + wid * HCOPY * cs;
    uint32_t *v = vw + (lane / (32 / HCOPY)) * cs;
    for (int c = threadIdx.x; c < pkb; c += RT) sc1[c] = c < kk ? (float)(inv[c + 1] * dscale) : 0.f;
    for (int i = lane; i < HCOPY * cs; i += 32) vw[i] = 0u;
    __syncthreads();
    // items come largest first; warps fetch them dynamically.  Rounds are
    // 256-arc aligned, so each aligned BLOCK_ROW_MAX window holds whole
    // rounds; RING rounds stay in flight (cp.async ring) within an item.
    for (;;) {
        int64_t it = 0;
        if (lane == 0) it = (int64_t)atomicAdd(counter, 1ull);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= n_items) break;
        const int64_t b0 = item_first[it], e1 = item_end[it];
        unsigned long long sum[HCOL];
#pragma unroll
        for (int j = 0; j < HCOL; j++) sum[j] = 0ull;
        int64_t ep = b0 & ~(int64_t)(BROUND - 1);
#pragma unroll
        for (int i = 0; i < RING; i++) {
            ring_issue<WEIGHTED, false>(ring, i, ep, e1, arcs, cls, w, lane);
            ep += BROUND;
        }
        int slot = 0;
        for (int64_t e0 = b0 & ~(int64_t)(BROUND - 1); e0 < e1; e0 += BROUND) {
            cp_wait<RING - 1>();
            const uint8_t *rs = ring + slot * RSLOT;
            const uint2 ca = *reinterpret_cast<const uint2 *>(rs + lane * BU);
            float wa[BU];
            if (WEIGHTED) {
                const float4 x0 = *reinterpret_cast<const float4 *>(rs + RING_CLS + lane * BU * 4);
                const float4 x1 = *reinterpret_cast<const float4 *>(rs + RING_CLS + lane * BU * 4 + 16);
                wa[0] = x0.x, wa[1] = x0.y, wa[2] = x0.z, wa[3] = x0.w;
                wa[4] = x1.x, wa[5] = x1.y, wa[6] = x1.z, wa[7] = x1.w;
            }
            const int64_t a0 = e0 + lane * BU;
            const bool full = a0 >= b0 && a0 + BU <= e1;
#pragma unroll
            for (int u = 0; u < BU; u++) {
                uint32_t c = __byte_perm(u < 4 ? ca.x : ca.y, 0u, 0x4440 + (u & 3));
                if (!full && (a0 + u < b0 || a0 + u >= e1)) c = 0u;
                if (c == 0u) continue;
                uint32_t *p = v + 3 + c;
                if (WEIGHTED) {
                    const unsigned long long qv = (unsigned long long)__float2ll_rn(wa[u] * qscale);
                    atomicAdd(p, (uint32_t)qv & ((1u << BLOCK_SPLIT) - 1u));
                    atomicAdd(p + pkb, (uint32_t)(qv >> BLOCK_SPLIT));
                } else {
                    atomicAdd(p, 1u);
                }
            }
            ring_issue<WEIGHTED, false>(ring, slot, ep, e1, arcs, cls, w, lane);
            ep += BROUND;
            slot = slot + 1 == RING ? 0 : slot + 1;
            // fold the window into the 64-bit sums at each aligned window end
            const int64_t en = e0 + BROUND;
            if ((en & (BLOCK_ROW_MAX - 1)) == 0 || en >= e1) {
                __syncwarp();
#pragma unroll
                for (int j = 0; j < HCOL; j++) {
                    const int c = lane + 32 * j;
                    if (c < kk) {
#pragma unroll
                        for (int q = 0; q < HCOPY; q++) {
                            uint32_t *p = vw + q * cs + 4 + c;
                            unsigned long long t = *p;
                            *p = 0u;
                            if (WEIGHTED) {
                                t += (unsigned long long)p[pkb] << BLOCK_SPLIT;
                                p[pkb] = 0u;
                            }
                            sum[j] += t;
                        }
                    }
                }
                __syncwarp();
            }
        }
        cp_wait<0>();
        const int32_t slotm = item_slot[it];
        if (slotm < 0) {  // the row's only item: write its Z row
            float *zr = z + (int64_t)item_row[it] * kk;
#pragma unroll
            for (int j = 0; j < HCOL; j++) {
                const int c = lane + 32 * j;
                if (c < kk) zr[c] = (WEIGHTED ? (float)(long long)sum[j] : (float)sum[j]) * sc1[c];
            }
        } else {
#pragma unroll
            for (int j = 0; j < HCOL; j++) {
                const int c = lane + 32 * j;
                if (c < kk && sum[j]) atomicAdd(&acc[(int64_t)slotm * kk + c], sum[j]);
            }
        }
    }
}

// Heavy-row finalize, one warp per heavy row: Z[row] = acc[h] * inv (and
// acc cleared for the next call).
template <bool WEIGHTED>
__global__ void k_heavy_finalize_rows(const int32_t *__restrict__ heavy_rows, int64_t n_heavy, int32_t k,
                                      unsigned long long *__restrict__ acc, const double *__restrict__ inv,
                                      double dscale, float *__restrict__ z)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t GW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t h = gw; h < n_heavy; h += GW) {
        unsigned long long *a = acc + h * k;
        float *zr = z + (int64_t)heavy_rows[h] * k;
        for (int c = lane; c < k; c += 32) {
            const unsigned long long s = a[c];
            a[c] = 0ull;
            const float f = WEIGHTED ? (float)(long long)s : (float)s;
            zr[c] = f * (float)(inv[c + 1] * dscale);
        }
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

static int reduce_blocks_impl(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                              const double *inv, int32_t k, int64_t heavy_arcs, const int32_t *heavy_rows,
                              int64_t n_heavy, const int64_t *chunk_first, const int32_t *chunk_heavy,
                              int64_t n_chunks, void *heavy_acc, float *z, void *stream, bool pad);

int gee_reduce_blocks(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                      const double *inv, int32_t k, int64_t heavy_arcs, const int32_t *heavy_rows, int64_t n_heavy,
                      const int64_t *chunk_first, const int32_t *chunk_heavy, int64_t n_chunks, void *heavy_acc,
                      float *z, void *stream)
{
    return reduce_blocks_impl(offsets, n, cls, w, scale_exp, inv, k, heavy_arcs, heavy_rows, n_heavy, chunk_first,
                              chunk_heavy, n_chunks, heavy_acc, z, stream, false);
}

int gee_reduce_blocks_pad8(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                           const double *inv, int32_t k, int64_t heavy_arcs, float *z, void *stream)
{
    return reduce_blocks_impl(offsets, n, cls, w, scale_exp, inv, k, heavy_arcs, nullptr, 0, nullptr, nullptr, 0,
                              nullptr, z, stream, true);
}

static int reduce_blocks_impl(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                              const double *inv, int32_t k, int64_t heavy_arcs, const int32_t *heavy_rows,
                              int64_t n_heavy, const int64_t *chunk_first, const int32_t *chunk_heavy,
                              int64_t n_chunks, void *heavy_acc, float *z, void *stream, bool pad)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs 1 <= k <= 255 (got %d)", k);
    GEE_REQUIRE(n >= 0 && n_heavy >= 0 && n_chunks >= 0 && heavy_arcs >= 1, GEE_ERR_INVALID, "bad sizes");
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && z && inv && cls, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(n_heavy == 0 || (heavy_rows && chunk_first && chunk_heavy && heavy_acc), GEE_ERR_INVALID,
                "heavy rows need their chunk list and accumulator");
    cudaStream_t st = gee::as_stream(stream);
    const bool weighted = w != nullptr;
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = weighted ? ldexp(1.0, -scale_exp) : 1.0;
    const size_t vec = (((size_t)k + 3) & ~(size_t)3) * (weighted ? 2 : 1) * sizeof(uint32_t);
    // slots per warp: up to 16, within ~64 KB per CTA so several CTAs fit per SM
    // slots per warp: up to 24 (+32 trash words), within the shared memory
    // share of one of the BLOCKS_MINB CTAs per SM
    const size_t planes = weighted ? 2 : 1;
    const size_t fixed = (size_t)block_vec_words(k) * sizeof(float) + (size_t)RW * BMETA * sizeof(int32_t) +
                         (size_t)RW * planes * 32 * sizeof(uint32_t);
    const size_t vecb = (size_t)block_vec_words(k) * planes * sizeof(uint32_t);
    const size_t budget = (size_t)(gee::smem_per_sm() / BLOCKS_MINB) - 1024;
    int nslots = (int)((budget - fixed) / (RW * vecb));
    if (nslots > 24) nslots = 24;
    if (nslots < 1) nslots = 1;
    const size_t sh = fixed + (size_t)RW * nslots * vecb;
    const bool vld = (reinterpret_cast<uintptr_t>(cls) & 7) == 0 && (!weighted || (reinterpret_cast<uintptr_t>(w) & 15) == 0);
    GEE_REQUIRE((reinterpret_cast<uintptr_t>(z) & 15) == 0, GEE_ERR_INVALID, "z must be 16-byte aligned");
    GEE_REQUIRE(heavy_arcs <= BLOCK_ROW_MAX, GEE_ERR_INVALID,
                "block reducer takes rows of at most %lld arcs (heavy_arcs %lld)", (long long)BLOCK_ROW_MAX,
                (long long)heavy_arcs);
    const int64_t nblocks = (n + 31) / 32;
    const int grid = grid_for(nblocks * 32, RT, 8);
    int rc;
    const char *ringenv = getenv("GEE_BLOCKS_RING");
    GEE_REQUIRE(!pad || !ringenv || atoi(ringenv) != 0, GEE_ERR_INVALID, "padded rows need the ring reducer");
    if (pad || !ringenv || atoi(ringenv) != 0) {
        // ring variant: RING rounds per warp in shared memory, 2 CTAs per SM
        const size_t ring = (size_t)RW * RING * (RING_CLS + (weighted ? RING_W : 0));
        const size_t budget2 = (size_t)(gee::smem_per_sm() / 2) - 1024;
        int ns = (int)((budget2 - fixed - ring) / (RW * vecb));
        if (ns > 24) ns = 24;
        if (ns >= 4) {
            const size_t shr = ring + fixed + (size_t)RW * ns * vecb;
            const int rgrid = (int)std::min<int64_t>((nblocks + RW - 1) / RW, (int64_t)gee::sm_count() * 2);
            auto kern = weighted ? (pad ? k_reduce_blocks_ring<true, true> : k_reduce_blocks_ring<true, false>)
                                 : (pad ? k_reduce_blocks_ring<false, true> : k_reduce_blocks_ring<false, false>);
            GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shr));
            kern<<<rgrid, RT, shr, st>>>(offsets, n, cls, w, qscale, dscale, inv, k, heavy_arcs, ns, z);
            if ((rc = gee::check_launch("k_reduce_blocks_ring"))) return rc;
            goto heavy;
        }
    }
    if (weighted) {
        GEE_CUDA(cudaFuncSetAttribute(k_reduce_blocks<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        k_reduce_blocks<true><<<grid, RT, sh, st>>>(offsets, n, cls, w, qscale, dscale, inv, k, heavy_arcs, nslots, vld, z);
    } else {
        GEE_CUDA(cudaFuncSetAttribute(k_reduce_blocks<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        k_reduce_blocks<false><<<grid, RT, sh, st>>>(offsets, n, cls, w, qscale, dscale, inv, k, heavy_arcs, nslots, vld, z);
    }
    if ((rc = gee::check_launch("k_reduce_blocks"))) return rc;
heavy:
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

int gee_reduce_heavy(const uint8_t *cls, const float *w, int64_t arcs, int32_t scale_exp, const double *inv,
                     int32_t k, const int64_t *item_first, const int64_t *item_end, const int32_t *item_row,
                     const int32_t *item_slot, int64_t n_items, const int32_t *mega_rows, int64_t n_mega,
                     void *mega_acc, int64_t *counter, float *z, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs 1 <= k <= 255 (got %d)", k);
    GEE_REQUIRE(n_items >= 0 && n_mega >= 0, GEE_ERR_INVALID, "bad sizes");
    if (n_items == 0) return GEE_OK;
    GEE_REQUIRE(cls && inv && z && item_first && item_end && item_row && item_slot, GEE_ERR_INVALID,
                "NULL array argument");
    GEE_REQUIRE(n_mega == 0 || (mega_rows && mega_acc), GEE_ERR_INVALID, "mega rows need their accumulator");
    GEE_REQUIRE(counter != nullptr, GEE_ERR_INVALID, "counter must not be NULL");
    cudaStream_t st = gee::as_stream(stream);
    const bool weighted = w != nullptr;
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = weighted ? ldexp(1.0, -scale_exp) : 1.0;
    const size_t sh = (size_t)RW * RING * (RING_CLS + (weighted ? RING_W : 0)) +
                      (size_t)block_vec_words(k) * sizeof(float) +
                      (size_t)RW * HCOPY * (block_vec_words(k) * (weighted ? 2 : 1) + 4) * sizeof(uint32_t);
    GEE_REQUIRE((reinterpret_cast<uintptr_t>(cls) & 7) == 0 && (!weighted || (reinterpret_cast<uintptr_t>(w) & 15) == 0),
                GEE_ERR_INVALID, "cls must be 8-byte and w 16-byte aligned");
    auto *acc = static_cast<unsigned long long *>(mega_acc);
    auto *ctr = reinterpret_cast<unsigned long long *>(counter);
    GEE_CUDA(cudaMemsetAsync(ctr, 0, sizeof(*ctr), st));
    const int hgrid = grid_for(n_items * 32, RT, 8);
    if (weighted)
        GEE_CUDA(cudaFuncSetAttribute(k_reduce_heavy_items<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    else
        GEE_CUDA(cudaFuncSetAttribute(k_reduce_heavy_items<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    if (weighted)
        k_reduce_heavy_items<true><<<hgrid, RT, sh, st>>>(item_first, item_end, item_row, item_slot, n_items, cls, w,
                                                          qscale, dscale, inv, k, arcs, acc, ctr, z);
    else
        k_reduce_heavy_items<false><<<hgrid, RT, sh, st>>>(item_first, item_end, item_row, item_slot, n_items, cls, w,
                                                           qscale, dscale, inv, k, arcs, acc, ctr, z);
    int rc;
    if ((rc = gee::check_launch("k_reduce_heavy_items"))) return rc;
    if (n_mega == 0) return GEE_OK;
    const int fgrid = grid_for(n_mega * 32, 256, 8);
    if (weighted)
        k_heavy_finalize_rows<true><<<fgrid, 256, 0, st>>>(mega_rows, n_mega, k, acc, inv, dscale, z);
    else
        k_heavy_finalize_rows<false><<<fgrid, 256, 0, st>>>(mega_rows, n_mega, k, acc, inv, dscale, z);
    return gee::check_launch("k_heavy_finalize_rows");
}

int gee_block_scale_exp(double max_row_abs, double max_abs, double min_abs_nz, int32_t *scale_exp, double *rel_err)
{
    gee::clear_error();
    GEE_REQUIRE(scale_exp != nullptr, GEE_ERR_INVALID, "scale_exp must not be NULL");
    int e = 126;
    int ex;
    if (max_row_abs > 0) {  // max_row_abs * 2^e < 2^62 (64-bit row sums, heavy path)
        frexp(max_row_abs, &ex);
        e = min(e, 62 - ex);
    }
    if (max_abs > 0) {  // max|w| * 2^e < 2^(BLOCK_SPLIT + 21): the split planes stay below 2^32
        frexp(max_abs, &ex);
        e = min(e, BLOCK_SPLIT + 21 - ex);
    }
    if (max_row_abs <= 0 && max_abs <= 0) e = 0;
    if (e < -126) e = -126;
    *scale_exp = e;
    if (rel_err) *rel_err = min_abs_nz > 0 ? ldexp(1.0, -(e + 1)) / min_abs_nz : 0.0;
    return GEE_OK;
}

}  // extern "C"
