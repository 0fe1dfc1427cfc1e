// K4b: the segmented class reduction of the split pull (light rows: one warp
// per 32-row block; heavy rows: work items).
//
// After gee_gather_labels has turned every arc x -> v of the padded,
// slot-sorted symmetric CSR into its class byte cls[e] = Y[v], the pull pass
// is a gather-free segmented histogram per row (reference arc rule,
// /root/reference/pkg/src/gee/_kernels.py:192-199, SOURCE_ONLY storage
// encoder.py:37-55):
//     Z[x, c] = inv[c+1] * sum_{e in row x, cls[e] = c+1} w[e].
//
// Sums are exact integers (unit weights: u32 counts; weighted: fixed point
// q = rint(w 2^e), split into two u32 planes, see BLOCK_SPLIT), so Z is
// bit-stable run to run and independent of arc order.  Every Z row is
// written exactly once (empty rows as zeros): no separate zero wave
// (zero_worker, _kernels.py:124-135).
#include <algorithm>
#include <cstdlib>

#include "gee_common.cuh"

namespace {

constexpr int RT = 256;       // threads per CTA
constexpr int RW = RT / 32;   // warps per CTA

template <bool WEIGHTED>
struct Acc {
    static constexpr int planes = WEIGHTED ? 2 : 1;
};

// Block reducer: one warp per block of 32 consecutive rows.  Lane i loads
// offsets[r0+i] (one coalesced load per block).  The block's arcs stream in
// rounds of 32 x 8 contiguous arcs through a per-warp cp.async ring.  Rows
// are padded to multiples of 8 arcs (gee_pad_rows), so each lane's 8 arcs
// belong to one row (block_round_pad).  Nonempty rows get compact slots in a
// warp-private window.  The block's Z range is zero-filled with 16-byte
// stores when it holds empty rows, then the nonempty rows are written from
// their slots; heavy rows are left to gee_reduce_heavy.  Blocks with more
// than `nslots` nonempty rows take several passes.
//
// Signed fixed point.  q = rint(w 2^e) is split as q = A 2^21 + B with
// B = q & (2^21 - 1) in [0, 2^21) and A = q >> 21 (arithmetic).  Each plane is
// summed in a u32 word: the B sum is below 2048 * 2^21 = 2^32 (no wrap), and
// gee_block_scale_exp keeps |q| < 2^41, so |A| <= 2^20 and the A sum over a
// row of <= 2048 arcs lies in [-2^31, 2^31): the u32 word holds its two's
// complement, and the decode sign-extends it (plane_sum).  Negative class
// sums are therefore exact, as the reference's any-finite-weight contract
// requires (graph.py:46-47).
constexpr int BU = 8;            // contiguous arcs per lane per round
constexpr int BLOCK_SPLIT = 21;  // weighted: low plane takes q's low 21 bits
constexpr int64_t BLOCK_ROW_MAX = 2048;  // longest row the block kernel takes (longer: heavy path)
constexpr int BROUND = 32 * BU;  // arcs per warp round
constexpr int BMETA = 96;        // per-warp ints: 3 x 8 mask words, 33 slot offsets, 32 rows (+pad)


// Window of one warp: per plane [nslots x vector | 32 trash words]; a slot's
// vector is [3 pad | unused | bin 1 .. bin k | pad] so that bin pairs
// (2j+1, 2j+2) are 8-byte aligned for the write-out.  Masked arcs (class 0,
// past the block, rows outside this pass) add into the lane's own trash
// word: no branch, and no two lanes on one address.
__host__ __device__ constexpr int block_vec_words(int k) { return 4 + ((k + 3) & ~3); }

// Exact plane decode: A (two's complement in a u32) * 2^21 + B.
__device__ __forceinline__ long long plane_sum(uint32_t lo, uint32_t hi)
{
    return (long long)(int32_t)hi * (1ll << BLOCK_SPLIT) + (long long)lo;
}


// One round over PADDED rows (every row's arc run is a multiple of BU, so
// each lane's 8 arcs belong to one row): the lane's owner rank is the count
// of rows started before the round plus the row starts at lane chunks <= its
// own -- one ballot, one OR-reduction, two popcounts, no shared masks.
template <bool WEIGHTED, int SHORT = 0>  // SHORT: <= 4 (the arcs' classes lie in the chunk's first word)
__device__ __forceinline__ void block_round_pad(uint32_t *__restrict__ vw, const int32_t *__restrict__ s_soff, int lane,
                                                bool owner, int32_t ol, int32_t lr, int32_t lend, int hoff, int trash,
                                                float qscale, const uint2 &ca, const float (&wa)[BU],
                                                float *__restrict__ zb, int kk, const float *__restrict__ sc1)
{
    const unsigned startm = __ballot_sync(0xffffffffu, owner && ol <= lr);
    const int32_t pos = ol - lr;
    const unsigned m = __reduce_or_sync(0xffffffffu, (owner && pos > 0 && pos < BROUND) ? 1u << (pos >> 3) : 0u);
    const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    const int r = __popc(startm) + __popc(m & upto);  // owner rank + 1 (0: before the block)
    const int so = s_soff[r];
    const bool inb = lr + lane * BU < lend;
    const bool ok = so >= 0 && inb;
    if (WEIGHTED && SHORT > 0 && so <= -2 && inb) {
        // a row of at most SHORT arcs (flagged at graph preparation; its
        // chunk is [the arcs | pads, class 0]): equal classes combine in
        // registers, exactly as the window would (plane_sum of the q's is
        // their sum), and the lane stores the row's nonzero entries into the
        // zero-filled Z row -- no window slot, no read-out.  Doing this for
        // every single-chunk row (8 arcs, 28 compares, 64-bit selects) cost
        // more than the window (C4 7.8 -> 9.1 ms); for the shortest rows it pays.
        GEE_DCHECK(-so - 2 < 32);
        float *zr = zb + (int64_t)(-so - 2) * kk;
        constexpr int NS = SHORT > 0 ? SHORT : 1;
        uint32_t cc[NS];
        long long qq[NS];
#pragma unroll
        for (int u = 0; u < SHORT; u++) {
            cc[u] = __byte_perm(ca.x, 0u, 0x4440 + u);
            GEE_DCHECK(cc[u] <= (uint32_t)kk);
            qq[u] = __float2ll_rn(wa[u] * qscale);
        }
#pragma unroll
        for (int u = 0; u < SHORT; u++) {
            bool first = cc[u] != 0u;
#pragma unroll
            for (int v = 0; v < u; v++) first = first && cc[v] != cc[u];
            if (first) {
                long long sum = qq[u];
#pragma unroll
                for (int v = u + 1; v < SHORT; v++) sum += cc[v] == cc[u] ? qq[v] : 0ll;
                zr[cc[u] - 1] = (float)sum * sc1[cc[u] - 1];
            }
        }
    }
    if (!WEIGHTED && so <= -2 && inb) {
        // a single-chunk row (padded length 8: <= 8 real arcs, all in this
        // lane's chunk; unit weights): equal classes combine in registers,
        // exactly as the window would, and the lane stores the row's nonzero
        // entries into the zero-filled Z row -- no atomics, no window slot,
        // no read-out.  C3 1.58 -> 1.48 ms.  Weighted rows keep the window:
        // the 64-bit combine, run in a divergent branch every round, cost
        // C4 7.8 -> 9.1 ms.
        GEE_DCHECK(-so - 2 < 32);
        float *zr = zb + (int64_t)(-so - 2) * kk;
        uint32_t cc[BU];
        unsigned long long qq[BU];
#pragma unroll
        for (int u = 0; u < BU; u++) {
            cc[u] = __byte_perm(u < 4 ? ca.x : ca.y, 0u, 0x4440 + (u & 3));
            qq[u] = WEIGHTED ? (unsigned long long)__float2ll_rn(wa[u] * qscale) : 1ull;
        }
#pragma unroll
        for (int u = 0; u < BU; u++) {
            bool first = cc[u] != 0u;
#pragma unroll
            for (int v = 0; v < u; v++) first = first && cc[v] != cc[u];
            if (first) {
                unsigned long long sum = qq[u];
#pragma unroll
                for (int v = u + 1; v < BU; v++) sum += cc[v] == cc[u] ? qq[v] : 0ull;
                zr[cc[u] - 1] = (WEIGHTED ? (float)(long long)sum : (float)sum) * sc1[cc[u] - 1];
            }
        }
    }
#pragma unroll
    for (int u = 0; u < BU; u++) {
        const uint32_t c = __byte_perm(u < 4 ? ca.x : ca.y, 0u, 0x4440 + (u & 3));
        // masked arcs (pads, unlabeled, other passes, past the block) add into
        // the lane's trash word: branch-free (predicating the atomics off
        // measured slower: 8.20 vs 8.01 ms on C4)
        GEE_DCHECK(c <= (uint32_t)kk);
        const int idx = (ok && c != 0u) ? so + (int)c : trash;
        GEE_DCHECK(idx >= 0 && idx < hoff);
        if (WEIGHTED) {
            const unsigned long long q = (unsigned long long)__float2ll_rn(wa[u] * qscale);
            atomicAdd(vw + idx, (uint32_t)q & ((1u << BLOCK_SPLIT) - 1u));
            atomicAdd(vw + hoff + idx, (uint32_t)(q >> BLOCK_SPLIT));
        } else {
            atomicAdd(vw + idx, 1u);
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
#ifndef GEE_RING
#define GEE_RING 3
#endif
#ifndef GEE_RING_H
#define GEE_RING_H 2
#endif
constexpr int RING = GEE_RING;      // block reducer
#ifndef GEE_BCTAS
#define GEE_BCTAS 2
#endif
constexpr int BCTAS = GEE_BCTAS;    // block-reducer CTAs per SM (shared memory and registers are sized for it)
constexpr int RING_H = GEE_RING_H;  // heavy items
#ifndef GEE_HSUB
#define GEE_HSUB 2
#endif
constexpr int HSUB = GEE_HSUB;            // 256-arc rounds per heavy ring slot (one pair of bulk copies each)
constexpr int HROUND = HSUB * BROUND;     // arcs per heavy ring slot
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

// Bulk-copy ring (Blackwell TMA unit): one elected lane per warp moves a
// round's class bytes and weights with two cp.async.bulk copies that
// complete_tx on the slot's mbarrier; the warp's lanes wait on the barrier's
// phase.  The copies bypass the LSU / L1TEX load path that the shared
// atomics saturate (the LDGSTS ring issued 96 lane copies per round).
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Per-block view shared by the warp (uniform fields) and per lane.
struct RingBlk {
    int64_t base, bend;      // arc range of the block
    unsigned nzm, hvm, anym, vm;
    int32_t ol, oh;          // this lane's row bounds, block-local
};

template <bool HV>
__device__ __forceinline__ RingBlk ring_open(int64_t r0, int64_t n, int64_t o_lo, int64_t o_hi31, int64_t heavy_arcs,
                                             int lane)
{
    RingBlk B;
    int64_t o_hi = __shfl_down_sync(0xffffffffu, o_lo, 1);
    if (lane == 31) o_hi = o_hi31;
    const bool valid = r0 + lane < n;
    const int64_t d = valid ? o_hi - o_lo : 0;
    const bool heavy = HV && d > heavy_arcs;  // !HV: the caller guarantees no row is longer (tile layout)
    GEE_DCHECK(HV || d <= BLOCK_ROW_MAX);
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
template <bool HV>
__device__ __forceinline__ int64_t ring_skip(const RingBlk &B, int64_t e, int lane)
{
    if (!HV || !B.hvm || e >= B.bend) return e;
    const int32_t lr = (int32_t)(e - B.base);
    const unsigned sm = __ballot_sync(0xffffffffu, ((B.anym >> lane) & 1u) && B.ol <= lr);
    if (!sm) return e;
    const int jr = 31 - __clz(sm);
    const int32_t hend = __shfl_sync(0xffffffffu, B.oh, jr);
    if (((B.hvm >> jr) & 1u) && B.base + hend >= e + BROUND) return (B.base + hend) & ~(int64_t)(BU - 1);
    return e;
}

// Arc span [lo, hi) of pass p0 (the nonempty light rows of ranks p0 ..
// p0 + nslots - 1): a block whose rows need several passes streams each
// pass's own arcs instead of the whole block again (C2: every block has 32
// nonempty rows for ~19 slots).  Rows are padded, so the bounds stay
// multiples of 8 arcs.  Warp-uniform.
__device__ __forceinline__ void pass_span(const RingBlk &B, unsigned winm, int p0, int nslots, int64_t &lo,
                                          int64_t &hi)
{
    const int nnz = __popc(winm);
    lo = B.base & ~(int64_t)(BU - 1);
    hi = B.bend;
    // the spans tile the block: a pass starts where the previous one ended,
    // so the single-chunk rows between two passes' rows are met exactly once
    if (p0 > 0) lo = B.base + __shfl_sync(0xffffffffu, B.oh, (int)__fns(winm, 0, p0));
    if (p0 + nslots < nnz) hi = B.base + __shfl_sync(0xffffffffu, B.oh, (int)__fns(winm, 0, p0 + nslots));
}

// Single-chunk rows (padded length BU) of a block: reduced in registers by
// the lane that holds their chunk (block_round_pad), not in the window
// (unit weights only).
template <bool WEIGHTED>
__device__ __forceinline__ unsigned single_rows(const RingBlk &B, int lane, unsigned one = 0u)
{
    // weighted: the short rows flagged at graph preparation (block_round_pad)
    return WEIGHTED ? (one & B.nzm) : __ballot_sync(0xffffffffu, ((B.nzm >> lane) & 1u) && B.oh - B.ol == BU);
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

// One round [e, e + BROUND) into ring slot `slot` by lane 0 (nothing when
// e >= bend).  e is a multiple of 16 (heavy items start their rounds at
// 256-arc boundaries, so class addresses are 16-byte aligned); the class stream is allocated
// with at least 64 bytes of slack, so a short last round may read the class
// bytes up to the next multiple of 16.  `arcs` is a multiple of 8 (padded
// rows), so the weights of a short round are a multiple of 32 bytes.
template <bool WEIGHTED>
__device__ __forceinline__ void ring_issue_bulk(uint8_t *ring, uint64_t *bars, int slot, int64_t e, int64_t bend,
                                                int64_t arcs, const uint8_t *__restrict__ cls,
                                                const float *__restrict__ w, int lane, uint64_t pol)
{
    if (lane != 0 || e >= bend) return;
    constexpr int RSLOT = HSUB * (RING_CLS + (WEIGHTED ? RING_W : 0));
    uint8_t *rs = ring + slot * RSLOT;
    int64_t na = arcs - e < HROUND ? arcs - e : HROUND;
    // no further than the 256-arc round that holds the item's last arc
    const int64_t need = ((bend - e + BROUND - 1) / BROUND) * BROUND;
    if (need < na) na = need;
    const uint32_t cb = (uint32_t)((na + 15) & ~(int64_t)15);
    const uint32_t wb = WEIGHTED ? (uint32_t)(na * 4) : 0u;
    mbar_expect_tx(bars + slot, cb + wb);
    bulk_g2s(rs, cls + e, cb, bars + slot, pol);
    if (WEIGHTED) bulk_g2s(rs + HSUB * RING_CLS, w + e, wb, bars + slot, pol);
}

// HV: rows longer than heavy_arcs may sit in the CSR (skipped here).  SHORT > 0 (weighted): one_arc[b]
// flags the rows of block b that hold at most SHORT arcs.
template <bool WEIGHTED, bool HV, int SHORT = 0>
__global__ void __launch_bounds__(RT, BCTAS)
k_reduce_blocks_ring(const int64_t *__restrict__ offsets, int64_t n, const uint8_t *__restrict__ cls,
                     const float *__restrict__ w, float qscale, double dscale, const double *__restrict__ inv,
                     int32_t k, int64_t heavy_arcs, int nslots, const uint32_t *__restrict__ one_arc,
                     float *__restrict__ z)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int kk = k;
    const int pkb = block_vec_words(kk);
    const int hoff = nslots * pkb + 32;
    const int wwords = hoff * Acc<WEIGHTED>::planes;
    constexpr int RSLOT = RING_CLS + (WEIGHTED ? RING_W : 0);
    uint8_t *ring_base = smem_raw;  // RW x RING x RSLOT (16-byte aligned)
    float *sc1 = reinterpret_cast<float *>(ring_base + RW * RING * RSLOT);
    int32_t *meta = reinterpret_cast<int32_t *>(sc1 + pkb);
    uint32_t *vbase = reinterpret_cast<uint32_t *>(meta + RW * BMETA);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *ring = ring_base + wid * RING * RSLOT;
    int32_t *s_soff = meta + wid * BMETA + 24;
    int32_t *s_row = s_soff + 36;
    uint32_t *vw = vbase + wid * wwords;
    for (int c = threadIdx.x; c < pkb; c += RT) sc1[c] = c < kk ? (float)(inv[c + 1] * dscale) : 0.f;
    for (int i = threadIdx.x; i < RW * wwords; i += RT) vbase[i] = 0u;
    for (int i = threadIdx.x; i < RW * BMETA; i += RT) meta[i] = -1;
    __syncthreads();
    const int trash = nslots * pkb + lane;
    const unsigned below = (1u << lane) - 1u;
    const int64_t nblocks = (n + 31) / 32;
    const int64_t gw = (int64_t)blockIdx.x * RW + wid, GW = (int64_t)gridDim.x * RW;
    const int64_t arcs = offsets[n];
    const int half = kk >> 1;

    // each warp takes a contiguous run of blocks: the last round of a block
    // overshoots into the next block's arcs, which this warp then reads again
    // at once (an L2 hit) instead of another warp much later (from DRAM)
    const int64_t b_end = ((gw + 1) * nblocks) / GW;
    int64_t b = (gw * nblocks) / GW;
    if (b >= b_end) return;
    // open the first block and prime its first rounds
    RingBlk B;
    {
        const int64_t r0 = 32 * b;
        const int64_t o_lo = __ldcs(offsets + min(r0 + lane, n));
        const int64_t o_31 = lane == 31 ? __ldcs(offsets + min(r0 + 32, n)) : 0;
        B = ring_open<HV>(r0, n, o_lo, o_31, heavy_arcs, lane);
    }
    unsigned one_b = SHORT ? __ldg(one_arc + b) : 0u;  // this block's short rows
    int64_t plo, phi;
    pass_span(B, B.nzm & ~single_rows<WEIGHTED>(B, lane, one_b), 0, nslots, plo, phi);
    int64_t ep = ring_skip<HV>(B, plo, lane);  // next round to issue
#pragma unroll
    for (int i = 0; i < RING; i++) {
        ring_issue<WEIGHTED>(ring, i, ep, phi, arcs, cls, w, lane);
        if (ep < phi) ep = ring_skip<HV>(B, ep + BROUND, lane);
    }
    int slot0 = 0;  // ring slot of the pass's first round
    for (; b < b_end; b++) {
        const int64_t r0 = 32 * b;
        const bool more = b + 1 < b_end;
        // next block's offsets, in flight during this block
        const int64_t nr0 = 32 * (b + 1);
        const int64_t o_lo_n = more ? __ldcs(offsets + min(nr0 + lane, n)) : 0;
        const int64_t o_31_n = (more && lane == 31) ? __ldcs(offsets + min(nr0 + 32, n)) : 0;
        const unsigned one_n = (SHORT && more) ? __ldg(one_arc + b + 1) : 0u;
        const unsigned singlem = single_rows<WEIGHTED>(B, lane, one_b);
        const unsigned winm = B.nzm & ~singlem;
        const int rank = __popc(winm & below);
        const int orank = __popc(B.anym & below);
        const int nnz = __popc(winm);
        const bool owner = (B.anym >> lane) & 1u;
        const bool nz = (winm >> lane) & 1u;
        const int32_t lend = (int32_t)(B.bend - B.base);
        const int rows = (int)min((int64_t)32, n - r0);
        float *zb = z + r0 * (int64_t)kk;
        if ((winm | B.hvm) != B.vm) {  // empty rows: zero-fill the block's Z range
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
            if (owner) s_soff[orank + 1] = mine ? (rank - p0) * pkb + 3 : (((singlem >> lane) & 1u) ? -2 - lane : -1);
            if (mine) s_row[rank - p0] = lane;
            const int npass = min(nslots, nnz - p0);
            __syncwarp();
            pass_span(B, winm, p0, nslots, plo, phi);
            int64_t ec = ring_skip<HV>(B, plo, lane);  // next round to consume
            int slot = slot0;
            while (ec < phi) {
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
                if (nnz > 0 || singlem)
                    block_round_pad<WEIGHTED, SHORT>(vw, s_soff, lane, owner, B.ol, (int32_t)(ec - B.base), lend, hoff,
                                              trash, qscale, ca, wa, zb, kk, sc1);
                __syncwarp();
                // refill the slot just consumed with the round RING ahead
                ring_issue<WEIGHTED>(ring, slot, ep, phi, arcs, cls, w, lane);
                if (ep < phi) ep = ring_skip<HV>(B, ep + BROUND, lane);
                slot = slot + 1 == RING ? 0 : slot + 1;
                ec = ring_skip<HV>(B, ec + BROUND, lane);
            }
            // prime the ring for what comes next: this block's next pass, or
            // the next block's first rounds (in flight during the write-out)
            const bool last = p0 + nslots >= nnz;
            int64_t nlo = 0, nhi = 0;
            if (!last) {
                pass_span(B, winm, p0 + nslots, nslots, nlo, nhi);
                ep = ring_skip<HV>(B, nlo, lane);
            } else if (more) {
                NB = ring_open<HV>(nr0, n, o_lo_n, o_31_n, heavy_arcs, lane);
                opened = true;
                pass_span(NB, NB.nzm & ~single_rows<WEIGHTED>(NB, lane, one_n), 0, nslots, nlo, nhi);
                ep = ring_skip<HV>(NB, nlo, lane);
            }
            if (!last || more) {
                const RingBlk &P = last ? NB : B;
#pragma unroll
                for (int i = 0; i < RING; i++) {
                    ring_issue<WEIGHTED>(ring, (slot + i) % RING, ep, nhi, arcs, cls, w, lane);
                    if (ep < nhi) ep = ring_skip<HV>(P, ep + BROUND, lane);
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
                            s0 = (float)plane_sum(lo.x, hi.x);
                            s1 = (float)plane_sum(lo.y, hi.y);
                        } else {
                            s0 = (float)lo.x;
                            s1 = (float)lo.y;
                        }
                        GEE_DCHECK(s_row[sl] >= 0 && s_row[sl] < 32 && r0 + s_row[sl] < n);
                        // (write-back, like the zero fill whose lines these rows overwrite in L2:
                        // 7.08 ms against 7.16 ms with streaming stores on C4)
                        *reinterpret_cast<float2 *>(zc + s_row[sl] * kk) = make_float2(s0 * f.x, s1 * f.y);
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
                            s0 = (float)plane_sum(lo, hi);
                        } else {
                            s0 = (float)lo;
                        }
                        zb[s_row[sl] * kk + c] = s0 * f;
                    }
                }
            }
            __syncwarp();
        }
        if (!more) break;
        B = opened ? NB : ring_open<HV>(nr0, n, o_lo_n, o_31_n, heavy_arcs, lane);
        one_b = one_n;
    }
    cp_wait<0>();
}


// Heavy rows for gee_reduce_heavy, one warp per work item: an item is a
// run of up to HEAVY_ITEM_ARCS arcs of one heavy row.  Lanes take 8
// contiguous arcs per round (one 8-byte class load, two 16-byte weight
// loads from the bulk-copy ring) into the carry-free split planes of the
// block kernel; before a plane can wrap, the window is folded into per-lane
// 64-bit sums in registers.  An item that is its row's only item writes the
// Z row itself; the items of longer (mega) rows meet in acc[m] through
// 64-bit atomics and a small finalize.
//
// Window copies per warp (heavy items).  All 32 lanes add into one row, and
// the kernel is bound by its shared atomics: on C4 (k = 50) it streams in
// 1.78 ms with no atomics, 1.86 ms with one per arc, 1.89 ms with two
// conflict-free ones and 2.50 ms with two into a copy-major window of 2
// copies (1 / 4 copies: 2.63 / 2.55 ms), whose banks are random.  A shared
// atomic serialises on lanes that meet in one bank -- on one word most of
// all.  The window is therefore kept in NC copies, INTERLEAVED: bin c of
// copy q is word c * NC + q of its plane, and lane l adds into copy l % NC.
// Lanes of different copies never share a bank; the 32 / NC lanes of one
// copy do when their classes agree mod 32 / NC.  A copy takes 1 / NC of the
// arcs, so the planes are folded every NC * 2048 arcs, by contiguous 16-byte
// loads; the copies of a bin meet by shuffles once per item.  C4: NC = 4 /
// 8 / 16 / 32 -> 2.31 / 2.25 / 2.37 / 4.30 ms (the window grows with NC:
// fewer warps per SM); C3 0.28 -> 0.18 ms.
#ifndef GEE_HNC
#define GEE_HNC 8
#endif
constexpr int HNC_SMALL = GEE_HNC;  // k <= 64
constexpr int HNC_LARGE = 4;        // k <= 255 (the window grows with k * NC)
__host__ __device__ constexpr int heavy_plane_words(int k, int nc) { return (((k + 1) * nc + 3) & ~3) + 32; }

__device__ __forceinline__ void red_shared_u32(uint32_t addr, uint32_t v)
{
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// One 256-arc round of a heavy item: the lane's 8 arcs add into its window
// copy (vb: shared byte address of bin 0 of the low plane; the high plane's
// bin lies pb bytes further).  Branch-free: class 0 (pads, unlabeled
// targets) and, in an item's first and last round (FULL = false), arcs
// outside the item add into the lane's own trash word tb, whose twin at
// tb + pb takes the high-plane add, so one select serves both planes.  A
// divergent skip per arc spent 30% of the kernel's instructions on branch
// bookkeeping (C4 2.58 -> 2.48 ms); dropping the per-arc mask test and the
// second select from the inner rounds halved the instructions again (22 ->
// 11 per arc) without changing the time: the shared atomics bind.
template <bool WEIGHTED, bool FULL, int NC>
__device__ __forceinline__ void heavy_round(uint32_t vb, uint32_t tb, uint32_t pb, const uint2 &ca,
                                            const float (&wa)[BU], float qscale, unsigned vm, int kk)
{
#pragma unroll
    for (int u = 0; u < BU; u++) {
        const uint32_t c = __byte_perm(u < 4 ? ca.x : ca.y, 0u, 0x4440 + (u & 3));
        const bool on = FULL ? c != 0u : (c != 0u && ((vm >> u) & 1u));
        GEE_DCHECK(!on || c <= (uint32_t)kk);  // (bytes past the item's last arc are whatever the ring slot held)
        const uint32_t a = on ? vb + (4u * NC) * c : tb;
        if (WEIGHTED) {
            const unsigned long long qv = (unsigned long long)__float2ll_rn(wa[u] * qscale);
            red_shared_u32(a, (uint32_t)qv & ((1u << BLOCK_SPLIT) - 1u));
            red_shared_u32(a + pb, (uint32_t)(qv >> BLOCK_SPLIT));
        } else {
            red_shared_u32(a, 1u);
        }
    }
}


template <bool WEIGHTED, int NC, int KMAX>  // NC copies (a multiple of 4), k <= KMAX
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
    constexpr int RSLOT = HSUB * (RING_CLS + (WEIGHTED ? RING_W : 0));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw) + wid * RING_H;
    uint8_t *ring_base = smem_raw + RW * RING_H * sizeof(uint64_t);
    uint8_t *ring = ring_base + wid * RING_H * RSLOT;
    float *sc1 = reinterpret_cast<float *>(ring_base + RW * RING_H * RSLOT);  // sc1[c] = inv[c+1] * dscale
    if (lane < RING_H) mbar_init(bars + lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t pol = policy_evict_first();
    uint32_t ph = 0;
    // the warp's window: per plane [bins (class, copy) | one trash word per
    // lane]; the high plane follows the low one, so a lane's trash word has
    // its twin pb bytes further, like every bin (never read)
    const int pw = heavy_plane_words(kk, NC), nbw = (kk + 1) * NC;  // plane words; bin words
    uint32_t *vw = reinterpret_cast<uint32_t *>(sc1 + pkb) + wid * (pw * Acc<WEIGHTED>::planes);
    const uint32_t vb = smem_u32(vw + (lane & (NC - 1))), tb = smem_u32(vw + pw - 32 + lane), pb = (uint32_t)pw * 4u;
    for (int c = threadIdx.x; c < pkb; c += RT) sc1[c] = c < kk ? (float)(inv[c + 1] * dscale) : 0.f;
    for (int i = lane; i < pw * Acc<WEIGHTED>::planes; i += 32) vw[i] = 0u;
    __syncthreads();
    // items come largest first; warps fetch them dynamically.  Rounds are
    // 256-arc aligned, so each aligned BLOCK_ROW_MAX window holds whole
    // rounds; RING_H rounds stay in flight (cp.async ring) within an item.
    for (;;) {
        int64_t it = 0;
        if (lane == 0) it = (int64_t)atomicAdd(counter, 1ull);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= n_items) break;
        const int64_t b0 = item_first[it], e1 = item_end[it];
        GEE_DCHECK(b0 >= 0 && b0 < e1 && e1 <= arcs);
        // fold mapping: lane l reads the 4 plane words [4l + 128m, +4) -- copies
        // 4(l % LPC) .. +3 of bin l / LPC + CPI m -- so a fold's loads are
        // contiguous across the warp; the LPC lanes of a bin meet at the item's end
        constexpr int LPC = NC / 4, CPI = 32 / LPC, NIT = (KMAX + CPI) / CPI;
        static_assert(NC % 4 == 0 && NC <= 32, "copies: a multiple of 4");
        unsigned long long sum[NIT];
#pragma unroll
        for (int j = 0; j < NIT; j++) sum[j] = 0ull;
        int64_t ep = b0 & ~(int64_t)(HROUND - 1);
#pragma unroll
        for (int i = 0; i < RING_H; i++) {
            ring_issue_bulk<WEIGHTED>(ring, bars, i, ep, e1, arcs, cls, w, lane, pol);
            ep += HROUND;
        }
        int slot = 0;
        for (int64_t e0 = b0 & ~(int64_t)(HROUND - 1); e0 < e1; e0 += BROUND) {
            const int sub = (int)((e0 & (HROUND - 1)) / BROUND);  // 256-arc round inside the slot
            if (sub == 0) {
                if (lane == 0) mbar_wait(bars + slot, (ph >> slot) & 1u);
                __syncwarp();
                ph ^= 1u << slot;
            }
            if (e0 + BROUND > b0) {  // (a slot's first round may lie wholly before the item: rounds are slot-aligned)
                const uint8_t *rs = ring + slot * RSLOT + sub * RING_CLS;
                const uint8_t *rw = ring + slot * RSLOT + HSUB * RING_CLS + sub * RING_W;
                const uint2 ca = *reinterpret_cast<const uint2 *>(rs + lane * BU);
                float wa[BU];
                if (WEIGHTED) {
                    const float4 x0 = *reinterpret_cast<const float4 *>(rw + lane * BU * 4);
                    const float4 x1 = *reinterpret_cast<const float4 *>(rw + lane * BU * 4 + 16);
                    wa[0] = x0.x, wa[1] = x0.y, wa[2] = x0.z, wa[3] = x0.w;
                    wa[4] = x1.x, wa[5] = x1.y, wa[6] = x1.z, wa[7] = x1.w;
                }
                // rounds that lie inside the item (all but its first and last) take
                // the mask-free body (warp-uniform choice)
                if (e0 >= b0 && e0 + BROUND <= e1) {
                    heavy_round<WEIGHTED, true, NC>(vb, tb, pb, ca, wa, qscale, 0xffu, kk);
                } else {
                    // arcs of this lane's chunk inside the item: bits [vlo, vhi)
                    const int64_t a0 = e0 + lane * BU;
                    const int vlo = (int)min((int64_t)BU, max((int64_t)0, b0 - a0));
                    const int vhi = (int)min((int64_t)BU, max((int64_t)0, e1 - a0));
                    heavy_round<WEIGHTED, false, NC>(vb, tb, pb, ca, wa, qscale, ((1u << vhi) - 1u) & ~((1u << vlo) - 1u), kk);
                }
            }
            if (sub == HSUB - 1 || e0 + BROUND >= e1) {
                __syncwarp();  // every lane has read the slot before it is refilled
                ring_issue_bulk<WEIGHTED>(ring, bars, slot, ep, e1, arcs, cls, w, lane, pol);
                ep += HROUND;
                slot = slot + 1 == RING_H ? 0 : slot + 1;
            }
            // fold the window into the 64-bit sums at each aligned window end: a
            // copy takes 1 / NC of every round's arcs, so its u32 planes hold
            // NC * BLOCK_ROW_MAX arcs of the item without wrapping
            const int64_t en = e0 + BROUND;
            if ((en & (NC * BLOCK_ROW_MAX - 1)) == 0 || en >= e1) {
                __syncwarp();
#pragma unroll
                for (int m = 0; m < NIT; m++) {
                    const int word = 4 * lane + 128 * m;
                    if (word < nbw) {
                        uint32_t *p = vw + word;
                        const uint4 lo = *reinterpret_cast<uint4 *>(p);
                        *reinterpret_cast<uint4 *>(p) = make_uint4(0u, 0u, 0u, 0u);
                        if (WEIGHTED) {
                            const uint4 hi = *reinterpret_cast<uint4 *>(p + pw);
                            *reinterpret_cast<uint4 *>(p + pw) = make_uint4(0u, 0u, 0u, 0u);
                            // wrapping u64 adds of the signed plane sums
                            sum[m] += (unsigned long long)plane_sum(lo.x, hi.x) + (unsigned long long)plane_sum(lo.y, hi.y) +
                                      (unsigned long long)plane_sum(lo.z, hi.z) + (unsigned long long)plane_sum(lo.w, hi.w);
                        } else {
                            sum[m] += (unsigned long long)lo.x + lo.y + lo.z + lo.w;
                        }
                    }
                }
                __syncwarp();
            }
        }
        const int32_t slotm = item_slot[it];
        float *zr = z + (int64_t)item_row[it] * kk;
#pragma unroll
        for (int m = 0; m < NIT; m++) {
            unsigned long long t = sum[m];
#pragma unroll
            for (int d = 1; d < LPC; d <<= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
            const int c = lane / LPC + CPI * m - 1;  // bin 0 is no class
            if (lane % LPC == 0 && c >= 0 && c < kk) {
                if (slotm < 0)  // the row's only item: write its Z row
                    zr[c] = (WEIGHTED ? (float)(long long)t : (float)t) * sc1[c];
                else if (t)
                    atomicAdd(&acc[(int64_t)slotm * kk + c], t);
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

static int reduce_blocks(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                         const double *inv, int32_t k, int64_t heavy_arcs, bool heavy_in_csr, const uint32_t *one_arc,
                         int32_t short_arcs, float *z, void *stream);

int gee_reduce_blocks_pad8(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                           const double *inv, int32_t k, int64_t heavy_arcs, float *z, void *stream)
{
    return reduce_blocks(offsets, n, cls, w, scale_exp, inv, k, heavy_arcs, true, nullptr, 0, z, stream);
}

int gee_reduce_blocks_light(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                            const double *inv, int32_t k, float *z, void *stream)
{
    return reduce_blocks(offsets, n, cls, w, scale_exp, inv, k, BLOCK_ROW_MAX, false, nullptr, 0, z, stream);
}

int gee_reduce_blocks_short(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                            const double *inv, int32_t k, const uint32_t *short_rows, int32_t short_arcs, float *z,
                            void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(short_rows == nullptr || (short_arcs >= 1 && short_arcs <= 4), GEE_ERR_INVALID,
                "short_arcs must be 1..4 (got %d)", short_arcs);
    return reduce_blocks(offsets, n, cls, w, scale_exp, inv, k, BLOCK_ROW_MAX, false, short_rows, short_arcs, z, stream);
}

static int reduce_blocks(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w, int32_t scale_exp,
                         const double *inv, int32_t k, int64_t heavy_arcs, bool heavy_in_csr, const uint32_t *one_arc,
                         int32_t short_arcs, float *z, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && k <= 255, GEE_ERR_INVALID, "class stream needs 1 <= k <= 255 (got %d)", k);
    GEE_REQUIRE(n >= 0 && heavy_arcs >= 1, GEE_ERR_INVALID, "bad sizes");
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && z && inv && cls, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(heavy_arcs <= BLOCK_ROW_MAX, GEE_ERR_INVALID,
                "block reducer takes rows of at most %lld arcs (heavy_arcs %lld)", (long long)BLOCK_ROW_MAX,
                (long long)heavy_arcs);
    GEE_REQUIRE(gee::aligned16(z), GEE_ERR_INVALID, "z must be 16-byte aligned");
    cudaStream_t st = gee::as_stream(stream);
    const bool weighted = w != nullptr;
    const float qscale = ldexpf(1.0f, scale_exp);
    const double dscale = weighted ? ldexp(1.0, -scale_exp) : 1.0;
    // RING rounds per warp in shared memory, 2 CTAs per SM; window slots per
    // warp: up to 24 (+32 trash words) in what is left of the CTA's share
    const size_t planes = weighted ? 2 : 1;
    const size_t fixed = (size_t)block_vec_words(k) * sizeof(float) + (size_t)RW * BMETA * sizeof(int32_t) +
                         (size_t)RW * planes * 32 * sizeof(uint32_t);
    const size_t vecb = (size_t)block_vec_words(k) * planes * sizeof(uint32_t);
    const size_t ring = (size_t)RW * RING * (RING_CLS + (weighted ? RING_W : 0));
    const size_t budget = (size_t)(gee::smem_per_sm() / BCTAS) - 1024;
    GEE_REQUIRE(budget > fixed + ring + RW * vecb, GEE_ERR_INVALID, "k = %d leaves no shared memory for the window", k);
    int ns = (int)((budget - fixed - ring) / (RW * vecb));
    if (ns > 24) ns = 24;
    const size_t shr = ring + fixed + (size_t)RW * ns * vecb;
    const int64_t nblocks = (n + 31) / 32;
    const int rgrid = (int)std::min<int64_t>((nblocks + RW - 1) / RW, (int64_t)gee::sm_count() * BCTAS);
    const int sh_arcs = (weighted && !heavy_in_csr && one_arc != nullptr) ? short_arcs : 0;
    auto kern = weighted ? (heavy_in_csr ? k_reduce_blocks_ring<true, true> : k_reduce_blocks_ring<true, false>)
                         : (heavy_in_csr ? k_reduce_blocks_ring<false, true> : k_reduce_blocks_ring<false, false>);
    if (sh_arcs == 1) kern = k_reduce_blocks_ring<true, false, 1>;
    if (sh_arcs == 2) kern = k_reduce_blocks_ring<true, false, 2>;
    if (sh_arcs == 3) kern = k_reduce_blocks_ring<true, false, 3>;
    if (sh_arcs == 4) kern = k_reduce_blocks_ring<true, false, 4>;
    const bool one = sh_arcs > 0;
    GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shr));
    kern<<<rgrid, RT, shr, st>>>(offsets, n, cls, w, qscale, dscale, inv, k, heavy_arcs, ns, one ? one_arc : nullptr, z);
    return gee::check_launch("k_reduce_blocks_ring");
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
    const int nc = k <= 64 ? HNC_SMALL : HNC_LARGE;
    const size_t sh = (size_t)RW * RING_H * (HSUB * (RING_CLS + (weighted ? RING_W : 0)) + sizeof(uint64_t)) +
                      (size_t)block_vec_words(k) * sizeof(float) +
                      (size_t)RW * heavy_plane_words(k, nc) * (weighted ? 2 : 1) * sizeof(uint32_t);
    GEE_REQUIRE((reinterpret_cast<uintptr_t>(cls) & 7) == 0 && (!weighted || (reinterpret_cast<uintptr_t>(w) & 15) == 0),
                GEE_ERR_INVALID, "cls must be 8-byte and w 16-byte aligned");
    auto *acc = static_cast<unsigned long long *>(mega_acc);
    auto *ctr = reinterpret_cast<unsigned long long *>(counter);
    GEE_CUDA(cudaMemsetAsync(ctr, 0, sizeof(*ctr), st));
    const int hgrid = grid_for(n_items * 32, RT, 8);
    auto kern = weighted ? (k <= 64 ? k_reduce_heavy_items<true, HNC_SMALL, 64> : k_reduce_heavy_items<true, HNC_LARGE, 255>)
                         : (k <= 64 ? k_reduce_heavy_items<false, HNC_SMALL, 64>
                                    : k_reduce_heavy_items<false, HNC_LARGE, 255>);
    GEE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    kern<<<hgrid, RT, sh, st>>>(item_first, item_end, item_row, item_slot, n_items, cls, w, qscale, dscale, inv, k, arcs,
                                acc, ctr, z);
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
    if (max_abs > 0) {  // |q| = max|w| * 2^e < 2^(BLOCK_SPLIT + 20): the signed high plane of a
        frexp(max_abs, &ex);  // 2048-arc row stays in [-2^31, 2^31), the low plane below 2^32
        e = min(e, BLOCK_SPLIT + 20 - ex);
    }
    if (max_row_abs <= 0 && max_abs <= 0) e = 0;
    if (e < -126) e = -126;
    *scale_exp = e;
    if (rel_err) *rel_err = min_abs_nz > 0 ? ldexp(1.0, -(e + 1)) / min_abs_nz : 0.0;
    return GEE_OK;
}

}  // extern "C"
