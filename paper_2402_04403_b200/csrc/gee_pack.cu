// Bit-width delta coding of the prepared targets, for shipping the graph
// over PCIe (stream.HostPipeline, the e2e path).  The reference hands its
// CsrGraph to embed_parallel in host memory (encoder.py:123-194, graph.py:54-91);
// on C4 the targets are 15.5 GB of the 33 GB that cross PCIe per call, and
// rows sorted by slot (gee_sort_rows) make them compressible.
//
// Layout.  The padded CSR (gee_pad_rows: rows are multiples of 8 arcs, pads
// are the sentinel slot at the row's end) is cut into groups of 8 arcs; a
// group never spans two rows.  Per group:
//   ctl[g]  = (b - 1) | pads << 5
//             b in 1..32 bits per value, pads 0..7 trailing sentinel arcs
//   payload = the group's 8 - pads real values as b-bit deltas (mod 2^32):
//             the first arc of a row is stored absolute, every other arc
//             relative to the previous arc of its row.
// The payload is one little-endian bit stream of u32 words; group g's values
// start at the sum of the earlier groups' (8 - pads) * b bits.  Row starts
// are not stored: the decoder marks them from the chunk's padded offsets,
// which cross PCIe anyway.  Unsorted rows still round-trip (deltas wrap mod
// 2^32); they compress less.  C4 (tools/pack_stats.py): 7.98 GB as byte-
// width groups, 6.40 GB as bit-width groups.
//
// Weights (weighted graphs) travel per group too, without the pads:
//   wctl[g] = B | e << 2: B = 0 raw f32 bits (4 bytes per real weight), or
//             B = 1..3 bytes per weight of an integer k with w = k * 2^-e
//             exactly (e in 0..63; all real weights of the group >= +0,
//             normal, and exactly representable that way) -- lossless
//             group fixed point; seeded (0,1] weights with 24-bit mantissas
//             take 3 bytes.  When every group of a chunk has the same wctl
//             the decoder takes it as one value (wctl_uniform) and the wctl
//             array need not travel.
//
// Decode (gee_unpack_targets, inside the timed e2e region; no allocation):
//   0. mark the row-start groups from the padded offsets;
//   1. exclusive scan over (payload bits, pads, weight bytes) per group ->
//      the group's bit offset and real-arc index (for the weight copy);
//   2. per group, the sum of its deltas; an inclusive segmented scan over
//      (sum, row_start) gives each group's last target;
//   3. per group, rebuild the 8 padded targets (sentinel for pads) and copy
//      the row's real weights into the padded weight layout (pads 0).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "gee_common.cuh"

namespace {

constexpr int PT = 256;

struct SegSum {  // segmented-scan element: running value, "a row starts here"
    uint32_t val;
    uint32_t flag;
};

struct SegOp {
    __device__ __forceinline__ SegSum operator()(const SegSum &a, const SegSum &b) const
    {
        return b.flag ? b : SegSum{a.val + b.val, a.flag};
    }
};

struct Pos {  // target payload bits, pad arcs and weight payload bytes before a group
    uint64_t bits;
    uint64_t pads;
    uint64_t wbytes;
};

struct PosSum {
    __host__ __device__ __forceinline__ Pos operator()(const Pos &a, const Pos &b) const
    {
        return Pos{a.bits + b.bits, a.pads + b.pads, a.wbytes + b.wbytes};
    }
};

__host__ __device__ __forceinline__ uint32_t ctl_bits(uint8_t c) { return (c & 31u) + 1u; }
__host__ __device__ __forceinline__ uint32_t ctl_pads(uint8_t c) { return (uint32_t)c >> 5; }

__host__ __device__ __forceinline__ Pos group_pos(uint8_t c, uint8_t wc, bool weighted)
{
    const uint32_t b = ctl_bits(c), pads = ctl_pads(c), real = 8u - pads;
    const uint32_t wb = (wc & 3u) ? (wc & 3u) : 4u;
    return Pos{(uint64_t)(real * b), (uint64_t)pads, weighted ? (uint64_t)(real * wb) : 0ull};
}

struct GroupToPos {  // group index -> its (payload bits, pads, weight bytes)
    const uint8_t *ctl, *wctl;
    int wuni;  // >= 0: every group's wctl (wctl unused)
    bool weighted;
    __device__ __forceinline__ Pos operator()(int64_t g) const
    {
        return group_pos(ctl[g], wuni >= 0 ? (uint8_t)wuni : (wctl ? wctl[g] : 0), weighted);
    }
};

__device__ __forceinline__ uint32_t bits_of(uint32_t d) { return d ? 32u - __clz(d) : 1u; }

__global__ void k_mark_row_starts(const int64_t *__restrict__ off, int64_t rows, uint8_t *__restrict__ start)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = off[r];
        if (off[r + 1] > a) start[a >> 3] = 1;
    }
}

// ctl byte per group (start[] holds the row-start flags, 0/1)
__global__ void k_pack_ctl(const int32_t *__restrict__ t, int64_t groups, uint32_t sentinel, uint8_t *__restrict__ ctl,
                           const uint8_t *__restrict__ start, int *__restrict__ bad)
{
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const bool rs = start[g] != 0;
        uint32_t prev = rs ? 0u : (uint32_t)t[8 * g - 1];
        uint32_t pads = 0, b = 1;
        for (int i = 0; i < 8; i++) {
            const uint32_t v = (uint32_t)t[8 * g + i];
            if (v == sentinel) {
                pads++;
                continue;
            }
            if (pads) atomicExch(bad, 1);  // a real arc after a pad: not the padded layout
            b = max(b, bits_of(v - prev));
            prev = v;
        }
        if (pads == 8) atomicExch(bad, 1);  // whole-pad group: not the padded layout
        ctl[g] = (uint8_t)((b - 1) | pads << 5);
    }
}

// OR the group's b-bit deltas into the zeroed payload words (neighbouring
// groups share boundary words)
__global__ void k_pack_payload(const int32_t *__restrict__ t, int64_t groups, const uint8_t *__restrict__ ctl,
                               const uint8_t *__restrict__ start, const Pos *__restrict__ pos,
                               uint32_t *__restrict__ payload)
{
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t c = ctl[g];
        const uint32_t b = ctl_bits(c), real = 8u - ctl_pads(c);
        uint64_t bp = pos[g].bits;
        uint32_t prev = start[g] ? 0u : (uint32_t)t[8 * g - 1];
        for (uint32_t i = 0; i < real; i++, bp += b) {
            const uint32_t v = (uint32_t)t[8 * g + i];
            const uint32_t d = v - prev;
            prev = v;
            const uint32_t sh = (uint32_t)(bp & 31u);
            uint32_t *wp = payload + (bp >> 5);
            atomicOr(wp, d << sh);
            if (sh && sh + b > 32u) atomicOr(wp + 1, d >> (32u - sh));
        }
    }
}

// Group fixed point: the smallest e (<= 63) with every real weight an integer
// multiple of 2^-e, and the bytes of the largest multiple; B = 0 (raw) when
// a weight is negative, -0.0, denormal, inf/nan or needs 4 bytes.
__device__ __forceinline__ uint32_t weight_ctl(const float *w, uint32_t real)
{
    int e = 0;
    bool ok = true;
    for (uint32_t i = 0; i < real; i++) {
        const uint32_t u = __float_as_uint(w[i]);
        if (u == 0u) continue;
        const uint32_t ef = u >> 23;  // sign bit set -> ef >= 256
        if (ef == 0u || ef >= 255u) {
            ok = false;
            continue;
        }
        const uint32_t sig = (u & 0x7fffffu) | 0x800000u;
        const int ei = 150 - (int)ef - (__ffs(sig) - 1);
        e = max(e, ei);
    }
    if (!ok || e > 63) return 0u;
    uint32_t kmax = 0;
    for (uint32_t i = 0; i < real; i++) {
        const uint32_t u = __float_as_uint(w[i]);
        if (u == 0u) continue;
        const int sh = (int)(u >> 23) - 150 + e;  // k = sig * 2^sh
        if (sh > 0) return 0u;                    // k >= 2^24
        kmax = max(kmax, ((u & 0x7fffffu) | 0x800000u) >> (-sh));
    }
    const uint32_t b = kmax < 0x100u ? 1u : kmax < 0x10000u ? 2u : kmax < 0x1000000u ? 3u : 0u;
    return b ? (b | (uint32_t)e << 2) : 0u;
}

__global__ void k_pack_wctl(const float *__restrict__ w, const uint8_t *__restrict__ ctl, int64_t groups,
                            uint8_t *__restrict__ wctl)
{
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x)
        wctl[g] = (uint8_t)weight_ctl(w + 8 * g, 8u - ctl_pads(ctl[g]));
}

__global__ void k_pack_wpayload(const float *__restrict__ w, const uint8_t *__restrict__ ctl,
                                const uint8_t *__restrict__ wctl, int64_t groups, const Pos *__restrict__ pos,
                                uint8_t *__restrict__ wpay)
{
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t real = 8u - ctl_pads(ctl[g]), wc = wctl[g], b = wc & 3u, e = wc >> 2;
        uint8_t *p = wpay + pos[g].wbytes;
        for (uint32_t i = 0; i < real; i++) {
            const uint32_t u = __float_as_uint(w[8 * g + i]);
            uint32_t v = u;
            if (b) v = u ? ((u & 0x7fffffu) | 0x800000u) >> (150 - (int)(u >> 23) - (int)e) : 0u;
            const uint32_t nb = b ? b : 4u;
            for (uint32_t q = 0; q < nb; q++) *p++ = (uint8_t)(v >> (8 * q));
        }
    }
}

__device__ __forceinline__ uint32_t ld_delta(const uint8_t *p, uint32_t w)
{
    uint32_t d = p[0];
    if (w > 1) d |= (uint32_t)p[1] << 8;
    if (w > 2) d |= (uint32_t)p[2] << 16;
    if (w > 3) d |= (uint32_t)p[3] << 24;
    return d;
}

// b-bit value at bit position bp of the payload stream (reads up to the
// word after the value's last word)
__device__ __forceinline__ uint32_t ld_bits(const uint32_t *__restrict__ p, uint64_t bp, uint32_t b)
{
    const uint32_t *wp = p + (bp >> 5);
    const uint32_t v = __funnelshift_r(__ldg(wp), __ldg(wp + 1), (uint32_t)(bp & 31u));
    return b == 32u ? v : v & ((1u << b) - 1u);
}

__global__ void __launch_bounds__(PT) k_unpack_sums(const uint8_t *__restrict__ ctl, const uint32_t *__restrict__ payload,
                                                    int64_t groups, const Pos *__restrict__ pos,
                                                    const uint8_t *__restrict__ start, SegSum *__restrict__ seg)
{
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t c = ctl[g];
        const uint32_t b = ctl_bits(c), real = 8u - ctl_pads(c);
        const uint64_t bp = pos[g].bits;
        uint32_t s = 0;
        for (uint32_t i = 0; i < real; i++) s += ld_bits(payload, bp + (uint64_t)i * b, b);
        seg[g] = SegSum{s, (uint32_t)start[g]};
    }
}

__global__ void __launch_bounds__(PT) k_unpack_rows(const uint8_t *__restrict__ ctl, const uint32_t *__restrict__ payload,
                                                    int64_t groups, const Pos *__restrict__ pos,
                                                    const uint8_t *__restrict__ start, const SegSum *__restrict__ last,
                                                    const uint8_t *__restrict__ wctl, int wuni,
                                                    const uint8_t *__restrict__ wpay, uint32_t sentinel,
                                                    int32_t *__restrict__ t, float *__restrict__ w_pad)
{
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t c = ctl[g];
        const uint32_t b = ctl_bits(c), real = 8u - ctl_pads(c);
        const Pos ps = pos[g];
        uint32_t v = (start[g] || g == 0) ? 0u : last[g - 1].val;
        uint32_t o[8];
#pragma unroll
        for (uint32_t i = 0; i < 8; i++) {
            if (i < real) {
                v += ld_bits(payload, ps.bits + (uint64_t)i * b, b);
                o[i] = v;
                GEE_DCHECK(v < sentinel);
            } else {
                o[i] = sentinel;
            }
        }
        int4 *tp = reinterpret_cast<int4 *>(t + 8 * g);
        __stcs(tp, make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]));
        __stcs(tp + 1, make_int4((int)o[4], (int)o[5], (int)o[6], (int)o[7]));
        if (w_pad) {
            const uint32_t wc = wuni >= 0 ? (uint32_t)wuni : wctl[g], wb = wc & 3u;
            const uint8_t *q = wpay + ps.wbytes;
            // w = k * 2^-e (exact: k < 2^24, e <= 63), or the raw bits
            const float scale = __uint_as_float((127u - (wc >> 2)) << 23);
            float x[8];
#pragma unroll
            for (uint32_t i = 0; i < 8; i++) {
                float v = 0.f;
                if (i < real) v = wb ? (float)ld_delta(q + i * wb, wb) * scale : __uint_as_float(ld_delta(q + 4 * i, 4));
                x[i] = v;
            }
            float4 *wp = reinterpret_cast<float4 *>(w_pad + 8 * g);
            __stcs(wp, make_float4(x[0], x[1], x[2], x[3]));
            __stcs(wp + 1, make_float4(x[4], x[5], x[6], x[7]));
        }
    }
}

inline int grid_of(int64_t items) { return (int)std::min<int64_t>((items + PT - 1) / PT, (int64_t)gee::sm_count() * 16); }

inline auto pos_iter(const uint8_t *ctl, const uint8_t *wctl, int wuni, bool weighted)
{
    return thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), GroupToPos{ctl, wctl, wuni, weighted});
}

size_t cub_scan_bytes(int64_t groups)
{
    size_t a = 0, b = 0;
    auto it = pos_iter(nullptr, nullptr, -1, false);
    cub::DeviceScan::ExclusiveScan(nullptr, a, it, (Pos *)nullptr, PosSum(), Pos{0, 0, 0}, groups);
    cub::DeviceScan::InclusiveScan(nullptr, b, (SegSum *)nullptr, (SegSum *)nullptr, SegOp(), groups);
    return std::max(a, b);
}

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

__global__ void k_widen_offsets(const int32_t *__restrict__ in, int64_t count, int64_t *__restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)__ldcs(in + i);
}

}  // namespace

extern "C" {

size_t gee_unpack_scratch_bytes(int64_t groups)
{
    if (groups <= 0) return 0;
    return align256((size_t)groups * sizeof(Pos)) + align256((size_t)groups * sizeof(SegSum)) +
           align256((size_t)groups) + align256(cub_scan_bytes(groups));
}

int gee_pack_targets(const int64_t *padded_offsets, int64_t rows, const int32_t *targets, const float *w_padded,
                     int64_t padded_arcs, int32_t sentinel, uint8_t *ctl, uint8_t *payload, int64_t *payload_bytes,
                     uint8_t *wctl, uint8_t *wpayload, int64_t *wpayload_bytes, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(rows >= 0 && padded_arcs >= 0 && (padded_arcs & 7) == 0, GEE_ERR_INVALID,
                "padded_arcs must be a nonnegative multiple of 8");
    GEE_REQUIRE(payload_bytes != nullptr, GEE_ERR_INVALID, "payload_bytes must not be NULL");
    *payload_bytes = 0;
    if (wpayload_bytes) *wpayload_bytes = 0;
    const int64_t groups = padded_arcs / 8;
    if (groups == 0) return GEE_OK;
    GEE_REQUIRE(padded_offsets && targets && ctl && payload, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(((uintptr_t)payload & 3) == 0, GEE_ERR_INVALID, "payload must be 4-byte aligned");
    GEE_REQUIRE(!w_padded || (wctl && wpayload && wpayload_bytes), GEE_ERR_INVALID,
                "weights need wctl, wpayload and wpayload_bytes");
    cudaStream_t st = gee::as_stream(stream);
    uint8_t *start = nullptr;
    Pos *pos = nullptr;
    int *bad = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = GEE_OK, hbad = 0;
    Pos tail[1];
    uint8_t last = 0, wlast = 0;
    Pos lp{0, 0, 0};
    auto it = pos_iter(ctl, w_padded ? wctl : nullptr, -1, w_padded != nullptr);
    auto fail = [&](int code, const char *msg) {
        gee::set_error("gee_pack_targets: %s", msg);
        rc = code;
    };
    if (cudaMallocAsync(&start, groups, st) != cudaSuccess || cudaMallocAsync(&pos, groups * sizeof(Pos), st) != cudaSuccess ||
        cudaMallocAsync(&bad, sizeof(int), st) != cudaSuccess) {
        fail(GEE_ERR_CUDA, "scratch alloc failed");
        goto out;
    }
    cudaMemsetAsync(start, 0, groups, st);
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    k_mark_row_starts<<<grid_of(rows), PT, 0, st>>>(padded_offsets, rows, start);
    k_pack_ctl<<<grid_of(groups), PT, 0, st>>>(targets, groups, (uint32_t)sentinel, ctl, start, bad);
    if (w_padded) k_pack_wctl<<<grid_of(groups), PT, 0, st>>>(w_padded, ctl, groups, wctl);
    cub::DeviceScan::ExclusiveScan(nullptr, tmp_bytes, it, pos, PosSum(), Pos{0, 0, 0}, groups, st);
    if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) {
        fail(GEE_ERR_CUDA, "scan scratch alloc failed");
        goto out;
    }
    cub::DeviceScan::ExclusiveScan(tmp, tmp_bytes, it, pos, PosSum(), Pos{0, 0, 0}, groups, st);
    cudaMemcpyAsync(tail, pos + groups - 1, sizeof(Pos), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&last, ctl + groups - 1, 1, cudaMemcpyDeviceToHost, st);
    if (w_padded) cudaMemcpyAsync(&wlast, wctl + groups - 1, 1, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        fail(GEE_ERR_CUDA, "sync failed");
        goto out;
    }
    if (hbad) {
        fail(GEE_ERR_INVALID, "targets are not in the padded layout (pads must end a row, < 8 per row)");
        goto out;
    }
    lp = group_pos(last, wlast, w_padded != nullptr);
    // whole u32 words of the bit stream (the payload buffer holds >= 4 * padded_arcs bytes)
    *payload_bytes = (int64_t)(((tail[0].bits + lp.bits + 31) >> 5) * 4);
    if (w_padded) *wpayload_bytes = (int64_t)(tail[0].wbytes + lp.wbytes);
    cudaMemsetAsync(payload, 0, (size_t)*payload_bytes, st);
    k_pack_payload<<<grid_of(groups), PT, 0, st>>>(targets, groups, ctl, start, pos, reinterpret_cast<uint32_t *>(payload));
    if (w_padded) k_pack_wpayload<<<grid_of(groups), PT, 0, st>>>(w_padded, ctl, wctl, groups, pos, wpayload);
    if ((rc = gee::check_launch("k_pack_payload"))) goto out;
    if (cudaStreamSynchronize(st) != cudaSuccess) fail(GEE_ERR_CUDA, "sync failed");
out:
    if (tmp) cudaFreeAsync(tmp, st);
    if (start) cudaFreeAsync(start, st);
    if (pos) cudaFreeAsync(pos, st);
    if (bad) cudaFreeAsync(bad, st);
    return rc;
}

int gee_unpack_targets(const uint8_t *ctl, const uint8_t *payload, int64_t groups, const int64_t *padded_offsets,
                       int64_t rows, const uint8_t *wctl, int32_t wctl_uniform, const uint8_t *wpayload,
                       int32_t sentinel, int32_t *targets, float *w_padded, void *scratch, size_t scratch_bytes,
                       void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(groups >= 0 && rows >= 0, GEE_ERR_INVALID, "groups and rows must be nonnegative");
    if (groups == 0) return GEE_OK;
    GEE_REQUIRE(wctl_uniform >= -1 && wctl_uniform <= 255, GEE_ERR_INVALID, "wctl_uniform must be -1 or a wctl byte");
    const bool weighted = w_padded != nullptr;
    GEE_REQUIRE(ctl && payload && padded_offsets && targets && scratch &&
                    (!weighted || (wpayload && (wctl || wctl_uniform >= 0))),
                GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(((uintptr_t)payload & 3) == 0, GEE_ERR_INVALID, "payload must be 4-byte aligned");
    GEE_REQUIRE(((uintptr_t)targets & 15) == 0 && (!w_padded || ((uintptr_t)w_padded & 15) == 0), GEE_ERR_INVALID,
                "targets / w_padded must be 16-byte aligned");
    GEE_REQUIRE(scratch_bytes >= gee_unpack_scratch_bytes(groups), GEE_ERR_INVALID,
                "scratch too small (gee_unpack_scratch_bytes)");
    cudaStream_t st = gee::as_stream(stream);
    auto *pos = static_cast<Pos *>(scratch);
    char *sp = static_cast<char *>(scratch) + align256((size_t)groups * sizeof(Pos));
    auto *seg = reinterpret_cast<SegSum *>(sp);
    sp += align256((size_t)groups * sizeof(SegSum));
    auto *start = reinterpret_cast<uint8_t *>(sp);
    void *tmp = sp + align256((size_t)groups);
    size_t tmp_bytes = cub_scan_bytes(groups);
    const int wuni = weighted ? (int)wctl_uniform : -1;
    const auto *pw = reinterpret_cast<const uint32_t *>(payload);
    GEE_CUDA(cudaMemsetAsync(start, 0, (size_t)groups, st));
    if (rows) k_mark_row_starts<<<grid_of(rows), PT, 0, st>>>(padded_offsets, rows, start);
    auto it = pos_iter(ctl, weighted ? wctl : nullptr, wuni, weighted);
    GEE_CUDA(cub::DeviceScan::ExclusiveScan(tmp, tmp_bytes, it, pos, PosSum(), Pos{0, 0, 0}, groups, st));
    k_unpack_sums<<<grid_of(groups), PT, 0, st>>>(ctl, pw, groups, pos, start, seg);
    int rc;
    if ((rc = gee::check_launch("k_unpack_sums"))) return rc;
    tmp_bytes = cub_scan_bytes(groups);
    GEE_CUDA(cub::DeviceScan::InclusiveScan(tmp, tmp_bytes, seg, seg, SegOp(), groups, st));
    k_unpack_rows<<<grid_of(groups), PT, 0, st>>>(ctl, pw, groups, pos, start, seg, weighted ? wctl : nullptr, wuni,
                                                  wpayload, (uint32_t)sentinel, targets, w_padded);
    return gee::check_launch("k_unpack_rows");
}

int gee_widen_offsets(const int32_t *in, int64_t count, int64_t *out, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(count >= 0, GEE_ERR_INVALID, "count must be nonnegative");
    if (count == 0) return GEE_OK;
    GEE_REQUIRE(in && out, GEE_ERR_INVALID, "NULL array argument");
    int64_t grid = (count + 255) / 256;
    if (grid > (int64_t)gee::sm_count() * 8) grid = (int64_t)gee::sm_count() * 8;
    k_widen_offsets<<<(int)grid, 256, 0, gee::as_stream(stream)>>>(in, count, out);
    return gee::check_launch("k_widen_offsets");
}

}  // extern "C"
