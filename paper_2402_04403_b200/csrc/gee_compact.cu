// Row-sparse form of Z for the device -> host copy of the streamed pass.
//
// The reference hands the caller a dense n x K embedding (embed_parallel's
// `out`, encoder.py:143-194).  On BASELINE C4 over 90% of Z's entries are
// zero (43% of the rows have no arcs, and a row of degree d fills at most
// min(d, K) classes), so HostPipeline ships each row chunk as
//     mask[r * mw + j]   u64, bit c of word j set iff Z[r, 64 j + c] != 0 (bit pattern)
//     vals[]             the nonzero values in row-major order
//     block_off[b]       index in vals of the first value of row b * GEE_ZC_BLOCK_ROWS
// and libgee_io's gee_io_expand_rows rebuilds the dense rows in the caller's
// host buffer.  Exact: every value crosses bit for bit (a -0.0 counts as
// nonzero), zeros are rewritten on the host.
//   k_zc_mask    one CTA per 1024-row block: ballots -> mask words, block count
//   k_zc_scan    exclusive scan of the block counts (one CTA)
//   k_zc_scatter one CTA per block: per-row popcount scan, then coalesced
//                re-read of the rows and packed stores of the nonzeros
#include "gee_common.cuh"

namespace {

constexpr int ZB = GEE_ZC_BLOCK_ROWS;  // rows per block (== threads of the scatter CTA)
constexpr int MT = 256;                // threads of the mask CTA

__global__ void __launch_bounds__(MT)
k_zc_mask(const float *__restrict__ z, int64_t rows, int32_t k, int32_t mw, unsigned long long *__restrict__ mask,
          int64_t *__restrict__ block_off)
{
    __shared__ int64_t part[MT / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * ZB;
    const int64_t r1 = r0 + ZB < rows ? r0 + ZB : rows;
    int64_t cnt = 0;
    for (int64_t r = r0 + wid; r < r1; r += MT / 32) {
        const uint32_t *zr = reinterpret_cast<const uint32_t *>(z) + r * k;
        for (int j = 0; j < mw; j++) {
            const int c0 = 64 * j + lane, c1 = c0 + 32;
            const uint32_t v0 = c0 < k ? __ldcs(zr + c0) : 0u;
            const uint32_t v1 = c1 < k ? __ldcs(zr + c1) : 0u;
            const uint32_t b0 = __ballot_sync(0xffffffffu, v0 != 0u);
            const uint32_t b1 = __ballot_sync(0xffffffffu, v1 != 0u);
            if (lane == 0) {
                mask[r * mw + j] = (unsigned long long)b0 | ((unsigned long long)b1 << 32);
                cnt += __popc(b0) + __popc(b1);
            }
        }
    }
    if (lane == 0) part[wid] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t s = 0;
        for (int i = 0; i < MT / 32; i++) s += part[i];
        block_off[blockIdx.x + 1] = s;
    }
}

// in-place exclusive scan: block_off[0] = 0, block_off[b + 1] holds block b's count
__global__ void __launch_bounds__(1024) k_zc_scan(int64_t *__restrict__ block_off, int64_t nblocks)
{
    __shared__ int64_t warp_sum[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0, block_off[0] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = 0; base < nblocks; base += 1024) {
        const int64_t i = base + threadIdx.x;
        int64_t v = i < nblocks ? block_off[i + 1] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += t;
        }
        if (lane == 31) warp_sum[wid] = v;
        __syncthreads();
        if (wid == 0) {
            int64_t ws = warp_sum[lane];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int64_t t = __shfl_up_sync(0xffffffffu, ws, d);
                if (lane >= d) ws += t;
            }
            warp_sum[lane] = ws;
        }
        __syncthreads();
        const int64_t incl = v + (wid ? warp_sum[wid - 1] : 0) + carry;
        if (i < nblocks) block_off[i + 1] = incl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = incl;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(ZB)
k_zc_scatter(const float *__restrict__ z, int64_t rows, int32_t k, int32_t mw,
             const unsigned long long *__restrict__ mask, const int64_t *__restrict__ block_off,
             float *__restrict__ vals)
{
    __shared__ int64_t row_off[ZB];
    __shared__ int64_t warp_sum[ZB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * ZB;
    const int64_t r1 = r0 + ZB < rows ? r0 + ZB : rows;
    // exclusive scan of the rows' popcounts within the block
    int64_t v = 0;
    if (r0 + threadIdx.x < r1)
        for (int j = 0; j < mw; j++) v += __popcll(mask[(r0 + threadIdx.x) * mw + j]);
    int64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += t;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t ws = warp_sum[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, ws, d);
            if (lane >= d) ws += t;
        }
        warp_sum[lane] = ws;
    }
    __syncthreads();
    row_off[threadIdx.x] = block_off[blockIdx.x] + x - v + (wid ? warp_sum[wid - 1] : 0);
    __syncthreads();
    // warps re-read their rows (coalesced) and pack the nonzeros
    for (int64_t r = r0 + wid; r < r1; r += ZB / 32) {
        const uint32_t *zr = reinterpret_cast<const uint32_t *>(z) + r * k;
        int64_t pos = row_off[r - r0];
        for (int j = 0; j < mw; j++) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int c = 64 * j + 32 * h + lane;
                const uint32_t val = c < k ? __ldcs(zr + c) : 0u;
                const uint32_t b = __ballot_sync(0xffffffffu, val != 0u);
                if (val) vals[pos + __popc(b & ((1u << lane) - 1u))] = __uint_as_float(val);
                pos += __popc(b);
            }
        }
    }
}

}  // namespace

extern "C" {

int64_t gee_zc_blocks(int64_t rows) { return rows <= 0 ? 0 : (rows + ZB - 1) / ZB; }

int gee_z_compact(const float *z, int64_t rows, int32_t k, unsigned long long *mask, int64_t *block_off, float *vals,
                  void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(rows >= 0 && k >= 1, GEE_ERR_INVALID, "rows must be >= 0 and k >= 1");
    GEE_REQUIRE(block_off != nullptr, GEE_ERR_INVALID, "block_off must not be NULL");
    cudaStream_t st = gee::as_stream(stream);
    const int64_t nb = gee_zc_blocks(rows);
    if (nb == 0) {
        GEE_CUDA(cudaMemsetAsync(block_off, 0, sizeof(int64_t), st));
        return GEE_OK;
    }
    GEE_REQUIRE(z && mask && vals, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(nb < INT32_MAX, GEE_ERR_RANGE, "too many rows");
    const int32_t mw = (k + 63) / 64;
    k_zc_mask<<<(unsigned)nb, MT, 0, st>>>(z, rows, k, mw, mask, block_off);
    if (int rc = gee::check_launch("k_zc_mask")) return rc;
    k_zc_scan<<<1, 1024, 0, st>>>(block_off, nb);
    if (int rc = gee::check_launch("k_zc_scan")) return rc;
    k_zc_scatter<<<(unsigned)nb, ZB, 0, st>>>(z, rows, k, mw, mask, block_off, vals);
    return gee::check_launch("k_zc_scatter");
}

}  // extern "C"
