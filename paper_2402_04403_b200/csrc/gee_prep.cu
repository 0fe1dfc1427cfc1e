// K5: graph preparation (outside the timed region, like the reference's
// build_csr, which bench.py:1-7 keeps out of its timers).
//
//   gee_build_sym_csr  symmetric CSR of a listed edge list: degree count,
//                      exclusive scan (CUB), atomic-cursor scatter.  The
//                      reference's counting sort is build_csr + csr_fill
//                      (graph.py:159-184, _kernels.py:229-238); here every
//                      list is mirrored because the edge pass applies both
//                      updates per listed edge (encoder.py:106-120).
//   gee_csr_rows       per-arc source row of a stored CSR (COO expansion).
//   gee_graph_stats    weight statistics that size the pull fixed point.
#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "gee_common.cuh"

namespace {

__global__ void k_degree(const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t s,
                         int64_t n, int symmetric, unsigned long long *__restrict__ deg,
                         unsigned long long *__restrict__ bad)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = src[i], v = dst[i];
        if (u < 0 || v < 0 || u >= n || v >= n) {
            atomicAdd(bad, 1ull);
            continue;
        }
        atomicAdd(&deg[u + 1], 1ull);
        if (symmetric) atomicAdd(&deg[v + 1], 1ull);
    }
}

// Unordered fill: atomic cursor per row (arc order within a row unspecified).
__global__ void k_scatter(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                          const float *__restrict__ w, int64_t s, int64_t n, int symmetric,
                          unsigned long long *__restrict__ cursor, int32_t *__restrict__ targets,
                          float *__restrict__ weights)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = src[i], v = dst[i];
        if (u < 0 || v < 0 || u >= n || v >= n) continue;
        unsigned long long pu = atomicAdd(&cursor[u], 1ull);
        targets[pu] = v;
        if (weights) weights[pu] = w[i];
        if (symmetric) {
            unsigned long long pv = atomicAdd(&cursor[v], 1ull);
            targets[pv] = u;
            if (weights) weights[pv] = w[i];
        }
    }
}

// Stable fill, step 1: arc a -> (row key, arc id).  Symmetric lists number
// the original arc 2i and its mirror 2i+1, so a stable sort by row gives
// build_csr's order: mirror right after the original (graph.py:170-176).
__global__ void k_arc_keys(const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t s,
                           int symmetric, uint32_t *__restrict__ keys, uint32_t *__restrict__ ids)
{
    const int64_t arcs = symmetric ? 2 * s : s;
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < arcs;
         a += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = symmetric ? a >> 1 : a;
        const bool mirror = symmetric && (a & 1);
        keys[a] = (uint32_t)(mirror ? dst[i] : src[i]);
        ids[a] = (uint32_t)a;
    }
}

// Stable fill, step 2: gather targets/weights in sorted arc order.
__global__ void k_arc_gather(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                             const float *__restrict__ w, int64_t arcs, int symmetric,
                             const uint32_t *__restrict__ ids, int32_t *__restrict__ targets,
                             float *__restrict__ weights)
{
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < arcs;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = ids[p];
        const int64_t i = symmetric ? a >> 1 : a;
        const bool mirror = symmetric && (a & 1);
        targets[p] = mirror ? src[i] : dst[i];
        if (weights) weights[p] = w[i];
    }
}

// Row-range shard of the symmetric CSR: keep arcs whose row is in [lo, hi).
__global__ void k_scatter_rows(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                               const float *__restrict__ w, int64_t s, int64_t lo, int64_t hi,
                               unsigned long long *__restrict__ cursor, int32_t *__restrict__ targets,
                               float *__restrict__ weights)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = src[i], v = dst[i];
        if (u >= lo && u < hi) {
            unsigned long long p = atomicAdd(&cursor[u - lo], 1ull);
            targets[p] = v;
            if (weights) weights[p] = w[i];
        }
        if (v >= lo && v < hi) {
            unsigned long long p = atomicAdd(&cursor[v - lo], 1ull);
            targets[p] = u;
            if (weights) weights[p] = w[i];
        }
    }
}

__global__ void k_rebase(const int64_t *__restrict__ full, int64_t lo, int64_t rows, int64_t *__restrict__ local,
                         unsigned long long *__restrict__ cursor)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = full[lo + r] - full[lo];
        local[r] = v;
        if (r < rows) cursor[r] = (unsigned long long)v;
    }
}

__global__ void k_csr_rows(const int64_t *__restrict__ offsets, int64_t n, int32_t *__restrict__ rows)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; r < n; r += warps) {
        const int64_t lo = offsets[r], hi = offsets[r + 1];
        for (int64_t e = lo + lane; e < hi; e += 32) rows[e] = (int32_t)r;
    }
}

// Non-negative doubles / floats order like their bit patterns.
__device__ __forceinline__ void atomic_max_pos(double *p, double v)
{
    atomicMax(reinterpret_cast<unsigned long long *>(p), (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_min_pos(double *p, double v)
{
    atomicMin(reinterpret_cast<unsigned long long *>(p), (unsigned long long)__double_as_longlong(v));
}

struct Stats {
    double max_row_abs;
    double min_abs_nz;
    double max_abs;
    int32_t nonfinite;
};

__global__ void k_graph_stats(const int64_t *__restrict__ offsets, const float *__restrict__ w, int64_t n,
                              Stats *__restrict__ out)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double best_row = 0.0, best_min = INFINITY, best_max = 0.0;
    int nonfinite = 0;
    for (int64_t r = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; r < n; r += warps) {
        const int64_t lo = offsets[r], hi = offsets[r + 1];
        double sum = 0.0;
        if (w) {
            for (int64_t e = lo + lane; e < hi; e += 32) {
                float x = fabsf(w[e]);
                if (!isfinite(x)) nonfinite = 1;
                sum += x;
                if (x > 0.f) best_min = fmin(best_min, (double)x);
                best_max = fmax(best_max, (double)x);
            }
            for (int d = 16; d; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
        } else {
            sum = (double)(hi - lo);
        }
        best_row = fmax(best_row, sum);
    }
    for (int d = 16; d; d >>= 1) {
        best_row = fmax(best_row, __shfl_xor_sync(0xffffffffu, best_row, d));
        best_min = fmin(best_min, __shfl_xor_sync(0xffffffffu, best_min, d));
        best_max = fmax(best_max, __shfl_xor_sync(0xffffffffu, best_max, d));
        nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, d);
    }
    if (lane == 0) {
        atomic_max_pos(&out->max_row_abs, best_row);
        if (best_min < INFINITY) atomic_min_pos(&out->min_abs_nz, best_min);
        atomic_max_pos(&out->max_abs, best_max);
        if (nonfinite) atomicOr(&out->nonfinite, 1);
    }
}

int grid_for(int64_t items, int per_block, int waves)
{
    int64_t want = (items + per_block - 1) / per_block;
    int64_t cap = (int64_t)gee::sm_count() * waves;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// first row r in [0, n] with offsets[r] >= target, one thread per target
__global__ void k_row_bounds(const int64_t *__restrict__ offsets, int64_t n, int64_t step, int64_t m,
                             int64_t *__restrict__ rows)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j > m) return;
    const int64_t t = j * step;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (offsets[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    rows[j] = j == m ? n : lo;
}

__global__ void k_rebase(const int64_t *__restrict__ offsets, int64_t r0, int64_t rows, int32_t *__restrict__ out)
{
    const int64_t base = offsets[r0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= rows; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)(offsets[r0 + i] - base);
}

// padded offsets: pout[r+1] = round_up(offsets[r+1] - offsets[r], align)
__global__ void k_pad_degrees(const int64_t *__restrict__ offsets, int64_t n, int64_t align, int64_t *__restrict__ pout)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = offsets[r + 1] - offsets[r];
        pout[r + 1] = (d + align - 1) / align * align;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) pout[0] = 0;
}

// one warp per row: copy its arcs, then fill the pad with (sentinel, 0)
__global__ void k_pad_copy(const int64_t *__restrict__ offsets, const int64_t *__restrict__ poff, int64_t n,
                           const int32_t *__restrict__ tin, const float *__restrict__ win, int32_t sentinel,
                           int32_t *__restrict__ tout, float *__restrict__ wout)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t GW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = gw; r < n; r += GW) {
        const int64_t a0 = offsets[r], d = offsets[r + 1] - a0;
        const int64_t b0 = poff[r], pd = poff[r + 1] - b0;
        for (int64_t j = lane; j < pd; j += 32) {
            const bool in = j < d;
            tout[b0 + j] = in ? tin[a0 + j] : sentinel;
            if (wout) wout[b0 + j] = in ? win[a0 + j] : 0.f;
        }
    }
}

}  // namespace

extern "C" {

int gee_build_csr(const int32_t *src, const int32_t *dst, const float *w, int64_t s, int64_t n,
                  int32_t symmetric, int32_t stable, int64_t *offsets, int32_t *targets, float *weights,
                  void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && s >= 0, GEE_ERR_INVALID, "n and s must be nonnegative");
    GEE_REQUIRE(n <= INT32_MAX, GEE_ERR_INVALID, "node count %lld exceeds CSR limit", (long long)n);
    GEE_REQUIRE(offsets != nullptr, GEE_ERR_INVALID, "offsets must not be NULL");
    const int64_t arcs = symmetric ? 2 * s : s;
    GEE_REQUIRE(!stable || arcs <= (int64_t)UINT32_MAX, GEE_ERR_INVALID,
                "stable CSR build supports at most 2^32-1 arcs");
    cudaStream_t st = gee::as_stream(stream);
    auto *deg = reinterpret_cast<unsigned long long *>(offsets);
    GEE_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (size_t)(n + 1), st));
    if (s == 0) return GEE_OK;
    GEE_REQUIRE(src && dst && targets, GEE_ERR_INVALID, "NULL array argument");
    GEE_REQUIRE(!w || weights, GEE_ERR_INVALID, "weights output required for weighted input");
    unsigned long long *bad = nullptr, *cursor = nullptr;
    uint32_t *kbuf = nullptr, *vbuf = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = GEE_OK;
    unsigned long long nbad = 0;
    GEE_CUDA(cudaMallocAsync((void **)&bad, sizeof(unsigned long long), st));
    GEE_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st));
    k_degree<<<grid_for(s, 256, 16), 256, 0, st>>>(src, dst, s, n, symmetric, deg, bad);
    if ((rc = gee::check_launch("k_degree"))) goto out;
    cudaMemcpyAsync(&nbad, bad, sizeof(nbad), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) { gee::set_error("sync failed"); rc = GEE_ERR_CUDA; goto out; }
    if (nbad) {
        gee::set_error("%llu edge endpoints outside [0, %lld)", nbad, (long long)n);
        rc = GEE_ERR_RANGE;
        goto out;
    }
    // inclusive scan of deg[1..n] in place gives offsets (offsets[0] = 0)
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, offsets + 1, offsets + 1, n, st);
    if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) { gee::set_error("scratch alloc failed"); rc = GEE_ERR_CUDA; goto out; }
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, offsets + 1, offsets + 1, n, st);
    if ((rc = gee::check_launch("DeviceScan::InclusiveSum"))) goto out;
    cudaFreeAsync(tmp, st);
    tmp = nullptr;
    if (!stable) {
        if (cudaMallocAsync((void **)&cursor, sizeof(unsigned long long) * (size_t)(n ? n : 1), st) != cudaSuccess) {
            gee::set_error("cursor alloc failed");
            rc = GEE_ERR_CUDA;
            goto out;
        }
        cudaMemcpyAsync(cursor, offsets, sizeof(int64_t) * (size_t)n, cudaMemcpyDeviceToDevice, st);
        k_scatter<<<grid_for(s, 256, 16), 256, 0, st>>>(src, dst, w, s, n, symmetric, cursor, targets,
                                                        w ? weights : nullptr);
        rc = gee::check_launch("k_scatter");
        goto out;
    }
    {
        // 4 buffers of `arcs` u32: keys/ids in, keys/ids out (cub::DoubleBuffer)
        if (cudaMallocAsync((void **)&kbuf, sizeof(uint32_t) * (size_t)arcs * 2, st) != cudaSuccess ||
            cudaMallocAsync((void **)&vbuf, sizeof(uint32_t) * (size_t)arcs * 2, st) != cudaSuccess) {
            gee::set_error("sort buffers alloc failed (%lld arcs)", (long long)arcs);
            rc = GEE_ERR_CUDA;
            goto out;
        }
        k_arc_keys<<<grid_for(arcs, 256, 16), 256, 0, st>>>(src, dst, s, symmetric, kbuf, vbuf);
        if ((rc = gee::check_launch("k_arc_keys"))) goto out;
        cub::DoubleBuffer<uint32_t> kd(kbuf, kbuf + arcs), vd(vbuf, vbuf + arcs);
        int end_bit = 1;
        while (end_bit < 32 && ((int64_t)1 << end_bit) < n) end_bit++;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kd, vd, arcs, 0, end_bit, st);
        if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) { gee::set_error("sort scratch alloc failed"); rc = GEE_ERR_CUDA; goto out; }
        cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kd, vd, arcs, 0, end_bit, st);
        if ((rc = gee::check_launch("DeviceRadixSort::SortPairs"))) goto out;
        k_arc_gather<<<grid_for(arcs, 256, 16), 256, 0, st>>>(src, dst, w, arcs, symmetric, vd.Current(), targets,
                                                              w ? weights : nullptr);
        rc = gee::check_launch("k_arc_gather");
    }
out:
    if (tmp) cudaFreeAsync(tmp, st);
    if (cursor) cudaFreeAsync(cursor, st);
    if (kbuf) cudaFreeAsync(kbuf, st);
    if (vbuf) cudaFreeAsync(vbuf, st);
    if (bad) cudaFreeAsync(bad, st);
    return rc;
}

int gee_build_sym_csr(const int32_t *src, const int32_t *dst, const float *w, int64_t s, int64_t n,
                      int64_t *offsets, int32_t *targets, float *weights, void *stream)
{
    return gee_build_csr(src, dst, w, s, n, 1, 0, offsets, targets, weights, stream);
}

int gee_sym_offsets(const int32_t *src, const int32_t *dst, int64_t s, int64_t n, int64_t *offsets,
                    void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && s >= 0, GEE_ERR_INVALID, "n and s must be nonnegative");
    GEE_REQUIRE(offsets != nullptr, GEE_ERR_INVALID, "offsets must not be NULL");
    cudaStream_t st = gee::as_stream(stream);
    GEE_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (size_t)(n + 1), st));
    if (s == 0 || n == 0) return GEE_OK;
    unsigned long long *bad = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    unsigned long long nbad = 0;
    int rc = GEE_OK;
    GEE_CUDA(cudaMallocAsync((void **)&bad, sizeof(unsigned long long), st));
    GEE_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st));
    k_degree<<<grid_for(s, 256, 16), 256, 0, st>>>(src, dst, s, n, 1, reinterpret_cast<unsigned long long *>(offsets),
                                                   bad);
    if ((rc = gee::check_launch("k_degree"))) goto out;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, offsets + 1, offsets + 1, n, st);
    if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) { gee::set_error("scratch alloc failed"); rc = GEE_ERR_CUDA; goto out; }
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, offsets + 1, offsets + 1, n, st);
    if ((rc = gee::check_launch("DeviceScan::InclusiveSum"))) goto out;
    cudaMemcpyAsync(&nbad, bad, sizeof(nbad), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) { gee::set_error("sync failed"); rc = GEE_ERR_CUDA; goto out; }
    if (nbad) {
        gee::set_error("%llu edge endpoints outside [0, %lld)", nbad, (long long)n);
        rc = GEE_ERR_RANGE;
    }
out:
    if (tmp) cudaFreeAsync(tmp, st);
    if (bad) cudaFreeAsync(bad, st);
    return rc;
}

int gee_build_sym_csr_rows(const int32_t *src, const int32_t *dst, const float *w, int64_t s, int64_t n,
                           int64_t row_lo, int64_t row_hi, const int64_t *full_offsets, int64_t *offsets,
                           int32_t *targets, float *weights, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(0 <= row_lo && row_lo <= row_hi && row_hi <= n, GEE_ERR_INVALID, "row range [%lld, %lld) outside [0, %lld]",
                (long long)row_lo, (long long)row_hi, (long long)n);
    GEE_REQUIRE(full_offsets && offsets, GEE_ERR_INVALID, "offsets must not be NULL");
    cudaStream_t st = gee::as_stream(stream);
    const int64_t rows = row_hi - row_lo;
    unsigned long long *cursor = nullptr;
    GEE_CUDA(cudaMallocAsync((void **)&cursor, sizeof(unsigned long long) * (size_t)(rows ? rows : 1), st));
    k_rebase<<<grid_for(rows + 1, 256, 16), 256, 0, st>>>(full_offsets, row_lo, rows, offsets, cursor);
    int rc = gee::check_launch("k_rebase");
    if (!rc && s > 0 && rows > 0) {
        k_scatter_rows<<<grid_for(s, 256, 16), 256, 0, st>>>(src, dst, w, s, row_lo, row_hi, cursor, targets,
                                                             w ? weights : nullptr);
        rc = gee::check_launch("k_scatter_rows");
    }
    cudaFreeAsync(cursor, st);
    return rc;
}

int gee_csr_rows(const int64_t *offsets, int64_t n, int64_t arcs, int32_t *rows, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && arcs >= 0, GEE_ERR_INVALID, "n and arcs must be nonnegative");
    if (n == 0 || arcs == 0) return GEE_OK;
    cudaStream_t st = gee::as_stream(stream);
    k_csr_rows<<<grid_for(n * 32, 256, 16), 256, 0, st>>>(offsets, n, rows);
    return gee::check_launch("k_csr_rows");
}

int gee_graph_stats(const int64_t *offsets, const float *w, int64_t n, int64_t arcs, double *max_row_abs,
                    double *min_abs_nz, double *max_abs, int32_t *nonfinite, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && arcs >= 0, GEE_ERR_INVALID, "n and arcs must be nonnegative");
    Stats h{0.0, INFINITY, 0.0, 0};
    if (n > 0 && arcs > 0) {
        cudaStream_t st = gee::as_stream(stream);
        Stats *d = nullptr;
        GEE_CUDA(cudaMallocAsync((void **)&d, sizeof(Stats), st));
        cudaMemcpyAsync(d, &h, sizeof(Stats), cudaMemcpyHostToDevice, st);
        k_graph_stats<<<grid_for(n * 32, 256, 16), 256, 0, st>>>(offsets, w, n, d);
        int rc = gee::check_launch("k_graph_stats");
        cudaMemcpyAsync(&h, d, sizeof(Stats), cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(d, st);
        GEE_CUDA(cudaStreamSynchronize(st));
        if (rc) return rc;
    }
    if (max_row_abs) *max_row_abs = h.max_row_abs;
    if (min_abs_nz) *min_abs_nz = h.min_abs_nz == INFINITY ? 0.0 : h.min_abs_nz;
    if (max_abs) *max_abs = h.max_abs;
    if (nonfinite) *nonfinite = h.nonfinite;
    return GEE_OK;
}

int gee_sort_rows(const int64_t *offsets, int64_t n, int32_t *targets, float *w, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0, GEE_ERR_INVALID, "n must be nonnegative");
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && targets, GEE_ERR_INVALID, "NULL array argument");
    cudaStream_t st = gee::as_stream(stream);
    int64_t arcs = 0;
    GEE_CUDA(cudaMemcpyAsync(&arcs, offsets + n, sizeof(arcs), cudaMemcpyDeviceToHost, st));
    GEE_CUDA(cudaStreamSynchronize(st));
    if (arcs == 0) return GEE_OK;
    // row chunks of at most STEP arcs (plus one row) for the int-sized CUB calls
    const int64_t STEP = (int64_t)1 << 29;
    const int64_t m = (arcs + STEP - 1) / STEP;
    int64_t *d_rows = nullptr;
    int32_t *d_off = nullptr, *k_out = nullptr;
    float *v_out = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    std::vector<int64_t> rows(m + 1);
    int rc = GEE_OK;
    int64_t max_rows = 0, max_arcs = 0;
    auto fail = [&](const char *what) {
        gee::set_error("%s", what);
        rc = GEE_ERR_CUDA;
    };
    if (cudaMallocAsync((void **)&d_rows, sizeof(int64_t) * (m + 1), st) != cudaSuccess) {
        fail("gee_sort_rows: alloc failed");
        goto out;
    }
    k_row_bounds<<<(int)((m + 1 + 255) / 256), 256, 0, st>>>(offsets, n, STEP, m, d_rows);
    if ((rc = gee::check_launch("k_row_bounds"))) goto out;
    cudaMemcpyAsync(rows.data(), d_rows, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        fail("gee_sort_rows: sync failed");
        goto out;
    }
    {
        std::vector<int64_t> off_h(m + 1);
        for (int64_t j = 0; j <= m; j++)
            cudaMemcpyAsync(&off_h[j], offsets + rows[j], sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        for (int64_t j = 0; j < m; j++) {
            max_rows = std::max(max_rows, rows[j + 1] - rows[j]);
            max_arcs = std::max(max_arcs, off_h[j + 1] - off_h[j]);
        }
        GEE_REQUIRE(max_arcs < INT32_MAX, GEE_ERR_RANGE, "a row exceeds 2^31 arcs");
        if (cudaMallocAsync((void **)&d_off, sizeof(int32_t) * (max_rows + 1), st) != cudaSuccess ||
            cudaMallocAsync((void **)&k_out, sizeof(int32_t) * max_arcs, st) != cudaSuccess ||
            (w && cudaMallocAsync((void **)&v_out, sizeof(float) * max_arcs, st) != cudaSuccess)) {
            fail("gee_sort_rows: scratch alloc failed");
            goto out;
        }
        for (int64_t j = 0; j < m; j++) {
            const int64_t r0 = rows[j], nr = rows[j + 1] - rows[j];
            const int64_t a0 = off_h[j], na = off_h[j + 1] - off_h[j];
            if (nr == 0 || na == 0) continue;
            k_rebase<<<(int)std::min<int64_t>((nr + 256) / 256, 4096), 256, 0, st>>>(offsets, r0, nr, d_off);
            if ((rc = gee::check_launch("k_rebase"))) goto out;
            size_t need = 0;
            if (w)
                cub::DeviceSegmentedSort::StableSortPairs(nullptr, need, targets + a0, k_out, w + a0, v_out, (int)na,
                                                          (int)nr, d_off, d_off + 1, st);
            else
                cub::DeviceSegmentedSort::StableSortKeys(nullptr, need, targets + a0, k_out, (int)na, (int)nr, d_off,
                                                         d_off + 1, st);
            if (need > tmp_bytes) {
                if (tmp) cudaFreeAsync(tmp, st);
                tmp = nullptr;
                if (cudaMallocAsync(&tmp, need, st) != cudaSuccess) {
                    fail("gee_sort_rows: sort scratch alloc failed");
                    goto out;
                }
                tmp_bytes = need;
            }
            cudaError_t e;
            if (w)
                e = cub::DeviceSegmentedSort::StableSortPairs(tmp, need, targets + a0, k_out, w + a0, v_out, (int)na,
                                                              (int)nr, d_off, d_off + 1, st);
            else
                e = cub::DeviceSegmentedSort::StableSortKeys(tmp, need, targets + a0, k_out, (int)na, (int)nr, d_off,
                                                             d_off + 1, st);
            if (e != cudaSuccess) {
                fail("gee_sort_rows: segmented sort failed");
                goto out;
            }
            cudaMemcpyAsync(targets + a0, k_out, sizeof(int32_t) * na, cudaMemcpyDeviceToDevice, st);
            if (w) cudaMemcpyAsync(w + a0, v_out, sizeof(float) * na, cudaMemcpyDeviceToDevice, st);
        }
        if ((rc = gee::check_launch("gee_sort_rows"))) goto out;
    }
out:
    if (tmp) cudaFreeAsync(tmp, st);
    if (d_rows) cudaFreeAsync(d_rows, st);
    if (d_off) cudaFreeAsync(d_off, st);
    if (k_out) cudaFreeAsync(k_out, st);
    if (v_out) cudaFreeAsync(v_out, st);
    if (rc == GEE_OK && cudaStreamSynchronize(st) != cudaSuccess) {
        gee::set_error("gee_sort_rows: sync failed");
        rc = GEE_ERR_CUDA;
    }
    return rc;
}

int gee_pad_offsets(const int64_t *offsets, int64_t n, int64_t align, int64_t *padded_offsets, int64_t *padded_arcs,
                    void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && align >= 1, GEE_ERR_INVALID, "bad n / align");
    GEE_REQUIRE(offsets && padded_offsets && padded_arcs, GEE_ERR_INVALID, "NULL argument");
    cudaStream_t st = gee::as_stream(stream);
    *padded_arcs = 0;
    if (n == 0) {
        GEE_CUDA(cudaMemsetAsync(padded_offsets, 0, sizeof(int64_t), st));
        return GEE_OK;
    }
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)gee::sm_count() * 16);
    k_pad_degrees<<<grid, 256, 0, st>>>(offsets, n, align, padded_offsets);
    int rc;
    if ((rc = gee::check_launch("k_pad_degrees"))) return rc;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, padded_offsets + 1, padded_offsets + 1, n, st);
    GEE_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, padded_offsets + 1, padded_offsets + 1, n, st);
    cudaFreeAsync(tmp, st);
    if ((rc = gee::check_launch("DeviceScan::InclusiveSum"))) return rc;
    GEE_CUDA(cudaMemcpyAsync(padded_arcs, padded_offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GEE_CUDA(cudaStreamSynchronize(st));
    return GEE_OK;
}

int gee_pad_rows(const int64_t *offsets, const int64_t *padded_offsets, int64_t n, const int32_t *targets,
                 const float *w, int32_t sentinel, int32_t *padded_targets, float *padded_w, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0, GEE_ERR_INVALID, "n must be nonnegative");
    if (n == 0) return GEE_OK;
    GEE_REQUIRE(offsets && padded_offsets && targets && padded_targets && (!w || padded_w), GEE_ERR_INVALID,
                "NULL array argument");
    const int grid = (int)std::min<int64_t>((n * 32 + 255) / 256, (int64_t)gee::sm_count() * 16);
    k_pad_copy<<<grid, 256, 0, gee::as_stream(stream)>>>(offsets, padded_offsets, n, targets, w, sentinel,
                                                         padded_targets, w ? padded_w : nullptr);
    return gee::check_launch("k_pad_copy");
}

}  // extern "C"
