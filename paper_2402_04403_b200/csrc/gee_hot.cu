// Hot-label tier (graph preparation, outside the timed region).
//
// R-MAT-like graphs concentrate label lookups on few vertices: at the C4
// configuration (scale 27) the top 6% of vertices by degree take 91% of the
// 3.6e9 lookups of a pass, the top 12% take 96%.  The pull pass gathers one
// label per arc, and random gathers into the full packed label array
// (107 MB at K=50) miss L2 (measured 36% hit rate; profiles/).
//
// gee_hot_plan ranks vertices by symmetric degree (stable radix sort,
// descending; ties by vertex id) and keeps the top `max_hot` with degree >=
// min_degree; gee_hot_encode rewrites CSR targets into label-table slots
// (rank for hot vertices, n_hot + v otherwise).  In the timed region
// gee_build_projection also writes the hot vertices' labels at their ranks:
// a dense prefix of the label table that stays in L2, and whose head each
// pull CTA stages in shared memory.
#include <cub/device/device_radix_sort.cuh>

#include "gee_common.cuh"

namespace {

__global__ void k_degree_keys(const int64_t *__restrict__ offsets, int64_t n, uint32_t *__restrict__ keys,
                              int32_t *__restrict__ ids)
{
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = offsets[v + 1] - offsets[v];
        keys[v] = d > 0xffffffffll ? 0xffffffffu : (uint32_t)d;
        ids[v] = (int32_t)v;
        }
}

__global__ void k_fill_i32(int32_t *__restrict__ a, int64_t n, int32_t v)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

// first index r < limit with keys[r] < min_degree (keys sorted descending)
__global__ void k_count_hot(const uint32_t *__restrict__ keys, int64_t limit, uint32_t min_degree,
                            unsigned long long *__restrict__ first_cold)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < limit; r += (int64_t)gridDim.x * blockDim.x)
        if (keys[r] < min_degree && (r == 0 || keys[r - 1] >= min_degree)) atomicMin(first_cold, (unsigned long long)r);
}

__global__ void k_assign_ranks(const int32_t *__restrict__ sorted_ids, const unsigned long long *__restrict__ n_hot,
                               int32_t *__restrict__ hot_rank, int32_t *__restrict__ hot_vertex)
{
    const int64_t h = (int64_t)*n_hot;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < h; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = sorted_ids[r];
        hot_rank[v] = (int32_t)r;
        if (hot_vertex) hot_vertex[r] = v;
    }
}

__global__ void k_hot_encode(int32_t *__restrict__ targets, int64_t arcs, const int32_t *__restrict__ hot_rank,
                             int32_t n_hot)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < arcs; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t = targets[e];
        const int32_t r = hot_rank[t];
        targets[e] = r >= 0 ? r : n_hot + t;
    }
}

int grid_for(int64_t items)
{
    int64_t want = (items + 255) / 256;
    int64_t cap = (int64_t)gee::sm_count() * 16;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" {

int gee_hot_plan(const int64_t *offsets, int64_t n, int64_t max_hot, int64_t min_degree, int32_t *hot_rank,
                 int32_t *hot_vertex, int64_t *n_hot, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 0 && max_hot >= 0, GEE_ERR_INVALID, "n and max_hot must be nonnegative");
    GEE_REQUIRE(n <= INT32_MAX, GEE_ERR_INVALID, "node count exceeds int32");
    GEE_REQUIRE(offsets && hot_rank && n_hot, GEE_ERR_INVALID, "NULL array argument");
    cudaStream_t st = gee::as_stream(stream);
    *n_hot = 0;
    if (n == 0) return GEE_OK;
    k_fill_i32<<<grid_for(n), 256, 0, st>>>(hot_rank, n, -1);
    int rc = gee::check_launch("k_fill_i32");
    if (rc || max_hot == 0) return rc;
    uint32_t *keys = nullptr;
    int32_t *ids = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    unsigned long long *d_first = nullptr;
    unsigned long long first = 0;
    const int64_t limit = max_hot < n ? max_hot : n;
    if (cudaMallocAsync((void **)&keys, sizeof(uint32_t) * (size_t)n * 2, st) != cudaSuccess ||
        cudaMallocAsync((void **)&ids, sizeof(int32_t) * (size_t)n * 2, st) != cudaSuccess ||
        cudaMallocAsync((void **)&d_first, sizeof(unsigned long long), st) != cudaSuccess) {
        gee::set_error("hot plan scratch alloc failed");
        rc = GEE_ERR_CUDA;
        goto out;
    }
    k_degree_keys<<<grid_for(n), 256, 0, st>>>(offsets, n, keys, ids);
    if ((rc = gee::check_launch("k_degree_keys"))) goto out;
    {
        cub::DoubleBuffer<uint32_t> kd(keys, keys + n);
        cub::DoubleBuffer<int32_t> vd(ids, ids + n);
        cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, kd, vd, n, 0, 32, st);
        if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) {
            gee::set_error("hot plan sort scratch alloc failed");
            rc = GEE_ERR_CUDA;
            goto out;
        }
        cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, kd, vd, n, 0, 32, st);
        if ((rc = gee::check_launch("SortPairsDescending"))) goto out;
        first = (unsigned long long)limit;
        cudaMemcpyAsync(d_first, &first, sizeof(first), cudaMemcpyHostToDevice, st);
        const uint32_t md = min_degree < 0 ? 0u : (min_degree > 0xffffffffll ? 0xffffffffu : (uint32_t)min_degree);
        k_count_hot<<<grid_for(limit), 256, 0, st>>>(kd.Current(), limit, md, d_first);
        if ((rc = gee::check_launch("k_count_hot"))) goto out;
        k_assign_ranks<<<grid_for(limit), 256, 0, st>>>(vd.Current(), d_first, hot_rank, hot_vertex);
        if ((rc = gee::check_launch("k_assign_ranks"))) goto out;
        cudaMemcpyAsync(&first, d_first, sizeof(first), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) {
            gee::set_error("hot plan sync failed");
            rc = GEE_ERR_CUDA;
            goto out;
        }
        *n_hot = (int64_t)first;
    }
out:
    if (tmp) cudaFreeAsync(tmp, st);
    if (keys) cudaFreeAsync(keys, st);
    if (ids) cudaFreeAsync(ids, st);
    if (d_first) cudaFreeAsync(d_first, st);
    return rc;
}

int gee_hot_encode(int32_t *targets, int64_t arcs, const int32_t *hot_rank, int64_t n_hot, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(arcs >= 0 && n_hot >= 0 && n_hot < INT32_MAX, GEE_ERR_INVALID, "bad arcs / n_hot");
    if (arcs == 0) return GEE_OK;
    GEE_REQUIRE(targets && hot_rank, GEE_ERR_INVALID, "NULL array argument");
    k_hot_encode<<<grid_for(arcs), 256, 0, gee::as_stream(stream)>>>(targets, arcs, hot_rank, (int32_t)n_hot);
    return gee::check_launch("k_hot_encode");
}

}  // extern "C"
