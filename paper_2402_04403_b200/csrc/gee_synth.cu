// Seeded synthetic inputs for the benchmark configurations (harness, not
// the edge pass).  Counter-based: element i of a stream is a pure function
// of (seed, i), so tests restate any element in numpy
// (paper_2402_04403_b200/synth.py) and a shard of a graph can be generated
// on its own.
//
//   R-MAT(a, b, c, d) (Chakrabarti et al.; Graph500 convention): `scale`
//   quadrant choices per edge, then a seeded bijective scramble of vertex
//   ids.  Self-loops and duplicates are kept (reference SPEC.md:102).
//   Erdos-Renyi G(n, s) with replacement, as generate_erdos_renyi
//   (reference graph.py:187-201).  Weights are fp32 1 - U[0,1) with 24-bit
//   U, i.e. in (0, 1].  Uniform labels in {1..k}.
#include "../../include/gee_synth.h"
#include "gee_common.cuh"

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Stream word `ctr` of stream `tag` under `seed`.
__host__ __device__ __forceinline__ uint64_t rnd(uint64_t seed, uint64_t tag, uint64_t ctr)
{
    return splitmix64(splitmix64(seed ^ (tag * 0xD1B54A32D192ED03ull)) + ctr);
}

// Bijective scramble of [0, 2^scale): odd multiply / xorshift rounds.
__device__ __forceinline__ uint64_t scramble(uint64_t x, int scale, uint64_t m1, uint64_t m2)
{
    const uint64_t mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1);
    const int h = scale / 2 > 0 ? scale / 2 : 1;
    x = (x * m1) & mask;
    x ^= x >> h;
    x = (x * m2) & mask;
    x ^= x >> (h + (scale & 1));
    x = (x * m1) & mask;
    return x;
}

__global__ void k_rmat(int32_t *__restrict__ src, int32_t *__restrict__ dst, float *__restrict__ w,
                       int64_t first, int64_t count, int scale, uint32_t ta, uint32_t tab, uint32_t tabc,
                       uint64_t seed, int scramble_ids, uint64_t m1, uint64_t m2)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)(first + t);
        uint64_t u = 0, v = 0, bits = 0;
        for (int l = 0; l < scale; l++) {
            if ((l & 1) == 0) bits = rnd(seed, 1, i * 32 + (uint64_t)(l >> 1));
            const uint32_t r = (l & 1) ? (uint32_t)(bits >> 32) : (uint32_t)bits;
            const uint64_t bu = r >= tab, bv = (r >= ta && r < tab) || r >= tabc;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        if (scramble_ids) {
            u = scramble(u, scale, m1, m2);
            v = scramble(v, scale, m1, m2);
        }
        src[t] = (int32_t)u;
        dst[t] = (int32_t)v;
        if (w) w[t] = 1.0f - (float)(rnd(seed, 2, i) >> 40) * (1.0f / 16777216.0f);
    }
}

__global__ void k_er(int32_t *__restrict__ src, int32_t *__restrict__ dst, float *__restrict__ w,
                     int64_t first, int64_t count, int64_t n, uint64_t seed)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)(first + t);
        const uint64_t r = rnd(seed, 3, i);
        src[t] = (int32_t)(((r & 0xffffffffull) * (uint64_t)n) >> 32);
        dst[t] = (int32_t)(((r >> 32) * (uint64_t)n) >> 32);
        if (w) w[t] = 1.0f - (float)(rnd(seed, 2, i) >> 40) * (1.0f / 16777216.0f);
    }
}

__global__ void k_uniform_labels(int32_t *__restrict__ y, int64_t n, int32_t k, uint64_t seed)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = 1 + (int32_t)(((rnd(seed, 4, (uint64_t)i) >> 32) * (uint64_t)k) >> 32);
}

int grid_for(int64_t items)
{
    int64_t want = (items + 255) / 256;
    int64_t cap = (int64_t)gee::sm_count() * 16;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" {

uint64_t gee_synth_word(uint64_t seed, uint64_t tag, uint64_t ctr) { return rnd(seed, tag, ctr); }

int gee_synth_rmat(int32_t *src, int32_t *dst, float *w, int64_t first, int64_t count, int32_t scale,
                   double a, double b, double c, uint64_t seed, int32_t scramble_ids, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(scale >= 1 && scale <= 31, GEE_ERR_INVALID, "scale must be in [1, 31]");
    GEE_REQUIRE(count >= 0 && first >= 0, GEE_ERR_INVALID, "first/count must be nonnegative");
    if (count == 0) return GEE_OK;
    const double two32 = 4294967296.0;
    const uint32_t ta = (uint32_t)(a * two32), tab = (uint32_t)((a + b) * two32),
                   tabc = (uint32_t)((a + b + c) * two32);
    const uint64_t m1 = splitmix64(seed ^ 0x5EED1ull) | 1ull, m2 = splitmix64(seed ^ 0x5EED2ull) | 1ull;
    k_rmat<<<grid_for(count), 256, 0, gee::as_stream(stream)>>>(src, dst, w, first, count, scale, ta, tab,
                                                               tabc, seed, scramble_ids, m1, m2);
    return gee::check_launch("k_rmat");
}

int gee_synth_er(int32_t *src, int32_t *dst, float *w, int64_t first, int64_t count, int64_t n,
                 uint64_t seed, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(n >= 1 && n <= INT32_MAX, GEE_ERR_INVALID, "n must be in [1, 2^31)");
    if (count <= 0) return GEE_OK;
    k_er<<<grid_for(count), 256, 0, gee::as_stream(stream)>>>(src, dst, w, first, count, n, seed);
    return gee::check_launch("k_er");
}

int gee_synth_uniform_labels(int32_t *y, int64_t n, int32_t k, uint64_t seed, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "k must be positive");
    if (n <= 0) return GEE_OK;
    k_uniform_labels<<<grid_for(n), 256, 0, gee::as_stream(stream)>>>(y, n, k, seed);
    return gee::check_launch("k_uniform_labels");
}

}  // extern "C"
