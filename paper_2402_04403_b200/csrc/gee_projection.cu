// K1: class-count histogram + projection scalars + packed labels.
//
// Restates build_projection (reference encoder.py:80-103): counts =
// np.bincount(labels, minlength=k+1) (:87), inv[c] = 1/counts[c] for
// nonempty classes, inv[0] = 0 (:95-97).  W is never materialised: the edge
// kernels look up inv[Y[x]].
//
// One pass over the int32 labels (HBM-bound: 4 B read + bits/8 B written per
// node).  Each thread builds one packed label word (gee_common.cuh
// LabelFmt); each CTA keeps up to 32 lane-privatised copies of the K+1 bin
// histogram in shared memory (u32 ATOMS.ADD, measured 8.5 op/clk/SM on
// B200) and flushes them with 64-bit global atomics.
#include "gee_common.cuh"

namespace {

constexpr int HIST_THREADS = 512;
constexpr int HIST_SMEM_WORDS = 12288;  // 48 KB of bins

__global__ void __launch_bounds__(HIST_THREADS)
k_label_hist(const int32_t *__restrict__ labels, int64_t n, int32_t k, gee::LabelFmt f,
             unsigned long long *__restrict__ counts, uint32_t *__restrict__ packed,
             unsigned long long *__restrict__ bad, int copies, const int32_t *__restrict__ hot_rank,
             void *__restrict__ hot_labels, int hot_bytes)
{
    extern __shared__ uint32_t hist[];  // copies * (k+1) bins
    const int bins = k + 1;
    const bool smem = copies > 0;
    if (smem)
        for (int i = threadIdx.x; i < copies * bins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    uint32_t *mine = smem ? hist + (threadIdx.x % copies) * bins : nullptr;
    uint32_t nbad = 0;
    const int64_t words = (n + f.per - 1) / f.per;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t wi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; wi < words; wi += stride) {
        uint32_t word = 0;
        const int64_t i0 = wi * f.per;
        for (uint32_t j = 0; j < f.per; j++) {
            const int64_t i = i0 + j;
            if (i >= n) break;
            int32_t c = __ldcs(labels + i);
            if ((uint32_t)c > (uint32_t)k) {  // outside [0, k] (LabelVector, labeling.py:24-29)
                nbad++;
                c = 0;
            } else if (smem) {
                atomicAdd(&mine[c], 1u);
            } else {
                atomicAdd(&counts[c], 1ull);
            }
            word |= ((uint32_t)c & f.mask) << (j * f.bits);
            if (hot_rank) {  // hot tier: dense rank-ordered copy (gee_hot.cu)
                const int32_t r = __ldcs(hot_rank + i);
                if (r >= 0) {
                    if (hot_bytes == 1) static_cast<uint8_t *>(hot_labels)[r] = (uint8_t)c;
                    else static_cast<uint16_t *>(hot_labels)[r] = (uint16_t)c;
                }
            }
        }
        if (packed) __stcs(packed + wi, word);
    }
    __syncthreads();
    if (smem) {
        for (int c = threadIdx.x; c < bins; c += blockDim.x) {
            uint32_t t = 0;
            for (int r = 0; r < copies; r++) t += hist[r * bins + c];
            if (t) atomicAdd(&counts[c], (unsigned long long)t);
        }
    }
    if (bad && nbad) atomicAdd(bad, (unsigned long long)nbad);
}

__global__ void k_inv(const unsigned long long *__restrict__ counts, int32_t k,
                      float *__restrict__ inv32, double *__restrict__ inv64)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > k) return;
    unsigned long long cnt = counts[c];
    double d = (c > 0 && cnt > 0) ? 1.0 / (double)cnt : 0.0;
    if (inv32) inv32[c] = (float)d;
    if (inv64) inv64[c] = d;
}

}  // namespace

extern "C" {

int gee_label_bits(int32_t k)
{
    static const int widths[] = {1, 2, 3, 4, 5, 6, 8, 10, 16};
    for (int b : widths)
        if (k <= (1 << b) - 1) return b;
    return 32;
}

int64_t gee_label_words(int64_t n, int32_t label_bits)
{
    if (label_bits != 32 && (label_bits < 1 || label_bits > 16)) return -1;
    const int64_t per = 32 / label_bits;
    return (n + per - 1) / per;
}

size_t gee_projection_work_bytes(int32_t) { return 0; }

int gee_build_projection_hot(const int32_t *labels, int64_t n, int32_t k, int64_t *counts, float *inv_f32,
                             double *inv_f64, uint32_t *packed, int64_t *bad, const int32_t *hot_rank,
                             void *hot_labels, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0, GEE_ERR_INVALID, "node count must be nonnegative");
    GEE_REQUIRE(n <= INT32_MAX, GEE_ERR_INVALID, "node count %lld exceeds int32", (long long)n);
    GEE_REQUIRE(counts != nullptr, GEE_ERR_INVALID, "counts must not be NULL");
    GEE_REQUIRE(n == 0 || labels != nullptr, GEE_ERR_INVALID, "labels must not be NULL");
    GEE_REQUIRE(!hot_rank || (hot_labels && k <= 65535), GEE_ERR_INVALID,
                "hot tier needs hot_labels and k <= 65535");
    cudaStream_t st = gee::as_stream(stream);
    GEE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)(k + 1), st));
    if (bad) GEE_CUDA(cudaMemsetAsync(bad, 0, sizeof(int64_t), st));
    auto *cnt = reinterpret_cast<unsigned long long *>(counts);
    if (n > 0) {
        const gee::LabelFmt f = gee::label_fmt(gee_label_bits(k));
        const int bins = k + 1;
        int copies = HIST_SMEM_WORDS / bins;
        if (copies > 32) copies = 32;
        size_t sh = copies > 0 ? (size_t)copies * bins * sizeof(uint32_t) : 0;
        const int64_t words = (n + f.per - 1) / f.per;
        int64_t want = (words + HIST_THREADS - 1) / HIST_THREADS;
        int64_t cap = (int64_t)gee::sm_count() * 4;
        int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
        k_label_hist<<<grid, HIST_THREADS, sh, st>>>(labels, n, k, f, cnt, packed,
                                                     reinterpret_cast<unsigned long long *>(bad), copies, hot_rank,
                                                     hot_labels, k <= 255 ? 1 : 2);
        int rc = gee::check_launch("k_label_hist");
        if (rc) return rc;
    }
    if (inv_f32 || inv_f64) {
        k_inv<<<(k + 1 + 255) / 256, 256, 0, st>>>(cnt, k, inv_f32, inv_f64);
        return gee::check_launch("k_inv");
    }
    return GEE_OK;
}

int gee_build_projection(const int32_t *labels, int64_t n, int32_t k, int64_t *counts, float *inv_f32,
                         double *inv_f64, uint32_t *packed, int64_t *bad, void *, void *stream)
{
    return gee_build_projection_hot(labels, n, k, counts, inv_f32, inv_f64, packed, bad, nullptr, nullptr, stream);
}

}  // extern "C"
