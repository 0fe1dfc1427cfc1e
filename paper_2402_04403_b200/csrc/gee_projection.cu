// K1: class-count histogram + projection scalars + compact labels.
//
// Restates build_projection (reference encoder.py:80-103): counts =
// np.bincount(labels, minlength=k+1) (:87), inv[c] = 1/counts[c] for
// nonempty classes, inv[0] = 0 (:95-97).  W is never materialised: the edge
// kernels look up inv[Y[x]].
//
// One pass over the int32 labels (HBM-bound: 4 B read + label_bytes written
// per node).  Each CTA keeps up to 32 lane-privatised copies of the K+1 bin
// histogram in shared memory (u32 ATOMS.ADD, measured 8.5 op/clk/SM on
// B200), flushes them with 64-bit global atomics, and narrows each label to
// u8/u16 on the way through so the edge kernels gather 1-2 B per endpoint.
#include "gee_common.cuh"

namespace {

constexpr int HIST_THREADS = 512;
constexpr int HIST_SMEM_WORDS = 12288;  // 48 KB of bins

template <typename LB>
__device__ __forceinline__ void put_label(LB *compact, int64_t i, int32_t c) { compact[i] = (LB)c; }

template <typename LB>
__global__ void __launch_bounds__(HIST_THREADS)
k_label_hist(const int32_t *__restrict__ labels, int64_t n, int32_t k,
             unsigned long long *__restrict__ counts, LB *__restrict__ compact,
             unsigned long long *__restrict__ bad, int copies, bool vec)
{
    extern __shared__ uint32_t hist[];  // copies * (k+1) bins
    const int bins = k + 1;
    const bool smem = copies > 0;
    if (smem)
        for (int i = threadIdx.x; i < copies * bins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    uint32_t *mine = smem ? hist + (threadIdx.x % copies) * bins : nullptr;
    uint32_t nbad = 0;

    auto count = [&](int64_t i, int32_t c) {
        if ((uint32_t)c > (uint32_t)k) {  // outside [0, k] (LabelVector, labeling.py:24-29)
            nbad++;
            c = 0;
        } else if (smem) {
            atomicAdd(&mine[c], 1u);
        } else {
            atomicAdd(&counts[c], 1ull);
        }
        if (compact) put_label(compact, i, c);
    };

    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t done = 0;
    if (vec) {
        const int64_t n4 = n >> 2;
        const int4 *l4 = reinterpret_cast<const int4 *>(labels);
        for (int64_t q = start; q < n4; q += stride) {
            int4 v = __ldcs(l4 + q);
            count(4 * q + 0, v.x);
            count(4 * q + 1, v.y);
            count(4 * q + 2, v.z);
            count(4 * q + 3, v.w);
        }
        done = n4 << 2;
    }
    for (int64_t i = done + start; i < n; i += stride) count(i, __ldcs(labels + i));

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

template <typename LB>
int launch_hist(const int32_t *labels, int64_t n, int32_t k, unsigned long long *counts,
                LB *compact, unsigned long long *bad, cudaStream_t st)
{
    const int bins = k + 1;
    int copies = HIST_SMEM_WORDS / bins;
    if (copies > 32) copies = 32;
    size_t sh = copies > 0 ? (size_t)copies * bins * sizeof(uint32_t) : 0;
    int64_t want = (n + HIST_THREADS * 4 - 1) / (HIST_THREADS * 4);
    int64_t cap = (int64_t)gee::sm_count() * 4;
    int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    bool vec = gee::aligned16(labels);
    k_label_hist<LB><<<grid, HIST_THREADS, sh, st>>>(labels, n, k, counts, compact, bad, copies, vec);
    return gee::check_launch("k_label_hist");
}

}  // namespace

extern "C" {

size_t gee_projection_work_bytes(int32_t) { return 0; }

int gee_build_projection(const int32_t *labels, int64_t n, int32_t k, int64_t *counts,
                         float *inv_f32, double *inv_f64, void *compact, int64_t *bad,
                         void *, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0, GEE_ERR_INVALID, "node count must be nonnegative");
    GEE_REQUIRE(counts != nullptr, GEE_ERR_INVALID, "counts must not be NULL");
    GEE_REQUIRE(n == 0 || labels != nullptr, GEE_ERR_INVALID, "labels must not be NULL");
    cudaStream_t st = gee::as_stream(stream);
    GEE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)(k + 1), st));
    if (bad) GEE_CUDA(cudaMemsetAsync(bad, 0, sizeof(int64_t), st));
    auto *cnt = reinterpret_cast<unsigned long long *>(counts);
    auto *nb = reinterpret_cast<unsigned long long *>(bad);
    int rc = GEE_OK;
    if (n > 0) {
        switch (gee_label_bytes(k)) {
        case 1: rc = launch_hist<uint8_t>(labels, n, k, cnt, (uint8_t *)compact, nb, st); break;
        case 2: rc = launch_hist<uint16_t>(labels, n, k, cnt, (uint16_t *)compact, nb, st); break;
        default: rc = launch_hist<int32_t>(labels, n, k, cnt, (int32_t *)compact, nb, st); break;
        }
        if (rc) return rc;
    }
    if (inv_f32 || inv_f64) {
        k_inv<<<(k + 1 + 255) / 256, 256, 0, st>>>(cnt, k, inv_f32, inv_f64);
        return gee::check_launch("k_inv");
    }
    return GEE_OK;
}

}  // extern "C"
