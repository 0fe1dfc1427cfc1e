// K1: class-count histogram + projection scalars + the label table.
//
// Restates build_projection (reference encoder.py:80-103): counts =
// np.bincount(labels, minlength=k+1) (:87), inv[c] = 1/counts[c] for
// nonempty classes, inv[0] = 0 (:95-97).  W is never materialised: the edge
// kernels look up inv[Y[x]].
//
// One pass over the int32 labels (HBM-bound: 4 B read, 1-2 B written per
// node, plus the optional hot-rank stream).  Each CTA keeps up to 32
// lane-privatised copies of the K+1 bin histogram in shared memory (u32
// ATOMS.ADD, measured 8.5 op/clk/SM on B200) and flushes them with 64-bit
// global atomics.  The label table (gee_common.cuh) receives every label at
// slot n_hot + v, and hot vertices' labels again at their degree rank.
#include "gee_common.cuh"

namespace {

constexpr int HIST_THREADS = 512;
constexpr int HIST_SMEM_WORDS = 12288;  // 48 KB of bins

template <typename LT>
__global__ void __launch_bounds__(HIST_THREADS)
k_label_hist(const int32_t *__restrict__ labels, int64_t n, int32_t k, unsigned long long *__restrict__ counts,
             LT *__restrict__ table, const int32_t *__restrict__ hot_rank, int64_t n_hot,
             unsigned long long *__restrict__ bad, int copies, const uint32_t *__restrict__ hot_bits,
             const int32_t *__restrict__ hot_pref, const int32_t *__restrict__ hot_list, int64_t count_lo,
             int64_t count_hi)
{
    extern __shared__ uint32_t hist[];  // copies * (k+1) bins
    const int bins = k + 1;
    const bool smem = copies > 0;
    if (smem)
        for (int i = threadIdx.x; i < copies * bins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    uint32_t *mine = smem ? hist + (threadIdx.x % copies) * bins : nullptr;
    uint32_t nbad = 0;
    LT *cold = table ? table + n_hot : nullptr;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;

    // count label c of node i (checked) and return it (0 when out of range);
    // only nodes in [count_lo, count_hi) are counted (a row shard's slice of
    // a sharded histogram; the table always receives every label)
    const uint64_t cspan = (uint64_t)(count_hi - count_lo);
    const bool ranged = count_lo > 0 || count_hi < n;  // uniform: the full-range path has no extra test
    auto count = [&](int64_t i, int32_t c) -> int32_t {
        const bool counted = !ranged || (uint64_t)(i - count_lo) < cspan;
        if ((uint32_t)c > (uint32_t)k) {  // outside [0, k] (LabelVector, labeling.py:24-29)
            if (counted) nbad++;
            return 0;
        }
        if (!counted) return c;
        if (smem)
            atomicAdd(&mine[c], 1u);
        else
            atomicAdd(&counts[c], 1ull);
        return c;
    };
    auto one = [&](int64_t i, int32_t c, int32_t r) {
        c = count(i, c);
        if (cold) {
            cold[i] = (LT)c;
            GEE_DCHECK(r < n_hot);
            if (r >= 0) table[r] = (LT)c;  // hot tier copy (gee_hot.cu)
        }
    };

    int64_t done = 0;
    if ((reinterpret_cast<uintptr_t>(labels) & 15) == 0 && (!hot_rank || (reinterpret_cast<uintptr_t>(hot_rank) & 15) == 0)) {
        const int64_t n4 = n >> 2;
        // u8 table with a 4-byte aligned cold tier: one 32-bit store per 4 labels
        const bool pack4 = sizeof(LT) == 1 && cold && (reinterpret_cast<uintptr_t>(cold) & 3) == 0;
        for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
            const int4 v = __ldcs(reinterpret_cast<const int4 *>(labels) + q);
            int4 r = make_int4(-1, -1, -1, -1);
            if (hot_rank) r = __ldcs(reinterpret_cast<const int4 *>(hot_rank) + q);
            if (hot_bits) {  // compact hot tier: bitmap word, its prefix, ranks in vertex order
                const uint32_t word = __ldg(hot_bits + (q >> 3)), sh = (uint32_t)(4 * q) & 31u;
                const uint32_t b4 = (word >> sh) & 15u;
                if (b4) {
                    const int32_t *lp = hot_list + __ldg(hot_pref + (q >> 3)) + __popc(word & ((1u << sh) - 1u));
                    int j = 0;
                    if (b4 & 1u) r.x = lp[j++];
                    if (b4 & 2u) r.y = lp[j++];
                    if (b4 & 4u) r.z = lp[j++];
                    if (b4 & 8u) r.w = lp[j++];
                }
            }
            if (pack4) {
                const int32_t c0 = count(4 * q, v.x), c1 = count(4 * q + 1, v.y), c2 = count(4 * q + 2, v.z),
                              c3 = count(4 * q + 3, v.w);
                reinterpret_cast<uint32_t *>(cold)[q] = (uint32_t)c0 | (uint32_t)c1 << 8 | (uint32_t)c2 << 16 |
                                                        (uint32_t)c3 << 24;
                GEE_DCHECK(r.x < n_hot && r.y < n_hot && r.z < n_hot && r.w < n_hot);
                if (r.x >= 0) table[r.x] = (LT)c0;
                if (r.y >= 0) table[r.y] = (LT)c1;
                if (r.z >= 0) table[r.z] = (LT)c2;
                if (r.w >= 0) table[r.w] = (LT)c3;
            } else {
                one(4 * q + 0, v.x, r.x);
                one(4 * q + 1, v.y, r.y);
                one(4 * q + 2, v.z, r.z);
                one(4 * q + 3, v.w, r.w);
            }
        }
        done = n4 << 2;
    }
    for (int64_t i = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int32_t r = hot_rank ? __ldcs(hot_rank + i) : -1;
        if (hot_bits) {
            const uint32_t word = hot_bits[i >> 5], bit = (uint32_t)i & 31u;
            if ((word >> bit) & 1u) r = hot_list[hot_pref[i >> 5] + __popc(word & ((1u << bit) - 1u))];
        }
        one(i, __ldcs(labels + i), r);
    }
    if (table && blockIdx.x == 0 && threadIdx.x == 0) table[n_hot + n] = (LT)0;  // sentinel slot
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

template <typename LT>
int launch_hist(const int32_t *labels, int64_t n, int32_t k, unsigned long long *counts, void *table,
                const int32_t *hot_rank, int64_t n_hot, unsigned long long *bad, cudaStream_t st,
                const uint32_t *hot_bits = nullptr, const int32_t *hot_pref = nullptr,
                const int32_t *hot_list = nullptr, int64_t count_lo = 0, int64_t count_hi = -1)
{
    if (count_hi < 0) count_hi = n;
    const int bins = k + 1;
    int copies = HIST_SMEM_WORDS / bins;
    if (copies > 32) copies = 32;
    const size_t sh = copies > 0 ? (size_t)copies * bins * sizeof(uint32_t) : 0;
    const int64_t want = (n + HIST_THREADS * 4 - 1) / (HIST_THREADS * 4);
    const int64_t cap = (int64_t)gee::sm_count() * 4;
    const int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    k_label_hist<LT><<<grid, HIST_THREADS, sh, st>>>(labels, n, k, counts, static_cast<LT *>(table), hot_rank, n_hot,
                                                     bad, copies, hot_bits, hot_pref, hot_list,
                                                     count_lo, count_hi);
    return gee::check_launch("k_label_hist");
}

}  // namespace

extern "C" {

int gee_label_bytes(int32_t k) { return k <= 255 ? 1 : (k <= 65535 ? 2 : 4); }

size_t gee_label_table_bytes(int64_t n, int64_t n_hot, int32_t k)
{
    const size_t b = (size_t)(n_hot + n + 1) * (size_t)gee_label_bytes(k);
    return (b + 15) & ~(size_t)15;
}

size_t gee_projection_work_bytes(int32_t) { return 0; }

int gee_build_projection(const int32_t *labels, int64_t n, int32_t k, int64_t *counts, float *inv_f32,
                         double *inv_f64, void *table, const int32_t *hot_rank, int64_t n_hot, int64_t *bad,
                         void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && n_hot >= 0, GEE_ERR_INVALID, "n and n_hot must be nonnegative");
    GEE_REQUIRE(n + n_hot < INT32_MAX, GEE_ERR_INVALID, "label table exceeds int32 slots");
    GEE_REQUIRE(counts != nullptr, GEE_ERR_INVALID, "counts must not be NULL");
    GEE_REQUIRE(n == 0 || labels != nullptr, GEE_ERR_INVALID, "labels must not be NULL");
    GEE_REQUIRE(!hot_rank || (table && n_hot > 0), GEE_ERR_INVALID, "hot_rank needs a table with n_hot > 0");
    cudaStream_t st = gee::as_stream(stream);
    GEE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)(k + 1), st));
    if (bad) GEE_CUDA(cudaMemsetAsync(bad, 0, sizeof(int64_t), st));
    auto *cnt = reinterpret_cast<unsigned long long *>(counts);
    auto *nb = reinterpret_cast<unsigned long long *>(bad);
    if (n > 0 || table) {
        int rc;
        switch (gee_label_bytes(k)) {
        case 1: rc = launch_hist<uint8_t>(labels, n, k, cnt, table, hot_rank, n_hot, nb, st); break;
        case 2: rc = launch_hist<uint16_t>(labels, n, k, cnt, table, hot_rank, n_hot, nb, st); break;
        default: rc = launch_hist<int32_t>(labels, n, k, cnt, table, hot_rank, n_hot, nb, st); break;
        }
        if (rc) return rc;
    }
    if (inv_f32 || inv_f64) {
        k_inv<<<(k + 1 + 255) / 256, 256, 0, st>>>(cnt, k, inv_f32, inv_f64);
        return gee::check_launch("k_inv");
    }
    return GEE_OK;
}

int gee_build_projection_hotc(const int32_t *labels, int64_t n, int32_t k, int64_t *counts, float *inv_f32,
                              double *inv_f64, void *table, const uint32_t *hot_bits, const int32_t *hot_pref,
                              const int32_t *hot_list, int64_t n_hot, int64_t *bad, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && n_hot >= 0, GEE_ERR_INVALID, "n and n_hot must be nonnegative");
    GEE_REQUIRE(n + n_hot < INT32_MAX, GEE_ERR_INVALID, "label table exceeds int32 slots");
    GEE_REQUIRE(counts != nullptr && table != nullptr, GEE_ERR_INVALID, "counts and table must not be NULL");
    GEE_REQUIRE(n == 0 || labels != nullptr, GEE_ERR_INVALID, "labels must not be NULL");
    GEE_REQUIRE(hot_bits && hot_pref && hot_list && n_hot > 0, GEE_ERR_INVALID,
                "the compact hot tier needs its bitmap, prefix and rank list and n_hot > 0");
    cudaStream_t st = gee::as_stream(stream);
    GEE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)(k + 1), st));
    if (bad) GEE_CUDA(cudaMemsetAsync(bad, 0, sizeof(int64_t), st));
    auto *cnt = reinterpret_cast<unsigned long long *>(counts);
    auto *nb = reinterpret_cast<unsigned long long *>(bad);
    int rc;
    switch (gee_label_bytes(k)) {
    case 1: rc = launch_hist<uint8_t>(labels, n, k, cnt, table, nullptr, n_hot, nb, st, hot_bits, hot_pref, hot_list); break;
    case 2: rc = launch_hist<uint16_t>(labels, n, k, cnt, table, nullptr, n_hot, nb, st, hot_bits, hot_pref, hot_list); break;
    default: rc = launch_hist<int32_t>(labels, n, k, cnt, table, nullptr, n_hot, nb, st, hot_bits, hot_pref, hot_list); break;
    }
    if (rc) return rc;
    if (inv_f32 || inv_f64) {
        k_inv<<<(k + 1 + 255) / 256, 256, 0, st>>>(cnt, k, inv_f32, inv_f64);
        return gee::check_launch("k_inv");
    }
    return GEE_OK;
}

int gee_build_projection_sharded(const int32_t *labels, int64_t n, int32_t k, int64_t *counts, void *table,
                                 const uint32_t *hot_bits, const int32_t *hot_pref, const int32_t *hot_list,
                                 int64_t n_hot, int64_t count_lo, int64_t count_hi, int64_t *bad, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1, GEE_ERR_INVALID, "class count k must be positive (got %d)", k);
    GEE_REQUIRE(n >= 0 && n_hot >= 0, GEE_ERR_INVALID, "n and n_hot must be nonnegative");
    GEE_REQUIRE(n + n_hot < INT32_MAX, GEE_ERR_INVALID, "label table exceeds int32 slots");
    GEE_REQUIRE(counts != nullptr && table != nullptr, GEE_ERR_INVALID, "counts and table must not be NULL");
    GEE_REQUIRE(n == 0 || labels != nullptr, GEE_ERR_INVALID, "labels must not be NULL");
    GEE_REQUIRE(0 <= count_lo && count_lo <= count_hi && count_hi <= n, GEE_ERR_INVALID,
                "count range [%lld, %lld) outside [0, %lld]", (long long)count_lo, (long long)count_hi, (long long)n);
    GEE_REQUIRE(n_hot == 0 || (hot_bits && hot_pref && hot_list), GEE_ERR_INVALID,
                "n_hot > 0 needs the compact hot tier (bitmap, prefix, rank list)");
    cudaStream_t st = gee::as_stream(stream);
    GEE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)(k + 1), st));
    if (bad) GEE_CUDA(cudaMemsetAsync(bad, 0, sizeof(int64_t), st));
    auto *cnt = reinterpret_cast<unsigned long long *>(counts);
    auto *nb = reinterpret_cast<unsigned long long *>(bad);
    const uint32_t *hb = n_hot ? hot_bits : nullptr;
    switch (gee_label_bytes(k)) {
    case 1: return launch_hist<uint8_t>(labels, n, k, cnt, table, nullptr, n_hot, nb, st, hb, hot_pref, hot_list,
                                        count_lo, count_hi);
    case 2: return launch_hist<uint16_t>(labels, n, k, cnt, table, nullptr, n_hot, nb, st, hb, hot_pref, hot_list,
                                         count_lo, count_hi);
    default: return launch_hist<int32_t>(labels, n, k, cnt, table, nullptr, n_hot, nb, st, hb, hot_pref, hot_list,
                                         count_lo, count_hi);
    }
}

int gee_projection_inv(const int64_t *counts, int32_t k, float *inv_f32, double *inv_f64, void *stream)
{
    gee::clear_error();
    GEE_REQUIRE(k >= 1 && counts != nullptr, GEE_ERR_INVALID, "counts must not be NULL and k positive");
    k_inv<<<(k + 1 + 255) / 256, 256, 0, gee::as_stream(stream)>>>(
        reinterpret_cast<const unsigned long long *>(counts), k, inv_f32, inv_f64);
    return gee::check_launch("k_inv");
}

}  // extern "C"
