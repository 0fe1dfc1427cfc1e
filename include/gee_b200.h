/*
 * gee_b200.h -- C ABI of the B200-native GEE edge pass (libgee_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/gee).  The reference has no C ABI: its boundary
 * is the Python encoder API plus the numba kernel signatures.  Each entry
 * point below names the reference interface it replaces (file:line).
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer unless noted; arrays are
 *     borrowed, never freed or reallocated by the library.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream) and returns a status code;
 *     0 = GEE_OK.  gee_last_error() returns a thread-local message for the
 *     last failing call on the calling thread.
 *   - Labels: int32 in [0, k]; 0 = unknown, class c is Z column c-1
 *     (labeling.py:10-26, encoder.py:3-10).
 *   - Z is a dense row-major (n, k) float32 array.  Its accumulator is exact
 *     integer arithmetic in the pull path and fp32 red.global in the push path.
 *   - Hot-path calls (gee_build_projection, gee_embed_coo, gee_embed_csr_pull)
 *     never allocate; graph-preparation calls (gee_build_sym_csr,
 *     gee_pull_plan, gee_graph_stats) may allocate stream-ordered scratch
 *     with cudaMallocAsync and free it before returning.
 */
#ifndef GEE_B200_H
#define GEE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GEE_OK 0
#define GEE_ERR_INVALID 1    /* argument violates the contract (ValidationError) */
#define GEE_ERR_CUDA 2       /* CUDA runtime / launch failure */
#define GEE_ERR_RANGE 3      /* label or endpoint outside its range (ValidationError) */

/* gee_embed_coo flags */
#define GEE_ZERO_Z 1u        /* memset Z before the pass (embed_serial's np.zeros, encoder.py:117) */
#define GEE_SOURCE_ONLY 2u   /* apply only Z[src] += ...: EdgeAccounting.SOURCE_ONLY arc lists (encoder.py:37-55) */
#define GEE_PRECOMBINE 4u    /* warp pre-combine equal Z addresses before red.global (__match_any_sync) */

/* Library version (major*10000 + minor*100 + patch). */
int gee_version(void);

/* Thread-local message of the last failing call ("" if none). */
const char *gee_last_error(void);

/* Packed label format.  gee_build_projection writes the labels as u32
 * words holding per = 32/bits labels of `bits` bits each, label i in word
 * i/per at bit (i%per)*bits; bits = gee_label_bits(k), the smallest of
 * {1,2,3,4,5,6,8,10,16} that holds k (32 = raw int32 labels, one per word).
 * K=50 -> 6 bits, 5 per word (C4's 134M labels: 107 MB, L2-resident). */
int gee_label_bits(int32_t k);
int64_t gee_label_words(int64_t n, int32_t label_bits);

/* ---------------------------------------------------------------- K1 ----
 * Class-count histogram + projection scalars.
 * Replaces build_projection (encoder.py:80-103: np.bincount at :87, inv at
 * :95-97) and class_counts (labeling.py:107-109).
 *   counts[k+1]   int64, bit-exact np.bincount(labels, minlength=k+1)
 *   inv_f32[k+1]  float, inv_f32[c] = (float)(1.0/counts[c]) or 0; inv[0] = 0
 *   inv_f64[k+1]  double, same in f64 (may be NULL)
 *   packed        gee_label_words(n, gee_label_bits(k)) packed label words (may be NULL)
 *   bad           int64 device scalar: number of labels outside [0,k] (may be
 *                 NULL).  Counts of out-of-range labels are dropped.
 *   work          device scratch of gee_projection_work_bytes(k) bytes
 */
size_t gee_projection_work_bytes(int32_t k);
int gee_build_projection(const int32_t *labels, int64_t n, int32_t k,
                         int64_t *counts, float *inv_f32, double *inv_f64,
                         uint32_t *packed, int64_t *bad, void *work, void *stream);

/* ---------------------------------------------------------------- K3 ----
 * Push edge map over a listed edge list (COO, structure of arrays).
 * Replaces serial_pass (_kernels.py:210-226, via embed_serial,
 * encoder.py:106-120) and, with GEE_SOURCE_ONLY on arc lists,
 * arc_pass_worker (_kernels.py:138-207).
 *   Per edge i (u=src[i], v=dst[i], w = w ? w[i] : 1):
 *     if Y[v]: Z[u, Y[v]-1] += inv[Y[v]] * w
 *     if Y[u] and !(flags & GEE_SOURCE_ONLY): Z[v, Y[u]-1] += inv[Y[u]] * w
 *   labels: packed words with label_bits = gee_label_bits(k), or raw int32
 *   labels with label_bits = 32.  inv: inv_f32[k+1].
 *   Accumulation order is unspecified (fp32 atomics): results match the
 *   serial f64 oracle within fp32 accumulation error.
 */
int gee_embed_coo(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                  const uint32_t *labels, int32_t label_bits, const float *inv,
                  int64_t n, int32_t k, float *z, uint32_t flags, void *stream);

/* ---------------------------------------------------------------- K5 ----
 * Symmetric CSR of a listed edge list: row u holds (v, w) and row v holds
 * (u, w) for every listed edge (self-loops appear twice in row u).  This is
 * build_csr's undirected layout (graph.py:159-184, csr_fill
 * _kernels.py:229-238) applied to EVERY list, because the edge pass applies
 * both updates per listed edge whatever `directed` says (encoder.py:106-120).
 * Arc order within a row is unspecified (the pull accumulator is exact
 * integer arithmetic, so Z does not depend on it).
 *   offsets[n+1] int64; targets[2s] int32; weights[2s] float (NULL if w NULL)
 */
int gee_build_sym_csr(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                      int64_t n, int64_t *offsets, int32_t *targets, float *weights,
                      void *stream);

/* build_csr itself (graph.py:159-184): symmetric != 0 stores the mirror arc
 * of every listed edge (undirected EdgeList); 0 stores one arc per edge
 * (directed).  stable != 0 keeps the reference's arc order exactly (input
 * order, mirror right after the original; CUB radix sort by row, at most
 * 2^32-1 arcs); stable == 0 fills rows through atomic cursors. */
int gee_build_csr(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                  int64_t n, int32_t symmetric, int32_t stable, int64_t *offsets,
                  int32_t *targets, float *weights, void *stream);

/* Multi-GPU row-range ownership: offsets[n+1] of the full
 * symmetric CSR (degree count + scan, no fill) for the partition planner,
 * then the shard of rows [row_lo, row_hi): offsets[rows+1] rebased to 0,
 * targets/weights of those rows' arcs (sized full_offsets[hi]-full_offsets[lo]). */
int gee_sym_offsets(const int32_t *src, const int32_t *dst, int64_t s, int64_t n,
                    int64_t *offsets, void *stream);
int gee_build_sym_csr_rows(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                           int64_t n, int64_t row_lo, int64_t row_hi,
                           const int64_t *full_offsets, int64_t *offsets, int32_t *targets,
                           float *weights, void *stream);

/* CSR (offsets, arcs) -> per-arc source row (COO src) for a stored CsrGraph,
 * so that a directed CsrGraph (EdgeAccounting.BOTH_ENDPOINTS) can be fed to
 * gee_build_sym_csr or gee_embed_coo.  rows[arcs] int32. */
int gee_csr_rows(const int64_t *offsets, int64_t n, int64_t arcs, int32_t *rows, void *stream);

/* Graph statistics that size the pull accumulator (host outputs):
 * max over rows of sum |w| (or max degree if w NULL), min nonzero |w|,
 * max |w|, and whether any weight is non-finite. */
int gee_graph_stats(const int64_t *offsets, const float *w, int64_t n, int64_t arcs,
                    double *max_row_abs, double *min_abs_nz, double *max_abs,
                    int32_t *nonfinite, void *stream);

/* ---------------------------------------------------------------- K4 ----
 * Pull (row-owner) edge map over a symmetric CSR.  Tile j covers arcs
 * [j*GEE_TILE_ARCS, (j+1)*GEE_TILE_ARCS) and owns the rows whose first arc
 * position offsets[r] falls in it; tile_row[j] = first such row
 * (gee_pull_plan).  Per row x:
 *     Z[x, c] = inv[c+1] * sum_{arcs x->v, Y[v]=c+1} w
 * accumulated exactly in integers (unit weights: counts; weighted: fixed
 * point w*2^scale_exp rounded to int64), so Z is bit-stable run to run and
 * independent of arc order.  Every row of Z is written exactly once; no
 * zeroing is needed.  Rows that span tiles are combined through `slots`
 * (gee_pull_slots_bytes bytes, zero on first use, left zero on return).
 *   w == NULL means unit weights (scale_exp ignored).
 *   inv: inv_f64[k+1].
 * Replaces embed_parallel's zero wave + arc wave (encoder.py:123-194,
 * zero_worker _kernels.py:124-135, arc_pass_worker _kernels.py:138-207)
 * for SOURCE_ONLY (symmetric) storage.
 */
#define GEE_TILE_ARCS 4096
int64_t gee_pull_tiles(int64_t arcs);
size_t gee_pull_slots_bytes(int64_t arcs, int32_t k);
int gee_pull_plan(const int64_t *offsets, int64_t n, int64_t arcs, int64_t *tile_row,
                  void *stream);
int gee_embed_csr_pull(const int64_t *offsets, const int32_t *targets, const float *w,
                       int64_t n, int64_t arcs, const int64_t *tile_row, int32_t scale_exp,
                       const uint32_t *labels, int32_t label_bits, const double *inv,
                       int32_t k, float *z, void *slots, void *stream);

/* Hot-label tier (graph preparation; see gee_hot.cu).  gee_hot_plan ranks
 * vertices by degree offsets[v+1]-offsets[v] (descending, ties by id) and
 * marks the top max_hot with degree >= min_degree: hot_rank[v] = rank or -1,
 * hot_vertex[rank] = v (may be NULL), *n_hot (host) = count.
 * gee_hot_encode rewrites targets t of hot vertices as 0x80000000|rank.
 * gee_build_projection_hot additionally scatters labels into hot_labels
 * (u8 if k <= 255 else u16, gee_hot_label_bytes) at their ranks, and
 * gee_embed_csr_pull_hot reads hot targets from that table (its head staged
 * in shared memory) and cold targets from the packed labels. */
int gee_hot_plan(const int64_t *offsets, int64_t n, int64_t max_hot, int64_t min_degree,
                 int32_t *hot_rank, int32_t *hot_vertex, int64_t *n_hot, void *stream);
int gee_hot_encode(int32_t *targets, int64_t arcs, const int32_t *hot_rank, void *stream);
int gee_hot_label_bytes(int32_t k);
int gee_build_projection_hot(const int32_t *labels, int64_t n, int32_t k, int64_t *counts,
                             float *inv_f32, double *inv_f64, uint32_t *packed, int64_t *bad,
                             const int32_t *hot_rank, void *hot_labels, void *stream);
int gee_embed_csr_pull_hot(const int64_t *offsets, const int32_t *targets, const float *w,
                           int64_t n, int64_t arcs, const int64_t *tile_row, int32_t scale_exp,
                           const uint32_t *labels, int32_t label_bits, const void *hot_labels,
                           int64_t n_hot, const double *inv, int32_t k, float *z, void *slots,
                           void *stream);

/* Choose the fixed-point exponent for a weighted pull: the largest e with
 * max_row_abs * 2^e < 2^62.  Returns the relative quantisation bound
 * 2^-(e+1)/min_abs_nz through *rel_err (host). */
int gee_pull_scale_exp(double max_row_abs, double min_abs_nz, int32_t *scale_exp,
                       double *rel_err);

#ifdef __cplusplus
}
#endif
#endif /* GEE_B200_H */
