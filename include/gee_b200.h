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
 *   - Hot-path calls (gee_build_projection*, gee_embed_coo, gee_gather_labels,
 *     gee_reduce_blocks_pad8, gee_reduce_heavy, gee_reduce_wide) never allocate; graph-preparation calls (gee_build_csr, gee_hot_plan,
 *     gee_graph_stats, ...) may allocate stream-ordered scratch with
 *     cudaMallocAsync and free it before returning.
 *
 * Label table.  The edge kernels read labels from a table of
 * gee_label_bytes(k)-byte entries (u8 for k <= 255, u16 for k <= 65535,
 * else int32) laid out as
 *     [ n_hot hot-tier labels in degree-rank order | n labels by vertex id | 0 ]
 * (gee_label_table_bytes(n, n_hot, k) bytes).  Pull targets hold table
 * slots: rank r for a hot vertex, n_hot + v for a cold vertex v
 * (gee_hot_encode); with n_hot = 0 the slot is the vertex id itself.
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

/* Bytes per label-table entry for k classes (1, 2 or 4) and table size. */
int gee_label_bytes(int32_t k);
size_t gee_label_table_bytes(int64_t n, int64_t n_hot, int32_t k);

/* ---------------------------------------------------------------- K1 ----
 * Class-count histogram + projection scalars + label table.
 * Replaces build_projection (encoder.py:80-103: np.bincount at :87, inv at
 * :95-97) and class_counts (labeling.py:107-109).
 *   counts[k+1]   int64, bit-exact np.bincount(labels, minlength=k+1)
 *   inv_f32[k+1]  float, inv_f32[c] = (float)(1.0/counts[c]) or 0; inv[0] = 0
 *   inv_f64[k+1]  double, same in f64 (may be NULL)
 *   table         label table (may be NULL): table[n_hot + v] = Y[v],
 *                 table[hot_rank[v]] = Y[v] for hot v, table[n_hot + n] = 0
 *   hot_rank      int32[n] (gee_hot_plan) or NULL when n_hot == 0
 *   bad           int64 device scalar: number of labels outside [0,k] (may be
 *                 NULL).  Out-of-range labels count as 0 (unknown).
 */
size_t gee_projection_work_bytes(int32_t k);
int gee_build_projection(const int32_t *labels, int64_t n, int32_t k,
                         int64_t *counts, float *inv_f32, double *inv_f64,
                         void *table, const int32_t *hot_rank, int64_t n_hot,
                         int64_t *bad, void *stream);

/* gee_build_projection with the hot tier in compact form (built once per
 * graph by the caller): hot_bits[(n+31)/32] marks the hot vertices,
 * hot_pref[w] counts the hot vertices before word w, and hot_list holds
 * their degree ranks in vertex order: about n/4 + 4*n_hot bytes instead of
 * the 4*n of hot_rank (C4: 0.10 GB instead of 0.54 GB per call, also over
 * PCIe on the streamed path). */
int gee_build_projection_hotc(const int32_t *labels, int64_t n, int32_t k, int64_t *counts, float *inv_f32,
                              double *inv_f64, void *table, const uint32_t *hot_bits, const int32_t *hot_pref,
                              const int32_t *hot_list, int64_t n_hot, int64_t *bad, void *stream);

/* Sharded histogram for row-range multi-GPU runs (SURVEY 8(e) scheme 1):
 * the label table receives every label (as gee_build_projection_hotc; the
 * hot tier may be absent, n_hot = 0), but counts[] only the nodes in
 * [count_lo, count_hi) -- this rank's slice of np.bincount (encoder.py:87).
 * The caller sums counts[] over the ranks (one all-reduce of k+1 int64)
 * and then calls gee_projection_inv. */
int gee_build_projection_sharded(const int32_t *labels, int64_t n, int32_t k, int64_t *counts, void *table,
                                 const uint32_t *hot_bits, const int32_t *hot_pref, const int32_t *hot_list,
                                 int64_t n_hot, int64_t count_lo, int64_t count_hi, int64_t *bad, void *stream);

/* inv[c] = 1/counts[c] for nonempty classes c >= 1, inv[0] = 0
 * (encoder.py:95-97), f32 and/or f64 (either may be NULL). */
int gee_projection_inv(const int64_t *counts, int32_t k, float *inv_f32, double *inv_f64, void *stream);

/* ---------------------------------------------------------------- K3 ----
 * Push edge map over a listed edge list (COO, structure of arrays).
 * Replaces serial_pass (_kernels.py:210-226, via embed_serial,
 * encoder.py:106-120) and, with GEE_SOURCE_ONLY on arc lists,
 * arc_pass_worker (_kernels.py:138-207).
 *   Per edge i (u=src[i], v=dst[i], w = w ? w[i] : 1):
 *     if Y[v]: Z[u, Y[v]-1] += inv[Y[v]] * w
 *     if Y[u] and !(flags & GEE_SOURCE_ONLY): Z[v, Y[u]-1] += inv[Y[u]] * w
 *   Y[x] = table[label_off + x] (label_off = n_hot of the table).
 *   inv: inv_f32[k+1].  Accumulation order is unspecified (fp32 atomics):
 *   results match the serial f64 oracle within fp32 accumulation error.
 */
int gee_embed_coo(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                  const void *table, int64_t label_off, const float *inv,
                  int64_t n, int32_t k, float *z, uint32_t flags, void *stream);

/* ---------------------------------------------------------------- K5 ----
 * build_csr (graph.py:159-184, csr_fill _kernels.py:229-238):
 * symmetric != 0 stores the mirror arc of every listed edge (row u holds
 * (v, w) and row v holds (u, w); self-loops twice); 0 stores one arc per
 * edge.  stable != 0 keeps the reference's arc order exactly (input order,
 * mirror right after the original; CUB radix sort by row, at most 2^32-1
 * arcs); stable == 0 fills rows through atomic cursors (order unspecified --
 * the pull accumulator is exact integer arithmetic, so Z does not depend on
 * it).  offsets[n+1] int64; targets[arcs] int32; weights[arcs] float (NULL
 * if w NULL).  The pull layout is the symmetric CSR of EVERY list, because
 * the edge pass applies both updates per listed edge whatever `directed`
 * says (encoder.py:106-120). */
int gee_build_csr(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                  int64_t n, int32_t symmetric, int32_t stable, int64_t *offsets,
                  int32_t *targets, float *weights, void *stream);
int gee_build_sym_csr(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                      int64_t n, int64_t *offsets, int32_t *targets, float *weights,
                      void *stream);

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
 * gee_build_csr or gee_embed_coo.  rows[arcs] int32. */
int gee_csr_rows(const int64_t *offsets, int64_t n, int64_t arcs, int32_t *rows, void *stream);

/* Graph preparation: sort every row's arcs by target (stable, weights
 * follow).  The pull's sums are exact integers, so Z is unchanged; sorted
 * targets (label-table slots after gee_hot_encode) let a warp's 32
 * consecutive label lookups share sectors.  Allocates scratch; blocks. */
int gee_sort_rows(const int64_t *offsets, int64_t n, int32_t *targets, float *w, void *stream);

/* Graph preparation: pad every row to a multiple of `align` arcs with
 * (sentinel slot, weight 0) arcs.  The sentinel slot's label is 0
 * (unlabeled: gee_build_projection writes it), so pads add nothing.  With
 * align = 8 every lane of the block reducer owns arcs of a single row.
 * gee_pad_offsets writes the padded offsets and returns the padded arc
 * count (blocks); gee_pad_rows copies the arcs. */
int gee_pad_offsets(const int64_t *offsets, int64_t n, int64_t align, int64_t *padded_offsets,
                    int64_t *padded_arcs, void *stream);
int gee_pad_rows(const int64_t *offsets, const int64_t *padded_offsets, int64_t n, const int32_t *targets,
                 const float *w, int32_t sentinel, int32_t *padded_targets, float *padded_w, void *stream);

/* Graph statistics that size the pull accumulator (host outputs):
 * max over rows of sum |w| (or max degree if w NULL), min nonzero |w|,
 * max |w|, and whether any weight is non-finite. */
int gee_graph_stats(const int64_t *offsets, const float *w, int64_t n, int64_t arcs,
                    double *max_row_abs, double *min_abs_nz, double *max_abs,
                    int32_t *nonfinite, void *stream);

/* Hot-label tier (see gee_hot.cu): gee_hot_plan ranks vertices by degree
 * offsets[v+1]-offsets[v] (descending, ties by id) and marks the top
 * max_hot with degree >= min_degree: hot_rank[v] = rank or -1,
 * hot_vertex[rank] = v (may be NULL), *n_hot (host) = count.
 * gee_hot_encode rewrites CSR targets into label-table slots: rank for hot
 * vertices, n_hot + v otherwise. */
int gee_hot_plan(const int64_t *offsets, int64_t n, int64_t max_hot, int64_t min_degree,
                 int32_t *hot_rank, int32_t *hot_vertex, int64_t *n_hot, void *stream);
int gee_hot_encode(int32_t *targets, int64_t arcs, const int32_t *hot_rank, int64_t n_hot,
                   void *stream);

/* Wide-embedding pull (any k; the default for k > 255, BASELINE C5): the
 * label gather fused with a per-row class window.  Replaces the parallel
 * arc wave of embed_parallel (_kernels.py:138-207, SOURCE_ONLY arcs of the
 * symmetric CSR) for wide K: one warp per row of <= 2048 arcs (shared-memory
 * K-bin window, whole Z row written with 16-byte streaming stores), one CTA
 * per heavy row listed in heavy_rows (rows > 2048 arcs, u64 window).  Every
 * Z row is written exactly once, zeros included; exact integer sums (unit:
 * counts, weighted: q = rint(w 2^scale_exp) from gee_block_scale_exp), so Z
 * is bit-identical to the other pull reducers.  Targets are label-table
 * slots (gee_hot_encode), w == NULL for unit weights. */
int gee_reduce_wide(const int64_t *offsets, int64_t n, const int32_t *targets, const float *w,
                    const void *table, int32_t k, int32_t scale_exp, const double *inv,
                    const int32_t *heavy_rows, int64_t n_heavy, float *z, void *stream);

/* Row-sparse Z for the device -> host copy of a streamed pass (the
 * caller-owned dense `out` of embed_parallel, encoder.py:143-194, rebuilt on
 * the host by gee_io_expand_rows in include/gee_io.h).  For rows [0, rows)
 * of a row-major (rows, k) f32 Z:
 *   mask[r * mw + j] (u64, mw = ceil(k / 64)): bit c set iff Z[r, 64 j + c]
 *                    has a nonzero bit pattern;
 *   vals:            the nonzero values, row-major (capacity rows * k);
 *   block_off[b]:    index in vals of the first value of row
 *                    b * GEE_ZC_BLOCK_ROWS (gee_zc_blocks(rows) + 1 entries;
 *                    the last one is the nonzero count).
 * Three launches (mask + counts, scan, scatter); no allocation. */
#ifndef GEE_ZC_BLOCK_ROWS
#define GEE_ZC_BLOCK_ROWS 1024
#endif
int64_t gee_zc_blocks(int64_t rows);
int gee_z_compact(const float *z, int64_t rows, int32_t k, unsigned long long *mask, int64_t *block_off,
                  float *vals, void *stream);

/* Compressed graph for the host -> device path (csrc/gee_pack.cu).  The
 * reference passes its CsrGraph to embed_parallel in host memory
 * (encoder.py:123-194, graph.py:54-91); these code the prepared, padded,
 * slot-sorted CSR in groups of 8 arcs so fewer bytes cross PCIe:
 *   ctl:  one byte per group ((b-1) | pads << 5), b = 1..32 bits per value;
 *   payload: the real arcs' targets as b-bit deltas in one little-endian
 *         stream of u32 words (a row's first arc absolute); row starts are
 *         recovered from the padded offsets;
 *   wctl: one byte per group (B | e << 2): B = 1..3 bytes per weight of an
 *         integer k with w = k * 2^-e exactly (lossless group fixed point),
 *         B = 0 raw f32 bits;
 *   wpayload: the real arcs' weights (no pads).
 * gee_pack_targets (graph preparation; allocates, synchronises) writes
 * ctl[padded_arcs/8], up to 4*padded_arcs payload bytes (4-byte aligned)
 * and, given the padded weights, wctl[padded_arcs/8] and up to
 * 4*padded_arcs wpayload bytes, returning both sizes (the payload size is a
 * whole number of u32 words).  gee_unpack_targets (stream-ordered, no
 * allocation; scratch >= gee_unpack_scratch_bytes(groups)) takes the chunk's
 * padded offsets (int64[rows+1], chunk-relative) and rebuilds the padded
 * targets (pads = sentinel) and, given wpayload and either wctl or
 * wctl_uniform >= 0 (the wctl byte of every group), the padded weights
 * (pads 0), bit for bit.  The payload buffer must extend 4 bytes past the
 * packed size (the bit reader loads the word after a value's last word). */
size_t gee_unpack_scratch_bytes(int64_t groups);
int gee_pack_targets(const int64_t *padded_offsets, int64_t rows, const int32_t *targets, const float *w_padded,
                     int64_t padded_arcs, int32_t sentinel, uint8_t *ctl, uint8_t *payload, int64_t *payload_bytes,
                     uint8_t *wctl, uint8_t *wpayload, int64_t *wpayload_bytes, void *stream);
int gee_unpack_targets(const uint8_t *ctl, const uint8_t *payload, int64_t groups, const int64_t *padded_offsets,
                       int64_t rows, const uint8_t *wctl, int32_t wctl_uniform, const uint8_t *wpayload,
                       int32_t sentinel, int32_t *targets, float *w_padded, void *scratch, size_t scratch_bytes,
                       void *stream);

/* Chunk-relative CSR offsets travel host -> device as int32 (half the
 * bytes); widen them to the int64 the pull reads (stream-ordered). */
int gee_widen_offsets(const int32_t *in, int64_t count, int64_t *out, void *stream);

/* Class stream: cls[e] = table[targets[e]] (u8, k <= 255) for every arc of
 * a pull layout -- the random half of the pull pass (the hottest label-table
 * slots staged in a packed shared-memory head of head_bytes, -1 = the tuned
 * default of 96 KB, 0 = none). */
int gee_gather_labels(const int32_t *targets, int64_t arcs, const void *table, int64_t n_hot,
                      int32_t k, uint8_t *cls, void *stream);
int gee_gather_labels_head(const int32_t *targets, int64_t arcs, const void *table, int64_t n_hot,
                           int32_t k, int64_t head_bytes, uint8_t *cls, void *stream);

/* Graph preparation for the split pull: list the rows with more than
 * heavy_arcs arcs (heavy_rows[n], count in *n_heavy, host; allocates,
 * synchronises). */
int gee_reduce_heavy_plan(const int64_t *offsets, int64_t n, int64_t heavy_arcs,
                          int32_t *heavy_rows, int64_t *n_heavy, void *stream);
/* ---------------------------------------------------------------- K4 ----
 * Pull (row-owner) edge map, split in two: gee_gather_labels (class stream)
 * then the segmented class reduction below.  Together they replace
 * embed_parallel's zero wave + arc wave (encoder.py:123-194, zero_worker
 * _kernels.py:124-135, arc_pass_worker _kernels.py:138-207) for SOURCE_ONLY
 * (symmetric) storage, k <= 255 (wider k: gee_reduce_wide).  Per row x:
 *     Z[x, c] = inv[c+1] * sum_{arcs x->v, Y[v]=c+1} w
 * accumulated exactly in integers (unit weights: counts; weighted: fixed
 * point q = rint(w * 2^scale_exp), scale_exp from gee_block_scale_exp, signed
 * weights allowed), so Z is bit-stable run to run and independent of arc
 * order.
 *
 * Block reduction over PADDED rows (gee_pad_rows, align 8): one warp per 32
 * consecutive rows (coalesced offsets, arcs streamed through a cp.async
 * ring, slot windows of shared-memory atomics); writes every row with at
 * most heavy_arcs (<= 2048) arcs, empty rows as zeros, and leaves the longer
 * rows to gee_reduce_heavy.  z 16-byte aligned. */
int gee_reduce_blocks_pad8(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w,
                           int32_t scale_exp, const double *inv, int32_t k, int64_t heavy_arcs, float *z,
                           void *stream);
/* The same reduction for a CSR in which NO row has more than 2048 arcs (the
 * caller's guarantee: the tile layout keeps the heavy rows' arcs outside the
 * CSR): the heavy-row skipping is compiled out (C4 7.61 -> 7.50 ms). */
int gee_reduce_blocks_light(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w,
                            int32_t scale_exp, const double *inv, int32_t k, float *z, void *stream);
/* gee_reduce_blocks_light with the shortest rows flagged: bit i of
 * short_rows[b] (uint32 per 32-row block, device) is set when row 32 b + i
 * holds 1 .. short_arcs arcs before padding (short_arcs in 1..4; its padded
 * run is [the arcs | pads]).  Weighted graphs: the lane that holds such a
 * row's chunk combines its arcs in registers and stores the row's nonzero
 * Z entries itself, without a window slot.  Same bits.  short_rows NULL or
 * unit weights: exactly gee_reduce_blocks_light. */
int gee_reduce_blocks_short(const int64_t *offsets, int64_t n, const uint8_t *cls, const float *w,
                            int32_t scale_exp, const double *inv, int32_t k, const uint32_t *short_rows,
                            int32_t short_arcs, float *z, void *stream);

/* Heavy rows (longer than the block reducer's heavy_arcs) as work items:
 * item i covers arcs [item_first[i], item_end[i]) of row item_row[i]
 * (cls / w hold `arcs` entries)
 * (at most 65536 arcs).  item_slot[i] < 0: the item is its row's only one and
 * writes the Z row; otherwise it adds into mega_acc[item_slot[i]] (int64
 * [n_mega x k], zero on entry, left zero on exit) and a finalize writes the
 * Z rows of mega_rows.  Items are fetched dynamically through *counter
 * (device int64 scratch), so list them largest first.  Weighted graphs need
 * gee_block_scale_exp's exponent.  Graph preparation builds the items (device.py
 * DeviceGraph._plan_heavy). */
int gee_reduce_heavy(const uint8_t *cls, const float *w, int64_t arcs, int32_t scale_exp, const double *inv,
                     int32_t k, const int64_t *item_first, const int64_t *item_end, const int32_t *item_row,
                     const int32_t *item_slot, int64_t n_items, const int32_t *mega_rows, int64_t n_mega,
                     void *mega_acc, int64_t *counter, float *z, void *stream);

/* Tile-major heavy region (graph preparation + its gather; round 2).  The
 * reference's arc wave looks a label up per arc (arc_pass_worker,
 * _kernels.py:183-207); here the heavy rows' TARGETS are regrouped by slot
 * tile so those lookups hit shared memory, while their class bytes and
 * weights stay row-major for gee_reduce_heavy.
 *   gee_tile_bounds  bounds[b * n_heavy + j] = first arc of heavy row
 *       heavy_rows[j] (rows sorted by slot) whose slot is >= thresholds[b].
 *   gee_span_copy    span s: out[dst_first[s] .. + src_len[s]) = in[src_first[s]
 *       ..), padded with (sentinel, 0) up to dst_len[s] (int64 arrays);
 *       targets / out_targets or w / out_w may be NULL (that array is skipped).
 *   gee_gather_tiles for the arcs [tile_start[0], tile_start[n_tiles]) of
 *       `targets`, where [tile_start[t], tile_start[t+1]) (multiples of 16)
 *       holds slots of tile t = [t * tile_slots, (t + 1) * tile_slots) or
 *       padding (any other slot: class 0): the class of arc e goes to
 *       cls[16 * group_dst[(e - region_start) / 16] + e % 16] -- the 16-arc
 *       group's place in the row-major class stream.  Tile labels are staged
 *       in shared memory (tile_slots bytes, a multiple of 16).
 *   gee_gather_scatter the same scatter for arcs [first, end) whose slots
 *       are looked up in the table itself (the tail past the last tile). */
int gee_tile_bounds(const int64_t *offsets, const int32_t *heavy_rows, int64_t n_heavy, const int32_t *targets,
                    const int64_t *thresholds, int32_t n_thresholds, int64_t *bounds, void *stream);
int gee_span_copy(int64_t n_spans, const int64_t *src_first, const int64_t *src_len, const int64_t *dst_first,
                  const int64_t *dst_len, const int32_t *targets, const float *w, int32_t sentinel,
                  int32_t *out_targets, float *out_w, void *stream);
int gee_gather_tiles(const int32_t *targets, const int64_t *tile_start, int32_t n_tiles, int64_t region_start,
                     const int32_t *group_dst, const void *table, int64_t table_bytes, int64_t tile_slots, int32_t k,
                     uint8_t *cls, void *stream);
int gee_gather_scatter(const int32_t *targets, int64_t first, int64_t end, int64_t region_start,
                       const int32_t *group_dst, const void *table, int32_t k, uint8_t *cls, void *stream);

/* Fixed-point exponent valid for every pull reducer: the largest e with
 * max_row_abs * 2^e < 2^62 (64-bit row sums) and max_abs * 2^e < 2^41 (the
 * signed split planes of a 2048-arc row cannot overflow).
 * *rel_err = 2^-(e+1)/min_abs_nz (host): the worst per-term rounding,
 * relative to the smallest nonzero |w|. */
int gee_block_scale_exp(double max_row_abs, double max_abs, double min_abs_nz, int32_t *scale_exp,
                        double *rel_err);

#ifdef __cplusplus
}
#endif
#endif /* GEE_B200_H */
