/* gee_io.h -- native host IO for the GEE path's data formats (libgee_io.so).
 *
 * the reference's text ingestion and binary
 * formats, rebuilt as multithreaded C++ behind a C ABI so that a 1.8e9-edge
 * graph can be parsed, cached and written at storage speed.  Every entry
 * point follows the reference function named in its comment (files under
 * /root/reference/pkg/src/gee): same accepted syntax, same check order, same
 * error text.  Python binds this with ctypes (paper_2402_04403_b200/io.py);
 * a maintainer of the reference would bind it the same way.
 *
 * Conventions
 *   - every call returns a status (GEE_IO_OK = 0); the message, formatted
 *     exactly as the reference's exception text, is in gee_io_last_error()
 *     (thread-local);
 *   - `threads` <= 0 means all hardware threads;
 *   - arrays are caller-owned host memory (pinned or pageable), never freed
 *     here; parse handles own their temporaries until *_free.
 */
#ifndef GEE_IO_H
#define GEE_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    GEE_IO_OK = 0,
    GEE_IO_ERR_OS = 1,      /* open/read/write failed; gee_io_last_errno() has errno (OSError) */
    GEE_IO_ERR_PARSE = 2,   /* malformed text (ParseError, errors.py:8-9) */
    GEE_IO_ERR_FORMAT = 3,  /* malformed binary file (FormatError, errors.py:12-13) */
    GEE_IO_ERR_VALUE = 4,   /* values outside a contract (ValidationError, errors.py:16-17) */
    GEE_IO_ERR_INVALID = 5  /* bad arguments to this API */
};

int gee_io_version(void);
const char *gee_io_last_error(void);
int gee_io_last_errno(void);

/* ---- text edge list: load_edge_list (graph.py:94-145) -------------------
 * Lines end at \n, \r\n or \r (Python universal newlines).  A line whose
 * first byte is '#' is a comment; a line of only whitespace is skipped;
 * otherwise it must hold 2 or 3 whitespace-separated fields: two integer
 * node ids (Python int() syntax: optional sign, ASCII digits, single '_'
 * between digits) and, when `weighted`, a finite Python float() weight.  An
 * unweighted parse ignores a third field, as the reference does.  The first
 * malformed line in file order is reported as
 * "<path>: line <L>: <reason>" with the reference's reasons.  n = 1 + max id
 * (0 for an empty file). */
typedef struct gee_io_edges gee_io_edges;
int gee_io_edges_parse(const char *path, int weighted, int threads, gee_io_edges **out);
int64_t gee_io_edges_count(const gee_io_edges *h);   /* listed edges s */
int64_t gee_io_edges_max_id(const gee_io_edges *h);  /* -1 when s == 0 */
/* Device dtypes (int32 ids, fp32 weights = fp32(f64 parse)); GEE_IO_ERR_VALUE
 * if an id exceeds INT32_MAX (the reference's CSR limit, graph.py:14-15).
 * w may be NULL (unweighted parse: unit weights). */
int gee_io_edges_copy_i32(const gee_io_edges *h, int32_t *src, int32_t *dst, float *w, int threads);
/* Reference dtypes (int64 ids, f64 weights; unweighted -> 1.0). */
int gee_io_edges_copy_i64(const gee_io_edges *h, int64_t *src, int64_t *dst, double *w, int threads);
void gee_io_edges_free(gee_io_edges *h);

/* write_edge_list (graph.py:148-156): "u v\n" when w == NULL, else
 * "u v <repr(float(w))>\n" with Python's shortest round-trip float repr. */
int gee_io_edges_write(const char *path, const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                       int threads);

/* ---- label files: load_labels / write_labels (labeling.py:33-84) -------
 * One field per line (line i labels node i) or "node label" pairs; '#'
 * comments and blank lines skipped; width fixed by the first data line;
 * errors "expected 1 or 2 fields", "mixed label formats", "fields must be
 * integers".  The range checks (node in [0,n), label in [0,k], row count)
 * are value checks done by the caller on the parsed columns, in file order
 * (labeling.py:61-73). */
typedef struct gee_io_labels gee_io_labels;
int gee_io_labels_parse(const char *path, int threads, gee_io_labels **out);
int gee_io_labels_width(const gee_io_labels *h); /* 0 = no data lines, 1 or 2 */
int64_t gee_io_labels_rows(const gee_io_labels *h);
/* col1 is required (and only written) for width 2.  Values beyond int64
 * saturate (they then fail the caller's range check). */
int gee_io_labels_copy(const gee_io_labels *h, int64_t *col0, int64_t *col1);
void gee_io_labels_free(gee_io_labels *h);
int gee_io_labels_write(const char *path, const int32_t *labels, int64_t n, int threads);

/* ---- GEECSR1 binary CSR cache (graph.py:204-235) ------------------------
 * "<8sBBQQ" header (magic "GEECSR1\0", version 1, directed, n, s), then
 * int64 offsets[n+1], int32 targets[s], f64 weights[s], little endian.
 * Header checks in the reference's order: truncated header, bad magic,
 * unsupported version, total size. */
int gee_io_csr_header(const char *path, int *directed, int64_t *n, int64_t *s);
/* Exactly one of w32 / w64 may be non-NULL (f32 = device dtype, converted
 * while reading; f64 = reference dtype); both NULL skips the weights. */
int gee_io_csr_read(const char *path, int64_t n, int64_t s, int64_t *offsets, int32_t *targets, float *w32,
                    double *w64, int threads);
/* w == NULL writes unit weights (1.0). */
int gee_io_csr_write(const char *path, int directed, int64_t n, int64_t s, const int64_t *offsets,
                     const int32_t *targets, const float *w, int threads);

/* ---- GEEEMB1 / csv embedding (encoder.py:209-237) -----------------------
 * binary: "<8sQQ" header (magic "GEEEMB1\0", n, k) + f64 values;
 * csv: numpy savetxt(fmt="%.17g", delimiter=",") byte for byte. */
int gee_io_emb_header(const char *path, int64_t *n, int64_t *k);
int gee_io_emb_read(const char *path, int64_t n, int64_t k, double *z, int threads);
/* z is float (z_is_f64 = 0) or double (1), row-major n x k; fmt 0 = csv,
 * 1 = binary.  f32 values are written as their exact f64 value. */
int gee_io_emb_write(const char *path, const void *z, int z_is_f64, int64_t n, int64_t k, int fmt, int threads);

/* ---- row-sparse Z -> dense host rows (the streamed pass's D2H) --------
 * Inverse of gee_z_compact (include/gee_b200.h): writes rows [0, rows) of
 * the dense row-major (rows, k) f32 Z from the u64 row masks, the packed
 * nonzero values and the per-block value offsets (GEE_ZC_BLOCK_ROWS rows
 * per block), zeros included, with streaming stores; blocks in parallel. */
#ifndef GEE_ZC_BLOCK_ROWS
#define GEE_ZC_BLOCK_ROWS 1024
#endif
int gee_io_expand_rows(const uint64_t *mask, const float *vals, const int64_t *block_off, int64_t rows, int32_t k,
                       float *z, int threads);

#ifdef __cplusplus
}
#endif
#endif /* GEE_IO_H */
