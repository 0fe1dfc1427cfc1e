/*
 * gee_oracle.c -- CPU restatement of the reference GEE edge pass.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py's reference arm.  The product path
 * (paper_2402_04403_b200/) never links, loads or calls it; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs do.
 *
 * Every function restates one piece of the reference package
 * (/root/reference/pkg/src/gee, "gee-embed" 0.1.0) in plain C, in the
 * reference's own dtypes: int64 node ids / labels, float64 weights,
 * float64 Z.  Citations are file:line into that package.
 *
 * Pinned against: the reference's known-answer tests (CHAIN, projection
 * KATs, mirror arcs, star, two-hub race graph, class counts) and golden
 * vectors produced by importing the reference itself
 * (tests/golden/make_golden.py writes tests/golden/ fixtures); see
 * tests/test_oracle.py.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* np.bincount(labels, minlength=k+1)  -- encoder.py:87, labeling.py:107-109.
 * Returns -1 if a label falls outside [0, k] (LabelVector forbids it,
 * labeling.py:24-29). */
int oracle_bincount(const int64_t *labels, int64_t n, int64_t k, int64_t *counts)
{
    memset(counts, 0, sizeof(int64_t) * (size_t)(k + 1));
    for (int64_t i = 0; i < n; i++) {
        int64_t c = labels[i];
        if (c < 0 || c > k)
            return -1;
        counts[c]++;
    }
    return 0;
}

/* build_projection -- encoder.py:80-103: inv[c] = 1/count[c] for nonempty
 * classes (inv[0] = 0), row_value = inv[labels]. */
int oracle_build_projection(const int64_t *labels, int64_t n, int64_t k,
                            int64_t *counts, double *inv, double *row_value)
{
    if (oracle_bincount(labels, n, k, counts))
        return -1;
    inv[0] = 0.0;
    for (int64_t c = 1; c <= k; c++)
        inv[c] = counts[c] > 0 ? 1.0 / (double)counts[c] : 0.0;
    if (row_value)
        for (int64_t i = 0; i < n; i++)
            row_value[i] = inv[labels[i]];
    return 0;
}

/* serial_pass -- _kernels.py:210-226 (called by embed_serial,
 * encoder.py:106-120).  Both updates for every listed edge, in list order,
 * f64; Z is NOT zeroed here (embed_serial allocates np.zeros, :117). */
void oracle_serial_pass(const int64_t *src, const int64_t *dst, const double *w,
                        int64_t s, const int64_t *labels, const double *wrow,
                        double *z, int64_t k)
{
    for (int64_t i = 0; i < s; i++) {
        int64_t u = src[i], v = dst[i];
        double wi = w[i];
        int64_t yv = labels[v];
        if (yv != 0)
            z[u * k + (yv - 1)] += wrow[v] * wi;
        int64_t yu = labels[u];
        if (yu != 0)
            z[v * k + (yu - 1)] += wrow[u] * wi;
    }
}

/* build_csr + csr_fill -- graph.py:159-184, _kernels.py:229-238.
 * Counting sort keeping input order; undirected input inserts the mirror arc
 * right after the original.  offsets has n+1 entries; targets/weights have
 * s (directed) or 2s (undirected) entries.  Caller allocates. */
void oracle_build_csr(const int64_t *src, const int64_t *dst, const double *w,
                      int64_t s, int64_t n, int directed,
                      int64_t *offsets, int32_t *targets, double *weights)
{
    memset(offsets, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < s; i++) {
        offsets[src[i] + 1]++;
        if (!directed)
            offsets[dst[i] + 1]++;
    }
    for (int64_t r = 0; r < n; r++)
        offsets[r + 1] += offsets[r];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    memcpy(cursor, offsets, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < s; i++) {
        int64_t p = cursor[src[i]]++;
        targets[p] = (int32_t)dst[i];
        weights[p] = w[i];
        if (!directed) {
            int64_t q = cursor[dst[i]]++;
            targets[q] = (int32_t)src[i];
            weights[q] = w[i];
        }
    }
    free(cursor);
}

/* ---- the parallel CPU edge map: embed_parallel (encoder.py:123-194) ---- */

/* _atomic_add_f64 -- _kernels.py:92-106: CAS retry loop on the 64-bit
 * pattern (monotonic ordering). */
static inline void atomic_add_f64(double *p, double delta)
{
    uint64_t *bits = (uint64_t *)p;
    uint64_t old = __atomic_load_n(bits, __ATOMIC_RELAXED);
    for (;;) {
        double cur;
        memcpy(&cur, &old, 8);
        double nv = cur + delta;
        uint64_t nb;
        memcpy(&nb, &nv, 8);
        if (__atomic_compare_exchange_n(bits, &old, nb, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED))
            return;
    }
}

typedef struct {
    const int64_t *offsets;
    const int32_t *targets;
    const double *weights;
    int unit_weights;
    const int32_t *labels;
    const double *wrow;
    double *z;
    int64_t n, k;
    int both_updates, use_atomics;
    int64_t *cursor;
    int64_t chunk;
    int64_t zlen;
} arc_job;

/* zero_worker -- _kernels.py:124-135 (chunked first-touch zeroing). */
static void *zero_worker(void *arg)
{
    arc_job *j = (arc_job *)arg;
    for (;;) {
        int64_t start = __atomic_fetch_add(j->cursor, j->chunk, __ATOMIC_RELAXED);
        if (start >= j->zlen)
            return NULL;
        int64_t stop = start + j->chunk < j->zlen ? start + j->chunk : j->zlen;
        memset(j->z + start, 0, sizeof(double) * (size_t)(stop - start));
    }
}

/* arc_pass_worker -- _kernels.py:138-207: dynamic node chunks off a shared
 * cursor; per arc the source-side update, plus the destination-side update
 * when both_updates (directed storage, EdgeAccounting.BOTH_ENDPOINTS). */
static void *arc_worker(void *arg)
{
    arc_job *j = (arc_job *)arg;
    const int64_t k = j->k;
    for (;;) {
        int64_t start = __atomic_fetch_add(j->cursor, j->chunk, __ATOMIC_RELAXED);
        if (start >= j->n)
            return NULL;
        int64_t stop = start + j->chunk < j->n ? start + j->chunk : j->n;
        for (int64_t u = start; u < stop; u++) {
            int64_t yu = j->labels[u];
            double wu = j->wrow[u];
            int64_t lo = j->offsets[u], hi = j->offsets[u + 1];
            double *zu = j->z + u * k;
            for (int64_t e = lo; e < hi; e++) {
                if (e + 8 < hi) { /* PREFETCH_DIST = 8, _kernels.py:16-19,184-188 */
                    int64_t vn = j->targets[e + 8];
                    __builtin_prefetch(j->labels + vn, 0, 3);
                    if (j->both_updates && yu != 0)
                        __builtin_prefetch(j->z + vn * k + (yu - 1), 1, 3);
                }
                int64_t v = j->targets[e];
                int64_t yv = j->labels[v];
                double w = j->unit_weights ? 1.0 : j->weights[e];
                if (yv != 0) {
                    double d = j->wrow[v] * w;
                    if (j->use_atomics) atomic_add_f64(zu + (yv - 1), d);
                    else zu[yv - 1] += d;
                }
                if (j->both_updates && yu != 0) {
                    double d = wu * w;
                    double *p = j->z + v * k + (yu - 1);
                    if (j->use_atomics) atomic_add_f64(p, d);
                    else *p += d;
                }
            }
        }
    }
}

static void run_wave(int workers, void *(*fn)(void *), arc_job *job)
{
    if (workers == 1) { /* _run_wave runs inline for one worker, encoder.py:199-201 */
        fn(job);
        return;
    }
    pthread_t *t = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)workers);
    for (int i = 0; i < workers; i++)
        pthread_create(&t[i], NULL, fn, job);
    for (int i = 0; i < workers; i++)
        pthread_join(t[i], NULL);
    free(t);
}

/* embed_parallel's zero wave + arc wave (encoder.py:164-193), chunk sizes as
 * the reference picks them (_ZERO_CHUNK = 2^21, _NODE_CHUNK_CAP = 8192,
 * encoder.py:33-34,171,174).  z is (n, k) row-major f64, overwritten. */
void oracle_embed_parallel(const int64_t *offsets, const int32_t *targets,
                           const double *weights, int unit_weights,
                           const int32_t *labels, const double *wrow,
                           double *z, int64_t n, int64_t k, int both_updates,
                           int use_atomics, int workers)
{
    int64_t zlen = n * k;
    if (zlen == 0)
        return;
    int64_t cursor = 0;
    arc_job j = {offsets, targets, weights, unit_weights, labels, wrow, z, n, k,
                 both_updates, use_atomics, &cursor, 0, zlen};
    int64_t zc = zlen / workers;
    j.chunk = zc < 1 ? 1 : (zc > (1 << 21) ? (1 << 21) : zc);
    run_wave(workers, zero_worker, &j);
    if (offsets[n] == 0)
        return;
    cursor = 0;
    int64_t nc = n / ((int64_t)workers * 8);
    if (nc < 1) nc = 1;
    j.chunk = nc > 8192 ? 8192 : nc;
    run_wave(workers, arc_worker, &j);
}

/* atomic_add_hammer -- _kernels.py:109-114 (test hook). */
typedef struct { double *z; int64_t idx, reps; double delta; } hammer_job;
static void *hammer(void *a)
{
    hammer_job *h = (hammer_job *)a;
    for (int64_t i = 0; i < h->reps; i++)
        atomic_add_f64(h->z + h->idx, h->delta);
    return NULL;
}
void oracle_atomic_hammer(double *z, int64_t idx, int64_t reps, double delta, int threads)
{
    hammer_job h = {z, idx, reps, delta};
    pthread_t t[64];
    if (threads > 64) threads = 64;
    for (int i = 0; i < threads; i++) pthread_create(&t[i], NULL, hammer, &h);
    for (int i = 0; i < threads; i++) pthread_join(t[i], NULL);
}

/* Sampled-row streaming oracle: accumulate only updates whose
 * target row r has keep[r] != 0 into zs[slot[r], :], in f64, in list order
 * -- the serial_pass rule restricted to a row sample, so that graphs whose
 * full f64 Z does not fit in host memory can still be checked.  Inputs are
 * the device dtypes (int32 ids, float32 weights, int32 labels) upcast the
 * way the reference's EdgeList.__post_init__ does (graph.py:33-36). */
void oracle_sampled_rows(const int32_t *src, const int32_t *dst, const float *w,
                         int64_t s, const int32_t *labels, const double *inv,
                         const int64_t *slot, double *zs, int64_t k)
{
    for (int64_t i = 0; i < s; i++) {
        int64_t u = src[i], v = dst[i];
        double wi = w ? (double)w[i] : 1.0;
        int64_t su = slot[u], sv = slot[v];
        if (su >= 0) {
            int64_t yv = labels[v];
            if (yv) zs[su * k + (yv - 1)] += inv[yv] * wi;
        }
        if (sv >= 0) {
            int64_t yu = labels[u];
            if (yu) zs[sv * k + (yu - 1)] += inv[yu] * wi;
        }
    }
}

/* The same sampled-row rule, threaded, plus the column mass, for the
 * full-size configurations (C3/C4/C5 at BASELINE sizes: up to 1.8e9 listed
 * edges, whose f64 Z does not fit the sampled-row budget of a serial scan).
 * Each thread takes a contiguous slice of the listed edges and accumulates
 * into its own zs / mass copies, which are then summed in thread order:
 * the f64 summation order differs from list order (as the reference's own
 * embed_parallel's does), nothing else.  `keep` is a bitmap of the sampled
 * rows (n bits) so that most edges are rejected from a 16 MB table;
 * slot[r] is the row's index in zs.  mass[c] = sum over listed edges of
 * w * inv[c] * ([Y[v]=c] + [Y[u]=c]) = sum_x Z[x, c] (the mass accounting
 * of the reference's test_parallel.py:54-64), c = 1..k, mass[0] unused. */
static inline double inv_mul(double inv, double w) { return inv * w; }

typedef struct {
    const int32_t *src, *dst;
    const float *w;
    int64_t lo, hi;
    const int32_t *labels;
    const double *inv;
    const uint64_t *keep;
    const int32_t *slot;
    double *zs, *mass;
    int64_t k;
} sampled_job;

static void *sampled_worker(void *arg)
{
    sampled_job *j = (sampled_job *)arg;
    const int64_t k = j->k;
    for (int64_t i = j->lo; i < j->hi; i++) {
        const int64_t u = j->src[i], v = j->dst[i];
        const double wi = j->w ? (double)j->w[i] : 1.0;
        const int64_t yu = j->labels[u], yv = j->labels[v];
        if (yv) j->mass[yv] += inv_mul(j->inv[yv], wi);
        if (yu) j->mass[yu] += inv_mul(j->inv[yu], wi);
        if (yv && ((j->keep[u >> 6] >> (u & 63)) & 1))
            j->zs[(int64_t)j->slot[u] * k + (yv - 1)] += j->inv[yv] * wi;
        if (yu && ((j->keep[v >> 6] >> (v & 63)) & 1))
            j->zs[(int64_t)j->slot[v] * k + (yu - 1)] += j->inv[yu] * wi;
    }
    return NULL;
}

void oracle_sampled_rows_par(const int32_t *src, const int32_t *dst, const float *w, int64_t s,
                             const int32_t *labels, const double *inv, const uint64_t *keep, const int32_t *slot,
                             int64_t n_rows, double *zs, double *mass, int64_t k, int threads)
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t t[256];
    sampled_job jobs[256];
    const size_t zlen = (size_t)(n_rows * k);
    for (int i = 0; i < threads; i++) {
        sampled_job jb = {src, dst, w, s * i / threads, s * (i + 1) / threads, labels, inv, keep, slot,
                          (double *)calloc(zlen ? zlen : 1, sizeof(double)),
                          (double *)calloc((size_t)(k + 1), sizeof(double)), k};
        jobs[i] = jb;
        pthread_create(&t[i], NULL, sampled_worker, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(t[i], NULL);
    memset(zs, 0, zlen * sizeof(double));
    memset(mass, 0, (size_t)(k + 1) * sizeof(double));
    for (int i = 0; i < threads; i++) {
        for (size_t q = 0; q < zlen; q++) zs[q] += jobs[i].zs[q];
        for (int64_t c = 0; c <= k; c++) mass[c] += jobs[i].mass[c];
        free(jobs[i].zs);
        free(jobs[i].mass);
    }
}

/* ---- seeded synthetic inputs for the CPU arm (bench.py --impl reference) ----
 *
 * A C restatement of the counter-based generator the workload uses
 * (paper_2402_04403_b200/synth.py: word_numpy, rmat_edges_numpy,
 * uniform_labels_numpy), so the reference arm builds the SAME C4 graph on the
 * host without loading the product library.  Pinned bit for bit against the
 * numpy restatement (tests/test_oracle.py) and, on the GPU, against
 * gee_synth_rmat (tests/test_gpu_parity.py). */
static inline uint64_t sm64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static inline uint64_t synth_word(uint64_t seed, uint64_t tag, uint64_t ctr)
{
    return sm64(sm64(seed ^ (tag * 0xD1B54A32D192ED03ull)) + ctr);
}

static inline uint64_t scramble(uint64_t x, int scale, uint64_t m1, uint64_t m2)
{
    const uint64_t mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1ull);
    const int h = scale / 2 > 1 ? scale / 2 : 1;
    x = (x * m1) & mask;
    x ^= x >> h;
    x = (x * m2) & mask;
    x ^= x >> (h + (scale & 1));
    return (x * m1) & mask;
}

typedef struct {
    int32_t *src, *dst;
    float *w;
    int64_t first, s;
    int scale, scramble;
    uint64_t seed, ta, tab, tabc, m1, m2;
    int64_t lo, hi;
} rmat_job;

static void *rmat_worker(void *arg)
{
    rmat_job *j = (rmat_job *)arg;
    for (int64_t q = j->lo; q < j->hi; q++) {
        const uint64_t i = (uint64_t)(j->first + q);
        uint64_t u = 0, v = 0, bits = 0;
        for (int lvl = 0; lvl < j->scale; lvl++) {
            if ((lvl & 1) == 0)
                bits = synth_word(j->seed, 1, i * 32u + (uint64_t)(lvl >> 1));
            const uint64_t r = (lvl & 1) ? (bits >> 32) : (bits & 0xFFFFFFFFull);
            const uint64_t bu = r >= j->tab;
            const uint64_t bv = ((r >= j->ta) && (r < j->tab)) || (r >= j->tabc);
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        if (j->scramble) {
            u = scramble(u, j->scale, j->m1, j->m2);
            v = scramble(v, j->scale, j->m1, j->m2);
        }
        j->src[q] = (int32_t)u;
        j->dst[q] = (int32_t)v;
        if (j->w)
            j->w[q] = 1.0f - (float)(synth_word(j->seed, 2, i) >> 40) * (1.0f / 16777216.0f);
    }
    return NULL;
}

/* rmat_edges_numpy(scale, s, seed, weighted, a, b, c, scramble, first). */
void oracle_rmat(int32_t *src, int32_t *dst, float *w, int64_t first, int64_t s, int scale, double a,
                 double b, double c, uint64_t seed, int do_scramble, int threads)
{
    const double two32 = 4294967296.0;
    rmat_job base = {src, dst, w, first, s, scale, do_scramble, seed,
                     (uint64_t)(a * two32), (uint64_t)((a + b) * two32), (uint64_t)((a + b + c) * two32),
                     sm64(seed ^ 0x5EED1ull) | 1ull, sm64(seed ^ 0x5EED2ull) | 1ull, 0, 0};
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t t[256];
    rmat_job jobs[256];
    for (int i = 0; i < threads; i++) {
        jobs[i] = base;
        jobs[i].lo = s * i / threads;
        jobs[i].hi = s * (i + 1) / threads;
        pthread_create(&t[i], NULL, rmat_worker, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(t[i], NULL);
}

/* uniform_labels_numpy(n, k, seed): 1 + ((word(seed, 4, i) >> 32) * k >> 32). */
void oracle_uniform_labels(int32_t *y, int64_t n, int64_t k, uint64_t seed)
{
    for (int64_t i = 0; i < n; i++)
        y[i] = (int32_t)(1 + (((synth_word(seed, 4, (uint64_t)i) >> 32) * (uint64_t)k) >> 32));
}

/* ---- build_csr for the CPU arm at full size ----
 *
 * graph.py:159-184 (directed storage: one arc per listed edge) with the
 * degree count and the fill spread over threads (atomic per-row cursors),
 * in the reference's dtypes: int64 offsets, int32 targets, f64 weights.
 * Arc order inside a row is not the reference's (that one is serial and
 * stable, oracle_build_csr above); it only changes the f64 summation order
 * of the timed pass, not its work.  Graph construction is outside the
 * reference's timed region (bench.py:1-7). */
typedef struct {
    const int32_t *src, *dst;
    const float *w;
    int64_t lo, hi;
    int64_t *cnt;
    int32_t *targets;
    double *weights;
} csr_job;

static void *csr_count(void *arg)
{
    csr_job *j = (csr_job *)arg;
    for (int64_t i = j->lo; i < j->hi; i++)
        __atomic_fetch_add(&j->cnt[j->src[i]], 1, __ATOMIC_RELAXED);
    return NULL;
}

static void *csr_fill_par(void *arg)
{
    csr_job *j = (csr_job *)arg;
    for (int64_t i = j->lo; i < j->hi; i++) {
        const int64_t p = __atomic_fetch_add(&j->cnt[j->src[i]], 1, __ATOMIC_RELAXED);
        j->targets[p] = j->dst[i];
        if (j->weights) j->weights[p] = j->w ? (double)j->w[i] : 1.0;
    }
    return NULL;
}

void oracle_build_csr_directed_par(const int32_t *src, const int32_t *dst, const float *w, int64_t s, int64_t n,
                                   int64_t *offsets, int32_t *targets, double *weights, int threads)
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    int64_t *cnt = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
    pthread_t t[256];
    csr_job jobs[256];
    for (int i = 0; i < threads; i++) {
        csr_job jb = {src, dst, w, s * i / threads, s * (i + 1) / threads, cnt, targets, weights};
        jobs[i] = jb;
        pthread_create(&t[i], NULL, csr_count, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(t[i], NULL);
    offsets[0] = 0;
    for (int64_t r = 0; r < n; r++) {
        offsets[r + 1] = offsets[r] + cnt[r];
        cnt[r] = offsets[r];
    }
    for (int i = 0; i < threads; i++) pthread_create(&t[i], NULL, csr_fill_par, &jobs[i]);
    for (int i = 0; i < threads; i++) pthread_join(t[i], NULL);
    free(cnt);
}
