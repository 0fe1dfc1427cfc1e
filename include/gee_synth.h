/*
 * gee_synth.h -- seeded synthetic graph/label generators (benchmark harness
 * support in libgee_b200.so; not part of the reference's hot path).
 *
 * The reference's only generator is generate_erdos_renyi
 * (/root/reference/pkg/src/gee/graph.py:187-201) plus random_labels
 * (labeling.py:87-104); the benchmark configurations also need R-MAT.
 * All streams are counter-based (element i depends only on seed and i),
 * so [first, first+count) slices can be generated independently and
 * restated exactly in numpy (paper_2402_04403_b200/synth.py).
 */
#ifndef GEE_SYNTH_H
#define GEE_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* splitmix64(splitmix64(seed ^ tag*C) + ctr): the word every stream uses. */
uint64_t gee_synth_word(uint64_t seed, uint64_t tag, uint64_t ctr);

/* R-MAT edges [first, first+count): probabilities a, b, c (d = 1-a-b-c);
 * w may be NULL (unit weights).  scramble_ids applies the seeded vertex
 * permutation. */
int gee_synth_rmat(int32_t *src, int32_t *dst, float *w, int64_t first, int64_t count,
                   int32_t scale, double a, double b, double c, uint64_t seed,
                   int32_t scramble_ids, void *stream);

/* G(n, s) with replacement, edges [first, first+count). */
int gee_synth_er(int32_t *src, int32_t *dst, float *w, int64_t first, int64_t count,
                 int64_t n, uint64_t seed, void *stream);

/* y[i] uniform in {1..k}. */
int gee_synth_uniform_labels(int32_t *y, int64_t n, int32_t k, uint64_t seed, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GEE_SYNTH_H */
