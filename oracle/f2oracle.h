/*
 * f2oracle.h — CPU ORACLE for the GF(2) block decomposition hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (paper_1209_5198_b200, libf2gpu.so) never links or calls it.
 *
 * Plain-C restatement of the reference algorithms (reference = /root/reference,
 * arXiv 1209.5198 artifact).  Every function cites the reference file:line it
 * follows.  Storage layout is the reference's PackedMatrix<uint64_t>
 * (proj/include/f2la/bit_matrix.hpp:74-81): word (i,q) at w[q*stride + i], bit k
 * of word (i,q) = entry (i, 64q+k), padding bits zero.
 *
 * Pinning: random_dense / m4rm_mult / transpose are pinned bit-exactly against
 * the reference headers compiled in place (oracle/_ref, see oracle/Makefile) and
 * the golden fixtures in tests/golden/.  buildZ and decompose_block have no
 * reference code (they are spec/paper only: PAPER.md:960-1017);
 * they are pinned by the SPEC known-answer tests, by property checks
 * (P*A = L*U, rank = Gaussian elimination, B'Z = I) and by agreement with the
 * oracle/_ref decomposition that runs the reference's own build_tables/mult_acc.
 */
#ifndef F2ORACLE_H
#define F2ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- PRNG: xorshift64*  (proj/include/f2la/prng.hpp:18-47) ---- */
uint64_t f2o_rng_seed(uint64_t seed);                 /* prng.hpp:20-21 */
uint64_t f2o_rng_next(uint64_t *state);               /* prng.hpp:23-30 */
uint64_t f2o_bernoulli_threshold(double density);     /* prng.hpp:40-42 */

/* random_dense (bit_matrix.hpp:125-142): one draw per entry, row-major.
 * w must hold ceil(m/64)*stride words and is fully overwritten. */
void f2o_random_dense(uint64_t *w, size_t n, size_t m, size_t stride,
                      double density, uint64_t seed);

/* ---- products ---- */
/* naive triple loop C = A*B (the SPEC.md:524 oracle) */
void f2o_mul_naive(const uint64_t *a, size_t n, size_t k, size_t sa,
                   const uint64_t *b, size_t m, size_t sb,
                   uint64_t *c, size_t sc);
/* m4rm_mult restated (m4rm.hpp:177-196): C = A*B, table size c (0 = cost model) */
void f2o_m4rm_mult(const uint64_t *a, size_t n, size_t k, size_t sa,
                   const uint64_t *b, size_t m, size_t sb,
                   uint64_t *c, size_t sc, unsigned tc);
/* C ^= A*B with A n x k (k<=64, one word per row), B k x m (rows b_row0.. of a
 * word-column-major matrix), i.e. the Schur update E ^= Y*C (m4rm.hpp:140-172). */
void f2o_m4rm_update(uint64_t *c, size_t sc, size_t c_row0,
                     const uint64_t *a_words, size_t n_rows, size_t k_bits,
                     const uint64_t *b, size_t sb, size_t b_row0,
                     size_t n_wcols, unsigned tc);

/* ---- tuning (tuning.hpp:11-41 declarations; formulas SPEC.md:404-434) ---- */
double   f2o_m4rm_cost(unsigned b, unsigned c, double n);
unsigned f2o_optimal_table_size(unsigned b, double n);
size_t   f2o_strassen_threshold(unsigned c);

/* ---- Procedure buildZ, literal transcription ----
 * A: panel words (r of them), modified in place by the row swaps.
 * P[64]: selected pre-swap row (relative) or -1 (insertion).
 * Z[64]: compressed pseudo-inverse rows (bit t = column t, t < rank).
 * swap_b[k] for k < rank: the k-th transposition is (k, swap_b[k]).
 * Returns the rank r_j. */
int f2o_build_z(uint64_t *A, size_t r, int64_t P[64], uint64_t Z[64],
                uint64_t swap_b[64]);

/* ---- decompose_block ----
 * In place on w (the overlay W).
 * perm[n] (uint32, (PA)_i = A_{perm[i]}, bit_matrix.hpp:350), rj[mu].
 * max_panels limits the number of panels processed (bounded CPU samples);
 * pass SIZE_MAX for a full decomposition.  Returns the rank. */
size_t f2o_decompose_block(uint64_t *w, size_t n, size_t m, size_t stride,
                           uint32_t *perm, uint32_t *rj, unsigned tc,
                           size_t max_panels);

/* rank by plain Gaussian elimination on a copy (SPEC.md:526 oracle) */
size_t f2o_rank_ge(const uint64_t *w, size_t n, size_t m, size_t stride);

/* transposed() (bit_matrix.hpp:220-238): out is m x n with stride so */
void f2o_transpose(const uint64_t *w, size_t n, size_t m, size_t stride,
                   uint64_t *out, size_t so);

/* Order-independent digest of an n x m packed matrix (rows < n, word-cols < mu):
 * sum over words of mix64(word ^ f(i,q)).  Also used for uint32 arrays. */
uint64_t f2o_digest(const uint64_t *w, size_t n, size_t m, size_t stride);
uint64_t f2o_digest_u32(const uint32_t *v, size_t n);

/* Given the overlay W + rj, form L (n x rank) and U (rank x m) packed.
 * (SPEC.md:308-316 LUFactors) */
void f2o_extract_lu(const uint64_t *w, size_t n, size_t m, size_t stride,
                    const uint32_t *rj, size_t rank,
                    uint64_t *L, size_t sl, uint64_t *U, size_t su);

/* Freivalds-style check: returns 1 iff (P*A)*X == L*(U*X) for X = 64 random
 * columns drawn from seed.  A is the original input; W/perm/rj the result. */
int f2o_check_plu(const uint64_t *a, const uint64_t *w, size_t n, size_t m,
                  size_t stride, const uint32_t *perm, const uint32_t *rj,
                  uint64_t seed);

int f2o_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
