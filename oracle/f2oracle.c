/*
 * f2oracle.c — CPU ORACLE (test infrastructure only; see f2oracle.h header).
 *
 * Plain-C restatement of the reference's GF(2) algorithms.  Nothing here is
 * compiled into, linked by, or called from the product library.
 */
#include "f2oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define WB 64

int f2o_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static inline size_t ceil64(size_t x) { return (x + 63) / 64; }
static inline uint64_t low_mask(size_t k) { return k >= 64 ? ~0ull : ((1ull << k) - 1); }

/* ------------------------------------------------------------------------- */
/* PRNG  (prng.hpp:18-47)                                                     */
/* ------------------------------------------------------------------------- */
uint64_t f2o_rng_seed(uint64_t seed) {               /* prng.hpp:20-21 */
    return seed != 0 ? seed : 0x9E3779B97F4A7C15ull;
}

static inline uint64_t step(uint64_t x) {            /* prng.hpp:24-28 */
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x;
}

uint64_t f2o_rng_next(uint64_t *state) {             /* prng.hpp:23-30 */
    uint64_t x = step(*state);
    *state = x;
    return x * 0x2545F4914F6CDD1Dull;
}

uint64_t f2o_bernoulli_threshold(double density) {   /* prng.hpp:40-42 */
    const double scaled = density * 18446744073709551616.0;
    return (uint64_t)scaled;
}

/* The state map is GF(2)-linear: represent T^(2^s) by its 64 column images. */
static void mat_apply(const uint64_t *cols, uint64_t x, uint64_t *out) {
    uint64_t y = 0;
    while (x) {
        int b = __builtin_ctzll(x);
        y ^= cols[b];
        x &= x - 1;
    }
    *out = y;
}

static uint64_t (*jump_tables(void))[64] {
    static uint64_t tab[64][64];
    static int ready = 0;
    if (!ready) {
#pragma omp critical(f2o_jump)
        {
            if (!ready) {
                for (int b = 0; b < 64; ++b) tab[0][b] = step(1ull << b);
                for (int s = 1; s < 64; ++s)
                    for (int b = 0; b < 64; ++b) mat_apply(tab[s - 1], tab[s - 1][b], &tab[s][b]);
                ready = 1;
            }
        }
    }
    return tab;
}

/* state after `t` further transitions */
static uint64_t jump(uint64_t state, uint64_t t) {
    uint64_t (*tab)[64] = jump_tables();
    for (int s = 0; t; ++s, t >>= 1)
        if (t & 1) mat_apply(tab[s], state, &state);
    return state;
}

/* random_dense (bit_matrix.hpp:125-142).  Rows are generated in parallel by
 * jumping the stream to draw i*m; the bits are identical to the serial loop. */
void f2o_random_dense(uint64_t *w, size_t n, size_t m, size_t stride, double density,
                      uint64_t seed) {
    const size_t mu = ceil64(m);
    memset(w, 0, mu * stride * sizeof(uint64_t));
    if (n == 0 || m == 0) return;
    if (density <= 0.0) return;                      /* :131 */
    if (density >= 1.0) {                            /* :132-139 no draws */
        for (size_t q = 0; q < mu; ++q) {
            uint64_t msk = (q + 1 == mu) ? low_mask(m - 64 * q) : ~0ull;
            for (size_t i = 0; i < n; ++i) w[q * stride + i] = msk;
        }
        return;
    }
    const uint64_t thr = f2o_bernoulli_threshold(density);
    const uint64_t s0 = f2o_rng_seed(seed);
    jump_tables();
    const size_t chunk = 64;
#pragma omp parallel for schedule(dynamic)
    for (size_t i0 = 0; i0 < n; i0 += chunk) {
        uint64_t st = jump(s0, (uint64_t)i0 * m);
        size_t i1 = i0 + chunk < n ? i0 + chunk : n;
        for (size_t i = i0; i < i1; ++i) {
            for (size_t q = 0; q < mu; ++q) {
                size_t kb = (q + 1 == mu) ? m - 64 * q : 64;
                uint64_t word = 0;
                for (size_t k = 0; k < kb; ++k) {
                    uint64_t v = f2o_rng_next(&st);
                    word |= (uint64_t)(v < thr) << k;
                }
                w[q * stride + i] = word;
            }
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Products                                                                   */
/* ------------------------------------------------------------------------- */
void f2o_mul_naive(const uint64_t *a, size_t n, size_t k, size_t sa, const uint64_t *b,
                   size_t m, size_t sb, uint64_t *c, size_t sc) {
    const size_t mu = ceil64(m);
    for (size_t q = 0; q < mu; ++q)
        for (size_t i = 0; i < n; ++i) c[q * sc + i] = 0;
#pragma omp parallel for schedule(static) if (n >= 256)
    for (size_t i = 0; i < n; ++i)
        for (size_t t = 0; t < k; ++t)
            if ((a[(t / 64) * sa + i] >> (t % 64)) & 1)
                for (size_t q = 0; q < mu; ++q) c[q * sc + i] ^= b[q * sb + t];
}

/* make_splits (m4rm.hpp:39-48) + doubling fill (m4rm.hpp:74-88) for one
 * word-column: tab must hold sum 2^{l_j} words. */
static size_t build_tab(const uint64_t *rows, size_t k_bits, unsigned c, uint64_t *tab,
                        unsigned *shifts, unsigned *sizes, size_t *offs) {
    size_t nt = 0, off = 0;
    for (size_t done = 0; done < k_bits;) {
        size_t l = (c < k_bits - done) ? c : k_bits - done;
        shifts[nt] = (unsigned)done;
        sizes[nt] = (unsigned)l;
        offs[nt] = off;
        uint64_t *t = tab + off;
        t[0] = 0;
        for (size_t bit = 0; bit < l; ++bit) {
            size_t base = (size_t)1 << bit;
            for (size_t g = base; g < 2 * base; ++g) t[g] = t[g - base] ^ rows[done + bit];
        }
        off += (size_t)1 << l;
        done += l;
        ++nt;
    }
    return nt;
}

/* mult_acc w==1 path (m4rm.hpp:147-160) */
static void sweep(uint64_t *dst, const uint64_t *a_words, size_t n_rows, const uint64_t *tab,
                  size_t nt, const unsigned *shifts, const unsigned *sizes, const size_t *offs) {
    for (size_t i = 0; i < n_rows; ++i) {
        uint64_t a = a_words[i];
        if (!a) continue;
        uint64_t acc = 0;
        for (size_t j = 0; j < nt; ++j) {
            uint64_t idx = (a >> shifts[j]) & low_mask(sizes[j]);
            acc ^= tab[offs[j] + idx];
        }
        dst[i] ^= acc;
    }
}

void f2o_m4rm_update(uint64_t *c, size_t sc, size_t c_row0, const uint64_t *a_words,
                     size_t n_rows, size_t k_bits, const uint64_t *b, size_t sb, size_t b_row0,
                     size_t n_wcols, unsigned tc) {
    if (k_bits == 0 || n_rows == 0 || n_wcols == 0) return;
    if (tc == 0) tc = 8;
#pragma omp parallel
    {
        uint64_t *tab = (uint64_t *)malloc(sizeof(uint64_t) * (64 + 64 * ((size_t)1 << tc)));
        unsigned shifts[64], sizes[64];
        size_t offs[64];
#pragma omp for schedule(dynamic)
        for (size_t q = 0; q < n_wcols; ++q) {
            size_t nt = build_tab(b + q * sb + b_row0, k_bits, tc, tab, shifts, sizes, offs);
            sweep(c + q * sc + c_row0, a_words, n_rows, tab, nt, shifts, sizes, offs);
        }
        free(tab);
    }
}

/* m4rm_mult (m4rm.hpp:177-196) */
void f2o_m4rm_mult(const uint64_t *a, size_t n, size_t k, size_t sa, const uint64_t *b,
                   size_t m, size_t sb, uint64_t *c, size_t sc, unsigned tc) {
    const size_t mu = ceil64(m), kb_n = ceil64(k);
    if (tc == 0) tc = f2o_optimal_table_size(64, n ? (double)n : 1.0);
    for (size_t q = 0; q < mu; ++q) memset(c + q * sc, 0, n * sizeof(uint64_t));
#pragma omp parallel
    {
        uint64_t *tab = (uint64_t *)malloc(sizeof(uint64_t) * (64 + 64 * ((size_t)1 << tc)));
        unsigned shifts[64], sizes[64];
        size_t offs[64];
#pragma omp for schedule(dynamic)
        for (size_t q = 0; q < mu; ++q)
            for (size_t kb = 0; kb < kb_n; ++kb) {
                size_t k_bits = (k - kb * 64) < 64 ? k - kb * 64 : 64;
                size_t nt = build_tab(b + q * sb + kb * 64, k_bits, tc, tab, shifts, sizes, offs);
                sweep(c + q * sc, a + kb * sa, n, tab, nt, shifts, sizes, offs);
            }
        free(tab);
    }
}

/* ------------------------------------------------------------------------- */
/* Tuning (tuning.hpp:20-41)                                 */
/* ------------------------------------------------------------------------- */
double f2o_m4rm_cost(unsigned b, unsigned c, double n) {
    return ((double)b / (double)c) * ((double)((1ull << c) - 1) + n);
}
unsigned f2o_optimal_table_size(unsigned b, double n) {
    unsigned hi = b < 16 ? b : 16, best = 2;
    double bc = f2o_m4rm_cost(b, 2, n);
    for (unsigned c = 3; c <= hi; ++c) {
        double v = f2o_m4rm_cost(b, c, n);
        if (v < bc) { bc = v; best = c; }
    }
    return best;
}
size_t f2o_strassen_threshold(unsigned c) { return 44 * (size_t)c + 6 * (((size_t)1 << c) - 1); }

/* ------------------------------------------------------------------------- */
/* Procedure buildZ, literal                              */
/* ------------------------------------------------------------------------- */
int f2o_build_z(uint64_t *A, size_t r, int64_t P[64], uint64_t Zout[64], uint64_t swap_b[64]) {
    uint64_t Z[64], M[64];
    size_t ib = 0;                                           /* :983 */
    for (int j = 0; j < 64; ++j) {                           /* :984-987 */
        Z[j] = 1ull << j;
        M[j] = 1ull << j;
        P[j] = -1;
    }
    for (int k = 0; k < 64; ++k) {                           /* :988 */
        uint64_t c = 1ull << k;                              /* :989 */
        for (int i = 0; i < k; ++i)                          /* :990-992 */
            if (M[i] & (1ull << k)) c ^= 1ull << i;
        for (size_t i = ib; i < r; ++i) {                    /* :993-1000 */
            if (__builtin_popcountll(c & A[i]) & 1) {
                P[k] = (int64_t)i;
                uint64_t t = A[i]; A[i] = A[ib]; A[ib] = t;
                M[k] = A[ib];
                swap_b[ib] = i;
                ++ib;
                break;
            }
        }
        uint64_t y = M[k];                                   /* :1001 */
        for (int j = 0; j < k; ++j)                          /* :1003-1006 */
            if (y & (1ull << j)) { Z[k] ^= Z[j]; M[k] ^= M[j]; }
        for (int j = 0; j < k; ++j)                          /* :1007-1010 */
            if (c & (1ull << j)) { Z[j] ^= Z[k]; M[j] ^= M[k]; }
    }
    uint64_t msk = 0;                                        /* :1012-1015 compression */
    for (int i = 0; i < 64; ++i) {
        if (P[i] == -1) {
            for (int j = 0; j < 64; ++j) Z[j] = ((Z[j] >> 1) & ~msk) ^ (Z[j] & msk);
        } else {
            msk = 2 * msk + 1;
        }
    }
    for (int j = 0; j < 64; ++j) Zout[j] = Z[j];
    return (int)ib;
}

/* ------------------------------------------------------------------------- */
/* decompose_block                        */
/* ------------------------------------------------------------------------- */
size_t f2o_decompose_block(uint64_t *w, size_t n, size_t m, size_t stride, uint32_t *perm,
                           uint32_t *rj, unsigned tc, size_t max_panels) {
    const size_t mu = ceil64(m);
    size_t R = 0;
    for (size_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
    for (size_t j = 0; j < mu; ++j) rj[j] = 0;
    if (tc == 0) tc = 8;
    uint64_t *ybuf = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    for (size_t j = 0; j < mu && j < max_panels; ++j) {
        if (R >= n) break;                 /* rank exhausted: remaining r_j = 0 */
        uint64_t *panel = w + j * stride + R;
        const size_t rows = n - R;
        int64_t P[64];
        uint64_t Z[64], sb[64];
        const int r = f2o_build_z(panel, rows, P, Z, sb);
        /* mirror the transpositions (k, sb[k]) on every other word-column and on
         * perm (row_swap bit_matrix.hpp:202-208; RowPermutation::swap :361) */
        if (r > 0) {
#pragma omp parallel for schedule(static) if (mu >= 16)
            for (size_t q = 0; q < mu; ++q) {
                if (q == j) continue;
                uint64_t *col = w + q * stride + R;
                for (int k = 0; k < r; ++k) {
                    uint64_t t = col[k]; col[k] = col[sb[k]]; col[sb[k]] = t;
                }
            }
            for (int k = 0; k < r; ++k) {
                uint32_t t = perm[R + k]; perm[R + k] = perm[R + sb[k]]; perm[R + sb[k]] = t;
            }
        }
        /* Y = D*Z written over D, then Schur E ^= Y*C */
        const size_t nd = rows - (size_t)r;
        uint64_t *D = panel + r;
        if (r == 0) {
            /* r_j = 0 implies D == 0 (every nonzero row passes some parity test) */
            rj[j] = 0;
            continue;
        }
        {
            uint64_t ztab[64 + 8 * 256];
            unsigned shifts[64], sizes[64];
            size_t offs[64];
            size_t nt = build_tab(Z, 64, tc, ztab, shifts, sizes, offs);
            memset(ybuf, 0, nd * sizeof(uint64_t));
            sweep(ybuf, D, nd, ztab, nt, shifts, sizes, offs);
            memcpy(D, ybuf, nd * sizeof(uint64_t));
        }
        if (j + 1 < mu && nd > 0)
            f2o_m4rm_update(w + (j + 1) * stride, stride, R + r, D, nd, (size_t)r,
                            w + (j + 1) * stride, stride, R, mu - j - 1, tc);
        rj[j] = (uint32_t)r;
        R += (size_t)r;
    }
    free(ybuf);
    return R;
}

size_t f2o_rank_ge(const uint64_t *w, size_t n, size_t m, size_t stride) {
    const size_t mu = ceil64(m);
    uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * (mu * stride + 1));
    memcpy(t, w, sizeof(uint64_t) * mu * stride);
    size_t rank = 0;
    for (size_t col = 0; col < m && rank < n; ++col) {
        size_t q = col / 64;
        uint64_t bit = 1ull << (col % 64);
        size_t piv = n;
        for (size_t i = rank; i < n; ++i)
            if (t[q * stride + i] & bit) { piv = i; break; }
        if (piv == n) continue;
        for (size_t qq = 0; qq < mu; ++qq) {
            uint64_t x = t[qq * stride + piv];
            t[qq * stride + piv] = t[qq * stride + rank];
            t[qq * stride + rank] = x;
        }
        for (size_t i = rank + 1; i < n; ++i)
            if (t[q * stride + i] & bit)
                for (size_t qq = q; qq < mu; ++qq) t[qq * stride + i] ^= t[qq * stride + rank];
        ++rank;
    }
    free(t);
    return rank;
}

/* transpose_tile (bit_matrix.hpp:59-70) restated as a plain 64x64 bit transpose */
static void tr64(uint64_t *x) {
    uint64_t m = 0x00000000FFFFFFFFull;
    for (int j = 32; j != 0; j >>= 1, m ^= (m << j)) {
        for (int k = 0; k < 64; k = (k + j + 1) & ~j) {
            uint64_t t = ((x[k] >> j) ^ x[k + j]) & m;
            x[k + j] ^= t;
            x[k] ^= t << j;
        }
    }
}

void f2o_transpose(const uint64_t *w, size_t n, size_t m, size_t stride, uint64_t *out, size_t so) {
    const size_t mu = ceil64(m), mo = ceil64(n);
    for (size_t q = 0; q < mo; ++q) memset(out + q * so, 0, m * sizeof(uint64_t));
#pragma omp parallel for schedule(static) if (mu > 1 && n >= 4096)
    for (size_t q = 0; q < mu; ++q) {
        uint64_t tile[64];
        size_t out_rows = (m - q * 64) < 64 ? m - q * 64 : 64;
        for (size_t tr = 0; tr < mo; ++tr) {
            size_t i0 = tr * 64, h = (n - i0) < 64 ? n - i0 : 64;
            for (size_t t = 0; t < 64; ++t) tile[t] = t < h ? w[q * stride + i0 + t] : 0;
            tr64(tile);
            for (size_t t = 0; t < out_rows; ++t) out[tr * so + q * 64 + t] = tile[t];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Digests / checks                                                           */
/* ------------------------------------------------------------------------- */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t f2o_digest(const uint64_t *w, size_t n, size_t m, size_t stride) {
    const size_t mu = ceil64(m);
    uint64_t s = mix64(n * 0x9E3779B97F4A7C15ull ^ m);
#pragma omp parallel for reduction(+ : s) schedule(static)
    for (size_t q = 0; q < mu; ++q) {
        uint64_t acc = 0;
        const uint64_t salt = mix64(q + 0x1234567ull);
        for (size_t i = 0; i < n; ++i) acc += mix64(w[q * stride + i] ^ (i * 0xD6E8FEB86659FD93ull) ^ salt);
        s += acc;
    }
    return s;
}

uint64_t f2o_digest_u32(const uint32_t *v, size_t n) {
    uint64_t s = mix64(n);
    for (size_t i = 0; i < n; ++i) s += mix64(((uint64_t)v[i] << 32) ^ i);
    return s;
}

void f2o_extract_lu(const uint64_t *w, size_t n, size_t m, size_t stride, const uint32_t *rj,
                    size_t rank, uint64_t *L, size_t sl, uint64_t *U, size_t su) {
    const size_t mu = ceil64(m), ml = ceil64(rank);
    for (size_t q = 0; q < ml; ++q) memset(L + q * sl, 0, n * sizeof(uint64_t));
    for (size_t q = 0; q < mu; ++q) memset(U + q * su, 0, rank * sizeof(uint64_t));
    size_t R = 0;
    for (size_t j = 0; j < mu && R < n; ++j) {
        size_t r = rj[j];
        if (r == 0) continue;
        /* L block column at bit offset R: I_r on pivot rows, Y below */
        for (size_t i = R; i < n; ++i) {
            uint64_t bits = (i < R + r) ? (1ull << (i - R)) : w[j * stride + i];
            if (!bits) continue;
            size_t qq = R / 64, s = R % 64;          /* xor_bits_at bit_matrix.hpp:402-413 */
            L[qq * sl + i] ^= bits << s;
            if (s && (bits >> (64 - s))) L[(qq + 1) * sl + i] ^= bits >> (64 - s);
        }
        /* U rows R..R+r: word-cols >= j of the pivot rows */
        for (size_t q = j; q < mu; ++q)
            for (size_t t = 0; t < r; ++t) U[q * su + R + t] = w[q * stride + R + t];
        R += r;
    }
}

int f2o_check_plu(const uint64_t *a, const uint64_t *w, size_t n, size_t m, size_t stride,
                  const uint32_t *perm, const uint32_t *rj, uint64_t seed) {
    const size_t mu = ceil64(m);
    /* X: m x 64 random (one word per row) */
    uint64_t *X = (uint64_t *)malloc(sizeof(uint64_t) * (m + 1));
    uint64_t st = f2o_rng_seed(seed);
    for (size_t i = 0; i < m; ++i) X[i] = f2o_rng_next(&st);
    /* AX: n words */
    uint64_t *ax = (uint64_t *)calloc(n + 1, sizeof(uint64_t));
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) {
        uint64_t acc = 0;
        for (size_t q = 0; q < mu; ++q) {
            uint64_t wd = a[q * stride + perm[i]];
            while (wd) { int b = __builtin_ctzll(wd); acc ^= X[q * 64 + b]; wd &= wd - 1; }
        }
        ax[i] = acc;
    }
    /* UX per pivot row (pivot rows are rows 0..rank-1 of W, U part = word-cols >= panel) */
    size_t rank = 0;
    for (size_t j = 0; j < mu; ++j) rank += rj[j];
    uint64_t *ux = (uint64_t *)calloc(rank + 1, sizeof(uint64_t));
    size_t *rowpanel = (size_t *)malloc(sizeof(size_t) * (rank + 1));
    size_t *panel_r0 = (size_t *)malloc(sizeof(size_t) * (mu + 1));
    {
        size_t R = 0;
        for (size_t j = 0; j < mu; ++j) {
            panel_r0[j] = R;
            for (size_t t = 0; t < rj[j]; ++t) rowpanel[R + t] = j;
            R += rj[j];
        }
    }
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < rank; ++i) {
        uint64_t acc = 0;
        for (size_t q = rowpanel[i]; q < mu; ++q) {
            uint64_t wd = w[q * stride + i];
            while (wd) { int b = __builtin_ctzll(wd); acc ^= X[q * 64 + b]; wd &= wd - 1; }
        }
        ux[i] = acc;
    }
    int ok = 1;
#pragma omp parallel for schedule(static) reduction(& : ok)
    for (size_t i = 0; i < n; ++i) {
        uint64_t acc = 0;
        for (size_t j = 0; j < mu; ++j) {
            size_t r = rj[j], R = panel_r0[j];
            if (r == 0) continue;
            if (i < R) break;
            if (i < R + r) { acc ^= ux[i]; break; }
            uint64_t y = w[j * stride + i];
            while (y) { int b = __builtin_ctzll(y); acc ^= ux[R + b]; y &= y - 1; }
        }
        if (acc != ax[i]) ok = 0;
    }
    free(X); free(ax); free(ux); free(rowpanel); free(panel_r0);
    return ok;
}
