// ref_shim.cpp — C entry points over the REFERENCE headers, compiled in place.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile against
// /root/reference/proj/include (never copied) into oracle/_ref/libf2la_ref.so.
// Used (a) to pin the plain-C oracle and generate tests/golden fixtures, and
// (b) as the `--impl reference` / cpu_baseline leg of bench.py.
//
// Exposes the reference's own code paths:
//   f2la::PackedMatrix::random_dense   bit_matrix.hpp:125-142
//   f2la::m4rm_mult                    m4rm.hpp:177-196
//   f2la::PackedMatrix::transposed     bit_matrix.hpp:220-238
// and a decomposition built on the reference's build_tables/mult_acc
// (m4rm.hpp:93-172) with the restated Procedure buildZ (oracle/f2oracle.c,
// PAPER.md:971-1015) — the reference ships no decomposition code.
#include <cstdint>
#include <cstring>
#include <vector>

#include "f2la/bit_matrix.hpp"
#include "f2la/m4rm.hpp"
#include "f2oracle.h"

using f2la::BitMatrix;

namespace {

BitMatrix from_raw(const uint64_t* w, size_t n, size_t m, size_t stride) {
    BitMatrix a(n, m);
    for (size_t q = 0; q < a.word_cols(); ++q)
        std::memcpy(a.col_block(q), w + q * stride, n * sizeof(uint64_t));
    return a;
}

void to_raw(const BitMatrix& a, uint64_t* w, size_t stride) {
    for (size_t q = 0; q < a.word_cols(); ++q) {
        std::memcpy(w + q * stride, a.col_block(q), a.rows() * sizeof(uint64_t));
        for (size_t i = a.rows(); i < stride; ++i) w[q * stride + i] = 0;
    }
}

}  // namespace

extern "C" {

// first `count` outputs of the reference Rng (prng.hpp:18-47) for a seed
void ref_rng_outputs(uint64_t seed, uint64_t* out, size_t count) {
    f2la::Rng rng(seed);
    for (size_t i = 0; i < count; ++i) out[i] = rng.next();
}

size_t ref_col_stride(size_t n_rows) {
    BitMatrix a(n_rows, 1);
    return a.col_stride();
}

void ref_random_dense(uint64_t* w, size_t n, size_t m, size_t stride, double density,
                      uint64_t seed) {
    to_raw(BitMatrix::random_dense(n, m, density, seed), w, stride);
}

// returns 0 ok, 1 invalid_argument
int ref_m4rm_mult(const uint64_t* a, size_t n, size_t k, size_t sa, const uint64_t* b,
                  size_t m, size_t sb, uint64_t* c, size_t sc, size_t tc) {
    try {
        BitMatrix A = from_raw(a, n, k, sa), B = from_raw(b, k, m, sb);
        to_raw(f2la::m4rm_mult(A, B, tc), c, sc);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// Same but with the matrices already in reference storage (no conversion in the
// timed region): handle-based for the CPU baseline.
void* ref_matrix_new(const uint64_t* w, size_t n, size_t m, size_t stride) {
    return new BitMatrix(from_raw(w, n, m, stride));
}
void* ref_matrix_random(size_t n, size_t m, double density, uint64_t seed) {
    return new BitMatrix(BitMatrix::random_dense(n, m, density, seed));
}
void ref_matrix_free(void* h) { delete static_cast<BitMatrix*>(h); }
void ref_matrix_read(void* h, uint64_t* w, size_t stride) {
    to_raw(*static_cast<BitMatrix*>(h), w, stride);
}
void* ref_matrix_mult(void* a, void* b, size_t tc) {
    return new BitMatrix(
        f2la::m4rm_mult(*static_cast<BitMatrix*>(a), *static_cast<BitMatrix*>(b), tc));
}

void ref_transpose(const uint64_t* w, size_t n, size_t m, size_t stride, uint64_t* out,
                   size_t so) {
    to_raw(from_raw(w, n, m, stride).transposed(), out, so);
}

// Decomposition driven by the reference's M4RM (build_tables + mult_acc, width 1)
// for Y = D*Z and the Schur update, with OpenMP over trailing word-columns.
// Operates in place on a reference BitMatrix handle.  max_panels bounds the
// number of panels processed (bounded CPU samples).
size_t ref_decompose_block(void* h, uint32_t* perm, uint32_t* rj, size_t tc,
                           size_t max_panels) {
    BitMatrix& W = *static_cast<BitMatrix*>(h);
    const size_t n = W.rows(), mu = W.word_cols();
    f2la::RowPermutation P = f2la::RowPermutation::identity(n);
    for (size_t j = 0; j < mu; ++j) rj[j] = 0;
    if (tc == 0) tc = 8;
    size_t R = 0;
    std::vector<uint64_t> y(n);
    for (size_t j = 0; j < mu && j < max_panels; ++j) {
        if (R >= n) break;
        uint64_t* panel = W.col_block(j) + R;
        const size_t rows = n - R;
        int64_t Pk[64];
        uint64_t Z[64], sb[64];
        const int r = f2o_build_z(panel, rows, Pk, Z, sb);
        if (r == 0) continue;
        // mirror the transpositions on the other word-columns (row_swap :202-208)
#pragma omp parallel for schedule(static) if (mu >= 16)
        for (size_t q = 0; q < mu; ++q) {
            if (q == j) continue;
            uint64_t* col = W.col_block(q) + R;
            for (int k = 0; k < r; ++k) std::swap(col[k], col[sb[k]]);
        }
        for (int k = 0; k < r; ++k) P.swap(R + k, R + sb[k]);
        const size_t nd = rows - size_t(r);
        // Y = D*Z via the bare-word table builder (m4rm.hpp:128-135) + mult_acc
        {
            const auto zt = f2la::build_tables<uint64_t>(std::span<const uint64_t>(Z, 64), tc);
            BitMatrix Y(nd, 64);
            f2la::mult_acc(Y, 0, 0, std::span<const uint64_t>(panel + r, nd), zt);
            std::memcpy(panel + r, Y.col_block(0), nd * sizeof(uint64_t));
        }
        // Schur: E[:, q] ^= Y * C[:, q]  (m4rm.hpp:93-113 + 140-172)
        if (nd > 0) {
            const auto splits = f2la::make_splits(size_t(r), tc);
            const std::span<const uint64_t> ys(panel + r, nd);
#pragma omp parallel for schedule(dynamic)
            for (size_t q = j + 1; q < mu; ++q) {
                const auto t = f2la::build_tables(W, R, size_t(r), q, 1,
                                                  std::span<const uint32_t>(splits));
                f2la::mult_acc(W, R + size_t(r), q, ys, t);
            }
        }
        rj[j] = uint32_t(r);
        R += size_t(r);
    }
    for (size_t i = 0; i < n; ++i) perm[i] = P.perm[i];
    return R;
}

}  // extern "C"
