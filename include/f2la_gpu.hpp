// f2la_gpu.hpp — C++ forwarding shim: the reference's f2la free-function API,
// executed by libf2gpu.so (hand-written sm_100a kernels) through the C-ABI in
// f2gpu.h.  Header-only; include AFTER the reference's "f2la/bit_matrix.hpp".
//
//   reference (header-only CPU)                       this shim (B200)
//   f2la::make_splits(k, c)        m4rm.hpp:39-48     f2la::gpu::make_splits(k, c)
//   f2la::build_tables(...) x4     m4rm.hpp:93-135    f2la::gpu::build_tables(...) x4
//   f2la::mult_acc(C, r0, q0, a, t) m4rm.hpp:140-172  f2la::gpu::mult_acc(C, r0, q0, a, t)
//   f2la::m4rm_mult(A, B, c)       m4rm.hpp:177-196   f2la::gpu::m4rm_mult(A, B, c)
//   strassen_mult(A, B, thr, c)    SPEC.md:192-200    f2la::gpu::strassen_mult(A, B, thr, c)
//   decompose_block(A)->LUFactors  SPEC.md:319-327    f2la::gpu::decompose_block(A)
//   rank(A)                        SPEC.md:346-353    f2la::gpu::rank(A)
//   decompose_recursive(A, mc)     SPEC.md:328-345    f2la::gpu::decompose_recursive(A, mc)
//   null_space(A), solve(A, rhs)   SPEC.md:354-362    f2la::gpu::null_space(A), f2la::gpu::solve(A, rhs)
//
// Matrices are passed in the reference layout (PackedMatrix<uint64_t>:
// col_block(q) + col_stride(), bit_matrix.hpp:74-81).  Errors are rethrown as
// the reference's exception types (std::invalid_argument / std::out_of_range).
// Only Word = std::uint64_t (BitMatrix) runs on the device.
//
// include/f2la_gpu_dropin.hpp goes one step further: included in place of
// "f2la/m4rm.hpp", it makes the reference's own unqualified call sites
// (f2la::build_tables / f2la::mult_acc / f2la::m4rm_mult ...) resolve here.
#ifndef F2LA_GPU_HPP
#define F2LA_GPU_HPP

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "f2gpu.h"

namespace f2la::gpu {

inline void check(int rc, const char* what) {
    if (rc == F2GPU_OK) return;
    const std::string msg = std::string(what) + ": " + f2gpu_last_error();
    if (rc == F2GPU_EINVAL) throw std::invalid_argument(msg);
    if (rc == F2GPU_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

/// Per-thread default context on device 0 (the reference contract is one call
/// per thread at a time).
inline f2gpu_ctx* context() {
    struct Holder {
        f2gpu_ctx* c = nullptr;
        Holder() { check(f2gpu_ctx_create(0, &c), "f2gpu_ctx_create"); }
        ~Holder() { f2gpu_ctx_destroy(c); }
    };
    thread_local Holder h;
    return h.c;
}

/// make_splits (m4rm.hpp:39-48): floor(k/c) groups of c plus the remainder.
inline std::vector<std::uint32_t> make_splits(std::size_t k_bits, std::size_t c) {
    if (c == 0) throw std::invalid_argument("make_splits: c must be positive");
    std::vector<std::uint32_t> splits;
    for (std::size_t done = 0; done < k_bits;) {
        const std::size_t l = std::min(c, k_bits - done);
        splits.push_back(static_cast<std::uint32_t>(l));
        done += l;
    }
    return splits;
}

/// M4rmTables (m4rm.hpp:21-35) for the device: the tables themselves are built in
/// shared memory inside the fused mult_acc kernel, so this records the B block
/// they cover (plus the reference's group metadata: shifts / sizes / masks /
/// offsets, computed as make_table_shell does, m4rm.hpp:52-70).  `entries` is not
/// materialised.  The B matrix must outlive the tables (the reference copies it).
template <class Word>
struct M4rmTables {
    static_assert(std::is_same_v<Word, std::uint64_t>, "f2la::gpu: only 64-bit words run on the device");
    std::size_t k_bits = 0;
    std::size_t width_words = 0;
    std::vector<std::uint32_t> shifts, sizes;
    std::vector<Word> masks;
    std::vector<std::size_t> offsets;
    // the B block: rows [row0, row0 + k_bits) x word-columns [wcol0, wcol0 + width_words)
    const Word* b_base = nullptr;
    std::size_t b_rows = 0, b_cols = 0, b_stride = 0, row0 = 0, wcol0 = 0;
    std::vector<Word> own_rows;  // the bare-word overload keeps its rows here
    std::size_t table_count() const noexcept { return sizes.size(); }
};

namespace detail {
template <class Word>
void table_shell(M4rmTables<Word>& t, std::size_t k_bits, std::size_t width, std::span<const std::uint32_t> splits) {
    t.k_bits = k_bits;
    t.width_words = width;
    std::size_t bit = 0, rows = 0;
    for (const std::uint32_t l : splits) {
        t.shifts.push_back(static_cast<std::uint32_t>(bit));
        t.sizes.push_back(l);
        t.masks.push_back(l >= 64 ? ~Word(0) : ((Word(1) << l) - 1));
        t.offsets.push_back(rows);
        bit += l;
        rows += l >= 64 ? 0 : (std::size_t(1) << l);
    }
    if (bit != k_bits) throw std::invalid_argument("build_tables: splits do not sum to k");
}
}  // namespace detail

/// build_tables(B, row0, k, wcol0, n, splits) (m4rm.hpp:93-113).
template <class Word>
M4rmTables<Word> build_tables(const PackedMatrix<Word>& b_mat, std::size_t row0, std::size_t k_bits,
                              std::size_t wcol0, std::size_t n_wcols, std::span<const std::uint32_t> splits) {
    if (k_bits > PackedMatrix<Word>::word_bits) throw std::invalid_argument("build_tables: block taller than a word");
    if (row0 + k_bits > b_mat.rows() || wcol0 + n_wcols > b_mat.word_cols())
        throw std::out_of_range("build_tables: block outside B");
    M4rmTables<Word> t;
    detail::table_shell(t, k_bits, n_wcols, splits);
    t.b_base = b_mat.word_cols() ? b_mat.col_block(0) : nullptr;
    t.b_rows = b_mat.rows();
    t.b_cols = b_mat.cols();
    t.b_stride = b_mat.col_stride();
    t.row0 = row0;
    t.wcol0 = wcol0;
    return t;
}
/// Whole-matrix convenience (m4rm.hpp:117-121): B has at most 64 rows.
template <class Word>
M4rmTables<Word> build_tables(const PackedMatrix<Word>& b_mat, std::span<const std::uint32_t> splits) {
    return gpu::build_tables(b_mat, 0, b_mat.rows(), 0, b_mat.word_cols(), splits);
}
/// m4rm.hpp:122-126.
template <class Word>
M4rmTables<Word> build_tables(const PackedMatrix<Word>& b_mat, std::size_t c) {
    const auto splits = gpu::make_splits(b_mat.rows(), c);
    return gpu::build_tables(b_mat, std::span<const std::uint32_t>(splits));
}
/// Bare words (m4rm.hpp:128-135; compute_Y's Y = D*Z): row r of B is rows[r].
template <class Word>
M4rmTables<Word> build_tables(std::span<const Word> rows, std::size_t c) {
    if (rows.size() > 64) throw std::invalid_argument("build_tables: block taller than a word");
    const auto splits = gpu::make_splits(rows.size(), c);
    M4rmTables<Word> t;
    detail::table_shell(t, rows.size(), 1, std::span<const std::uint32_t>(splits));
    t.own_rows.assign(rows.begin(), rows.end());
    t.b_rows = rows.size();
    t.b_cols = 64;
    t.b_stride = rows.size();
    return t;
}

/// mult_acc(C, c_row0, c_wcol0, a_words, tables) (m4rm.hpp:140-172): C rows
/// [c_row0 + i] x word-columns [c_wcol0, c_wcol0 + width) ^= a_words[i] * B.
template <class Word>
void mult_acc(PackedMatrix<Word>& c_mat, std::size_t c_row0, std::size_t c_wcol0, std::span<const Word> a_words,
              const M4rmTables<Word>& tables) {
    const std::size_t w = tables.width_words;
    if (c_row0 + a_words.size() > c_mat.rows() || c_wcol0 + w > c_mat.word_cols())
        throw std::out_of_range("mult_acc: destination outside C");
    if (a_words.empty() || w == 0 || tables.k_bits == 0) return;
    const Word* b = tables.own_rows.empty() ? tables.b_base : tables.own_rows.data();
    check(f2gpu_mult_acc_host(context(), c_mat.col_block(0), c_mat.rows(), c_mat.cols(), c_mat.col_stride(), c_row0,
                              c_wcol0, a_words.data(), a_words.size(), b, tables.b_rows, tables.b_cols,
                              tables.b_stride, tables.row0, tables.k_bits, tables.wcol0, w),
          "mult_acc");
}

/// C = A*B over F2 (m4rm.hpp:177-196).  `c` is accepted for signature parity.
template <class Matrix>
Matrix m4rm_mult(const Matrix& a, const Matrix& b, std::size_t c = 0) {
    if (a.cols() != b.rows()) throw std::invalid_argument("m4rm_mult: shape mismatch");
    Matrix out(a.rows(), b.cols());
    if (a.rows() == 0 || b.cols() == 0) return out;
    check(f2gpu_m4rm_mult_host(context(), a.col_block(0), a.rows(), a.cols(), a.col_stride(),
                               b.col_block(0), b.cols(), b.col_stride(), out.col_block(0),
                               out.col_stride(), unsigned(c)),
          "m4rm_mult");
    return out;
}

/// Strassen-Winograd with M4RM leaves; threshold 0 = default.
template <class Matrix>
Matrix strassen_mult(const Matrix& a, const Matrix& b, std::size_t threshold = 0,
                     std::size_t /*c*/ = 0) {
    if (a.cols() != b.rows()) throw std::invalid_argument("strassen_mult: shape mismatch");
    Matrix out(a.rows(), b.cols());
    if (a.rows() == 0 || b.cols() == 0) return out;
    check(f2gpu_strassen_mult_host(context(), a.col_block(0), a.rows(), a.cols(), a.col_stride(),
                                   b.col_block(0), b.cols(), b.col_stride(), out.col_block(0),
                                   out.col_stride(), threshold),
          "strassen_mult");
    return out;
}

/// LUFactors + the device overlay W it is derived from.
template <class Matrix>
struct LUFactors {
    std::vector<std::uint32_t> P;      // (P A)_i = A_{P[i]}   (bit_matrix.hpp:350)
    Matrix L;                          // n x rank, unit lower trapezoidal
    Matrix U;                          // rank x m, block staircase
    std::size_t rank = 0;
    std::vector<std::size_t> block_ranks;
    Matrix overlay;                    // W: L below/left of the staircase, U on pivot rows
};

/// decompose_block: P*A = L*U, column-swap free; A unmodified.
template <class Matrix>
LUFactors<Matrix> decompose_block(const Matrix& a) {
    const std::size_t n = a.rows(), m = a.cols(), mu = a.word_cols();
    LUFactors<Matrix> f;
    f.overlay = Matrix(n, m);
    f.P.resize(n);
    std::vector<std::uint32_t> rj(mu);
    std::size_t rank = 0;
    if (n && m)
        check(f2gpu_decompose_block_host(context(), a.col_block(0), n, m, a.col_stride(),
                                         f.overlay.col_block(0), f.P.data(), rj.data(), &rank),
              "decompose_block");
    else
        for (std::size_t i = 0; i < n; ++i) f.P[i] = std::uint32_t(i);
    f.rank = rank;
    f.block_ranks.assign(rj.begin(), rj.end());
    f.L = Matrix(n, rank);
    f.U = Matrix(rank, m);
    std::size_t R = 0;
    for (std::size_t j = 0; j < mu; ++j) {
        const std::size_t r = rj[j];
        if (!r) continue;
        for (std::size_t i = R; i < n; ++i) {  // [I_r; Y^(j)] at bit offset R
            const std::uint64_t bits = i < R + r ? (std::uint64_t(1) << (i - R))
                                                 : f.overlay.word(i, j);
            xor_bits_at(f.L, i, R, bits);  // reference helper, bit_matrix.hpp:402-413
        }
        for (std::size_t q = j; q < mu; ++q)
            for (std::size_t t = 0; t < r; ++t) f.U.word(R + t, q) = f.overlay.word(R + t, q);
        R += r;
    }
    return f;
}

/// decompose_recursive(A, min_cols): same LUFactors contract;
/// exact arithmetic and 64-aligned splits make it bit-identical to decompose_block.
template <class Matrix>
LUFactors<Matrix> decompose_recursive(const Matrix& a, std::size_t min_cols = 0) {
    const std::size_t n = a.rows(), m = a.cols();
    LUFactors<Matrix> f;
    f2gpu_mat* w = nullptr;
    check(f2gpu_mat_alloc(context(), n, m, &w), "mat_alloc");
    struct Free { f2gpu_mat* p; ~Free() { f2gpu_mat_free(p); } } guard{w};
    if (n && m) check(f2gpu_mat_upload(context(), w, a.col_block(0), a.col_stride()), "upload");
    f.overlay = Matrix(n, m);
    f.P.resize(n);
    std::vector<std::uint32_t> rj(a.word_cols());
    std::size_t rank = 0;
    check(f2gpu_decompose_recursive(context(), w, min_cols, f.P.data(), rj.data(), &rank),
          "decompose_recursive");
    if (n && m) check(f2gpu_mat_download(context(), w, f.overlay.col_block(0), f.overlay.col_stride()),
                      "download");
    f.rank = rank;
    f.block_ranks.assign(rj.begin(), rj.end());
    f.L = Matrix(n, rank);
    f.U = Matrix(rank, m);
    std::size_t R = 0;
    for (std::size_t j = 0; j < a.word_cols(); ++j) {
        const std::size_t r = rj[j];
        if (!r) continue;
        for (std::size_t i = R; i < n; ++i)
            xor_bits_at(f.L, i, R, i < R + r ? (std::uint64_t(1) << (i - R)) : f.overlay.word(i, j));
        for (std::size_t q = j; q < a.word_cols(); ++q)
            for (std::size_t t = 0; t < r; ++t) f.U.word(R + t, q) = f.overlay.word(R + t, q);
        R += r;
    }
    return f;
}

/// rank(A) = sum r_j, transposing wide inputs.
template <class Matrix>
std::size_t rank(const Matrix& a) {
    std::size_t r = 0;
    if (a.rows() && a.cols())
        check(f2gpu_rank_host(context(), a.col_block(0), a.rows(), a.cols(), a.col_stride(), &r),
              "rank");
    return r;
}

namespace detail {
template <class Matrix>
f2gpu_mat* upload(const Matrix& a) {
    f2gpu_mat* d = nullptr;
    check(f2gpu_mat_alloc(context(), a.rows(), a.cols(), &d), "mat_alloc");
    if (a.rows() && a.cols()) {
        const int rc = f2gpu_mat_upload(context(), d, a.col_block(0), a.col_stride());
        if (rc != F2GPU_OK) {
            f2gpu_mat_free(d);
            check(rc, "mat_upload");
        }
    }
    return d;
}
struct MatFree {
    f2gpu_mat* m;
    ~MatFree() { f2gpu_mat_free(m); }
};
}  // namespace detail

/// m x (m - rank) basis N with A*N = 0 and independent columns.
template <class Matrix>
Matrix null_space(const Matrix& a) {
    detail::MatFree A{detail::upload(a)};
    f2gpu_mat* n = nullptr;
    std::size_t nul = 0;
    check(f2gpu_null_space(context(), A.m, &n, &nul), "null_space");
    detail::MatFree N{n};
    Matrix out(a.cols(), nul);
    if (a.cols() && nul) check(f2gpu_mat_download(context(), n, out.col_block(0), out.col_stride()), "download");
    return out;
}

/// x with A x = rhs over F2 (one bit per element), or nullopt for an inconsistent
/// system -- signalled, not an error.
template <class Matrix>
std::optional<std::vector<std::uint8_t>> solve(const Matrix& a, const std::vector<std::uint8_t>& rhs) {
    if (rhs.size() != a.rows()) throw std::invalid_argument("solve: rhs length must equal rows");
    detail::MatFree A{detail::upload(a)};
    std::vector<std::uint64_t> b((a.rows() + 63) / 64 + 1, 0), x((a.cols() + 63) / 64 + 1, 0);
    for (std::size_t i = 0; i < rhs.size(); ++i)
        if (rhs[i] & 1) b[i / 64] |= std::uint64_t(1) << (i % 64);
    int ok = 0;
    check(f2gpu_solve(context(), A.m, b.data(), x.data(), &ok), "solve");
    if (!ok) return std::nullopt;
    std::vector<std::uint8_t> out(a.cols());
    for (std::size_t j = 0; j < out.size(); ++j) out[j] = std::uint8_t((x[j / 64] >> (j % 64)) & 1);
    return out;
}

}  // namespace f2la::gpu

#endif
