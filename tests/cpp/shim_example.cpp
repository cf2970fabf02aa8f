// Drop-in usage of the GPU shim next to the reference's own headers.
// Built by tests/test_abi.py (compile + link check) in the build container; when
// a B200 is present it runs the reference m4rm_mult and the GPU one side by side.
#include <cstdio>

#include "f2la/bit_matrix.hpp"
#include "f2la/m4rm.hpp"
#include "f2la_gpu.hpp"

namespace f2la::tuning {  // the reference declares but never defines these (tuning.hpp:26)
unsigned optimal_table_size(unsigned, double) { return 8; }
}  // namespace f2la::tuning

int main() {
    using f2la::BitMatrix;
    f2gpu_ctx* probe = nullptr;
    if (f2gpu_ctx_create(0, &probe) != F2GPU_OK) {
        std::printf("no B200: %s\n", f2gpu_last_error());
        return 0;
    }
    f2gpu_ctx_destroy(probe);
    const BitMatrix a = BitMatrix::random_dense(777, 1000, 0.5, 1);
    const BitMatrix b = BitMatrix::random_dense(1000, 333, 0.5, 2);
    const bool mult_ok = f2la::gpu::m4rm_mult(a, b) == f2la::m4rm_mult(a, b, 8);
    const auto f = f2la::gpu::decompose_block(a);
    // P*A == L*U with the reference's own product and gather_rows
    const BitMatrix pa = f2la::gather_rows(a, std::span<const std::uint32_t>(f.P));
    const bool lu_ok = f2la::m4rm_mult(f.L, f.U, 8) == pa;
    const bool rank_ok = f2la::gpu::rank(a) == f.rank && f.rank == 777;
    const auto g = f2la::gpu::decompose_recursive(a, 128);
    const bool rec_ok = g.P == f.P && g.overlay == f.overlay && g.L == f.L && g.U == f.U;
    // null space of a rank-deficient product, checked with the reference's own product
    const BitMatrix x = BitMatrix::random_dense(300, 90, 0.5, 3), y = BitMatrix::random_dense(90, 500, 0.5, 4);
    const BitMatrix xy = f2la::m4rm_mult(x, y, 8);
    const BitMatrix ns = f2la::gpu::null_space(xy);
    const bool ns_ok = ns.cols() == 500 - f2la::gpu::rank(xy) && f2la::m4rm_mult(xy, ns, 8) == BitMatrix(300, ns.cols());
    // solve a consistent system b = A * e_0 (column 0 of A)
    std::vector<std::uint8_t> rhs(a.rows());
    for (std::size_t i = 0; i < a.rows(); ++i) rhs[i] = std::uint8_t(a.get(i, 0));
    const auto sol = f2la::gpu::solve(a, rhs);
    bool solve_ok = sol.has_value();
    if (solve_ok) {
        BitMatrix xv(a.cols(), 1);
        for (std::size_t j = 0; j < a.cols(); ++j) xv.set(j, 0, (*sol)[j]);
        const BitMatrix ax = f2la::m4rm_mult(a, xv, 8);
        for (std::size_t i = 0; i < a.rows(); ++i) solve_ok = solve_ok && ax.get(i, 0) == bool(rhs[i]);
    }
    // build_tables + mult_acc (m4rm.hpp:93-172): the reference's own Schur-update
    // calls and the shim's on identical inputs, bit-for-bit -- several k, widths,
    // offsets, the bare-word overload, and the reference's exception types
    bool macc_ok = true;
    {
        const BitMatrix bb = BitMatrix::random_dense(300, 1000, 0.5, 11);
        BitMatrix c_ref = BitMatrix::random_dense(900, 777, 0.5, 12), c_gpu = c_ref;
        const BitMatrix av = BitMatrix::random_dense(900, 128, 0.5, 13);
        struct Case { std::size_t row0, k, wcol0, n, c_row0, c_wcol0, rows, c; };
        const Case cases[] = {{0, 64, 0, 12, 0, 0, 900, 8}, {17, 64, 3, 5, 100, 4, 800, 13},
                              {250, 50, 7, 1, 3, 11, 500, 5}, {0, 1, 0, 12, 0, 0, 900, 8},
                              {100, 33, 2, 9, 899, 3, 1, 6}, {36, 64, 15, 1, 10, 0, 890, 16}};
        for (const Case& t : cases) {
            const auto splits = f2la::make_splits(t.k, t.c);
            const auto sp = std::span<const std::uint32_t>(splits);
            const auto a_words = av.col_words(t.c % 2, t.c_row0, t.rows);  // bits >= k must be ignored
            f2la::mult_acc(c_ref, t.c_row0, t.c_wcol0, a_words, f2la::build_tables(bb, t.row0, t.k, t.wcol0, t.n, sp));
            f2la::gpu::mult_acc(c_gpu, t.c_row0, t.c_wcol0, a_words,
                                f2la::gpu::build_tables(bb, t.row0, t.k, t.wcol0, t.n, sp));
            macc_ok = macc_ok && c_ref == c_gpu;
        }
        const BitMatrix small = BitMatrix::random_dense(40, 200, 0.5, 14);  // whole-matrix overloads
        f2la::mult_acc(c_ref, 5, 2, av.col_words(0, 5, 700), f2la::build_tables(small, std::size_t(8)));
        f2la::gpu::mult_acc(c_gpu, 5, 2, av.col_words(0, 5, 700), f2la::gpu::build_tables(small, std::size_t(8)));
        macc_ok = macc_ok && c_ref == c_gpu;
        std::vector<std::uint64_t> z(64);  // bare words (compute_Y: Y = D * Z)
        for (std::size_t t = 0; t < z.size(); ++t) z[t] = bb.word(t, 1);
        const auto zs = std::span<const std::uint64_t>(z);
        f2la::mult_acc(c_ref, 0, 6, av.col_words(1, 0, 900), f2la::build_tables(zs, std::size_t(8)));
        f2la::gpu::mult_acc(c_gpu, 0, 6, av.col_words(1, 0, 900), f2la::gpu::build_tables(zs, std::size_t(8)));
        macc_ok = macc_ok && c_ref == c_gpu;
        int thrown = 0;
        const auto s8 = f2la::make_splits(64, 8);
        try { f2la::gpu::build_tables(bb, 0, 65, 0, 1, std::span<const std::uint32_t>(f2la::make_splits(65, 8))); }
        catch (const std::invalid_argument&) { ++thrown; }
        try { f2la::gpu::build_tables(bb, 280, 64, 0, 1, std::span<const std::uint32_t>(s8)); }
        catch (const std::out_of_range&) { ++thrown; }
        try {
            f2la::gpu::mult_acc(c_gpu, 850, 0, av.col_words(0, 0, 100),
                                f2la::gpu::build_tables(bb, 0, 64, 0, 1, std::span<const std::uint32_t>(s8)));
        } catch (const std::out_of_range&) { ++thrown; }
        macc_ok = macc_ok && thrown == 3;
    }
    std::printf("mult %d  plu %d  rank %d (%zu)  recursive %d  null_space %d  solve %d  mult_acc %d\n", mult_ok,
                lu_ok, rank_ok, f.rank, rec_ok, ns_ok, solve_ok, macc_ok);
    return (mult_ok && lu_ok && rank_ok && rec_ok && ns_ok && solve_ok && macc_ok) ? 0 : 1;
}
