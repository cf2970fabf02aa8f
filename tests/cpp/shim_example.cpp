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
    std::printf("mult %d  plu %d  rank %d (%zu)  recursive %d  null_space %d  solve %d\n", mult_ok, lu_ok,
                rank_ok, f.rank, rec_ok, ns_ok, solve_ok);
    return (mult_ok && lu_ok && rank_ok && rec_ok && ns_ok && solve_ok) ? 0 : 1;
}
