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
    std::printf("mult %d  plu %d  rank %d (%zu)  recursive %d\n", mult_ok, lu_ok, rank_ok, f.rank,
                rec_ok);
    return (mult_ok && lu_ok && rank_ok && rec_ok) ? 0 : 1;
}
