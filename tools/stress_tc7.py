"""Stress the fp4 pair leaf (k_gemm_tc7): many shapes x repeats, each result
against the M4RM kernel's (bit-exact by construction).  Prints mismatch counts."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402

lib = f2._lib.load()
ctx = f2.Context(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
bad = total = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 200):
    n = int(rng.integers(1, 9000))
    k = int(rng.integers(1, 9000))
    m = 256 * int(rng.integers(1, 24))
    A, B = f2.DeviceMatrix(n, k, ctx), f2.DeviceMatrix(k, m, ctx)
    A.random_dense(0.5, it)
    B.random_dense([0.5, 0.95, 0.05][it % 3], it + 1000)
    C1, C2 = f2.DeviceMatrix(n, m, ctx), f2.DeviceMatrix(n, m, ctx)
    f2._lib.check(lib.f2gpu_m4rm_mult(ctx.handle, A.handle, B.handle, C1.handle, 0))
    want = C1.download().words
    for rep in range(3):
        f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C2.handle, rep % 2))
        got = C2.download().words
        ref = want if rep % 2 == 0 else np.zeros_like(want)  # acc=1 over C = A*B gives 0
        if rep % 2 == 1:
            ok = not (got[:, :n] != 0).any()
        else:
            ok = np.array_equal(got[:, :n], ref[:, :n])
        total += 1
        if not ok:
            bad += 1
            print("MISMATCH", (n, k, m, rep), flush=True)
    for x in (A, B, C1, C2):
        x.free()
print(f"stress_tc7: {bad} mismatches in {total} products")
sys.exit(1 if bad else 0)
