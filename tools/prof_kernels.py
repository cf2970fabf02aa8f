"""Launch the hot kernels a few times for ncu (one process, one GPU).

  python tools/prof_kernels.py update   # north-star unit C(65536^2) ^= A(65536x64) B(64x65536)
  python tools/prof_kernels.py gemm     # cfg2 16384^3 M4RM product
  python tools/prof_kernels.py panel    # a few panels of the 65536^2 decomposition
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "update"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = _lib.load()
ctx = f2.Context(0)
if what == "update":
    n = 65536
    Cm = f2.DeviceMatrix(n, n, ctx); Cm.random_dense(0.5, 101)
    Bm = f2.DeviceMatrix(64, n, ctx); Bm.random_dense(0.5, 102)
    a = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda")
    for _ in range(reps):
        _lib.check(lib.f2gpu_mult_acc(ctx.handle, Cm.handle, 0, 0, n // 64, C.c_void_p(a.data_ptr()),
                                      n, 64, Bm.handle, 0, 0))
elif what == "gemm":
    n = 16384
    A, B, Cm = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
    A.random_dense(0.5, 2); B.random_dense(0.5, 3)
    for _ in range(reps):
        _lib.check(lib.f2gpu_m4rm_mult(ctx.handle, A.handle, B.handle, Cm.handle, 0))
elif what == "strassen":
    n = 16384
    cut = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
    A, B, Cm = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
    A.random_dense(0.5, 2); B.random_dense(0.5, 3)
    for _ in range(reps):
        _lib.check(lib.f2gpu_strassen_mult(ctx.handle, A.handle, B.handle, Cm.handle, cut))
elif what == "decompose_rec":
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
    mc = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    A = f2.DeviceMatrix(n, n, ctx); A.random_dense(0.5, 6)
    import numpy as np
    perm = np.zeros(n, np.uint32); rj = np.zeros(n // 64, np.uint32); rk = C.c_size_t()
    for _ in range(reps):
        _lib.check(lib.f2gpu_decompose_recursive(ctx.handle, A.handle, mc, perm.ctypes.data, rj.ctypes.data, C.byref(rk)))
elif what == "decompose":
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
    A = f2.DeviceMatrix(n, n, ctx); A.random_dense(0.5, 6)
    import numpy as np
    perm = np.zeros(n, np.uint32); rj = np.zeros(n // 64, np.uint32); rk = C.c_size_t()
    for _ in range(reps):
        _lib.check(lib.f2gpu_decompose_block(ctx.handle, A.handle, perm.ctypes.data, rj.ctypes.data, C.byref(rk)))
ctx.sync()
print("done", what, ctx.launches())
