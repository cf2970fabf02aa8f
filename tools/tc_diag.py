"""Repeatability check of the tensor-core leaf on multi-wave shapes: TC vs M4RM,
mismatching word counts per run (diagnostic tool)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

lib = _lib.load()
ctx = f2.Context(0)
for (n, k, m) in [(4096, 4096, 4096), (16384, 1024, 16384), (16384, 16384, 16384)]:
    A, B, Ct, Cm = f2.DeviceMatrix(n, k, ctx), f2.DeviceMatrix(k, m, ctx), f2.DeviceMatrix(n, m, ctx), f2.DeviceMatrix(n, m, ctx)
    A.random_dense(0.5, 2)
    B.random_dense(0.5, 3)
    _lib.check(lib.f2gpu_m4rm_mult(ctx.handle, A.handle, B.handle, Cm.handle, 0))
    ctx.sync()
    ref = torch.from_numpy(Cm.download().words.view("int64").copy())
    bad = []
    for rep in range(4):
        _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, Ct.handle, 0))
        ctx.sync()
        got = torch.from_numpy(Ct.download().words.view("int64").copy())
        d = (got ^ ref)[:, :n]
        nz = d.nonzero()
        bad.append(int(nz.shape[0]))
        if nz.shape[0] and rep == 0:
            print("  first bad (wcol,row):", nz[:4].tolist(), flush=True)
    print(f"{n}x{k}x{m}: mismatching words per run {bad}", flush=True)
