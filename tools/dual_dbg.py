import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1209_5198_b200 as f2
from oracle import pyoracle as po
ctx = f2.Context(0)
lib = f2._lib.load()
def tc(n, k, m, seed):
    a = po.random_dense(n, k, 0.5, seed); b = po.random_dense(k, m, 0.5, seed + 1)
    A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, k, a), ctx); B = f2.DeviceMatrix.from_host(f2.BitMatrix(k, m, b), ctx)
    C = f2.DeviceMatrix(n, m, ctx)
    f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C.handle, 0))
    got = C.download().words; want = po.m4rm_mult(a, n, k, b, m)
    bad = np.nonzero((got[:, :n] != want[:, :n]).any(axis=1))[0]
    return len(bad)
for (n, k, m) in [(512, 512, 512), (1024, 512, 1024), (4096, 512, 4096), (512, 1024, 512), (4096, 1024, 4096), (20000, 512, 2048), (512, 64, 512*40)]:
    print(os.environ.get("F2GPU_TC7_MODE"), (n, k, m), "bad word-cols:", tc(n, k, m, n + k))
def strass(n, leaf):
    a = po.random_dense(n, n, 0.5, 5); b = po.random_dense(n, n, 0.5, 6)
    try:
        ctx.set_tc(True, leaf)
        got = f2.strassen_mult(f2.BitMatrix(n, n, a), f2.BitMatrix(n, n, b), threshold=0, ctx=ctx)
    finally:
        ctx.set_tc(True)
    want = po.m4rm_mult(a, n, n, b, n)
    return int((got.words[:, :n] != want[:, :n]).any(axis=1).sum())
for n, leaf in [(2048, 512), (2048, 1024), (4096, 1024), (4096, 512)]:
    print("strassen", n, leaf, "bad:", strass(n, leaf))
