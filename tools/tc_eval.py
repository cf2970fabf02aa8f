"""Evaluate the tensor-core GF(2) leaf (k_gemm_tc) against the oracle and time it
against the M4RM GEMM on 16384^3 (BASELINE configs[1])."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

lib = _lib.load()
ctx = f2.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
ok = True
import os  # noqa: E402

SH = [(256, 64, 128), (256, 128, 128), (512, 64, 256), (256, 640, 384), (256, 64, 256), (512, 192, 512), (1024, 1024, 1024),
      (2048, 4096, 1536)]
if os.environ.get("F2GPU_TC_KIND", "f4")[0] != "i":  # fp4 leaf: ragged n and k, m % 256 == 0
    SH = [(240, 64, 256), (1, 1, 256), (7, 100, 512), (480, 320, 256), (1000, 777, 768), (2048, 4096, 1536),
          (4097, 130, 256), (3000, 5000, 1024)]
for (n, k, m) in SH:
    a = po.random_dense(n, k, 0.5, n + k)
    b = po.random_dense(k, m, 0.5, k + m)
    want = po.m4rm_mult(a, n, k, b, m)
    A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, k, a), ctx)
    B = f2.DeviceMatrix.from_host(f2.BitMatrix(k, m, b), ctx)
    Cm = f2.DeviceMatrix(n, m, ctx)
    _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, Cm.handle, 0))
    got = Cm.download()
    eq = np.array_equal(got.words[:, :n], want[:, :n])
    ok &= eq
    print(f"tc {n}x{k}x{m}: {'OK' if eq else 'MISMATCH'}", flush=True)
    if not eq:
        d = got.words[:, :n] ^ want[:, :n]
        print("  mismatching words:", int(np.count_nonzero(d)), "of", d.size)
if not ok and not os.environ.get("F2GPU_TC_MODE"):
    sys.exit(1)
n = 16384
A, B, Cm = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
A.random_dense(0.5, 2)
B.random_dense(0.5, 3)
res = {}
for name, fn in (("tc", lambda: _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, Cm.handle, 0))),
                 ("m4rm", lambda: _lib.check(lib.f2gpu_m4rm_mult(ctx.handle, A.handle, B.handle, Cm.handle, 0)))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5
    res[name] = {"ms": round(t, 3), "Gbitop_s": round(n ** 3 / (t * 1e-3) / 1e9, 1)}
    if name == "tc":
        d_tc = po.digest(Cm.download().words, n, n)
    else:
        d_m = po.digest(Cm.download().words, n, n)
res["tc_equals_m4rm_16384"] = d_tc == d_m
print(json.dumps(res))
