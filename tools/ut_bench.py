"""Time the tensor-core trailing update on the north-star shape as a rank-128 pass:
C(65536^2) ^= A(65536 x 128) * B(128 x 65536), vs two rank-64 M4RM updates."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

lib = _lib.load()
ctx = f2.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
kw = int(sys.argv[2]) if len(sys.argv) > 2 else 2
Cm = f2.DeviceMatrix(n, n, ctx); Cm.random_dense(0.5, 101)
A = f2.DeviceMatrix(n, 64 * kw, ctx); A.random_dense(0.5, 102)
BT = f2.DeviceMatrix(n, 64 * kw, ctx); BT.random_dense(0.5, 103)
Bm = f2.DeviceMatrix(64, n, ctx); Bm.random_dense(0.5, 104)
a = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda")


def tc():
    _lib.check(lib.f2gpu_update_tc(ctx.handle, Cm.handle, 0, n, 0, n // 64, A.handle, 0, kw, BT.handle))


def m4rm():
    for _ in range(kw):
        _lib.check(lib.f2gpu_mult_acc(ctx.handle, Cm.handle, 0, 0, n // 64, C.c_void_p(a.data_ptr()), n, 64,
                                      Bm.handle, 0, 0))


res = {"n": n, "rank": 64 * kw}
for name, fn in (("tc", tc), ("m4rm", m4rm)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    bytes_ = 2 * n * (n // 64) * 8
    res[name] = {"us": round(us, 1), "c_gbs": round(bytes_ / (us * 1e-6) / 1e9, 1)}
print(json.dumps(res))
