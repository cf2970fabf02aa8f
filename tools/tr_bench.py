"""Bandwidth of the 64x64 bit-tile transpose (k_transpose) on a few shapes."""
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
for n, m in ((32768, 32768), (16384, 32768), (8192, 65536), (65536, 8192)):
    A = f2.DeviceMatrix(n, m, ctx)
    A.random_dense(0.5, 1)
    T = f2.DeviceMatrix(m, n, ctx)
    for _ in range(3):
        _lib.check(lib.f2gpu_mat_transpose(ctx.handle, A.handle, T.handle))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        _lib.check(lib.f2gpu_mat_transpose(ctx.handle, A.handle, T.handle))
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    gb = 2 * n * m / 8 / 1e9
    print(json.dumps({"n": n, "m": m, "us": round(us, 1), "GBs": round(gb / (us * 1e-6), 1)}))
    A.free()
    T.free()
