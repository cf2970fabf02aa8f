"""Time the fused M4RM Schur update (f2gpu_mult_acc, C ^= A*B with a rank-64 B)
on several shapes; the kernel is chosen by F2GPU_UPDATE (3 or 4).  Prints one
JSON line: {shape: us per launch}.  The north-star unit is 65536 x 65536."""
import ctypes as C
import json
import os
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
out = {"update": os.environ.get("F2GPU_UPDATE", "default")}
for n, m in [(65536, 65536), (65536, 8192), (16384, 16384), (4096, 4096)]:
    mu = m // 64
    Cm = f2.DeviceMatrix(n, m, ctx)
    Cm.random_dense(0.5, 101)
    Bm = f2.DeviceMatrix(64, m, ctx)
    Bm.random_dense(0.5, 102)
    a = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda")

    def launch():
        _lib.check(lib.f2gpu_mult_acc(ctx.handle, Cm.handle, 0, 0, mu, C.c_void_p(a.data_ptr()), n, 64,
                                      Bm.handle, 0, 0))

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        launch()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    gbs = (n * 8 + 64 * m // 8 + 2 * n * m // 8) / (us * 1e-6) / 1e9
    out[f"{n}x{m}"] = [round(us, 1), round(gbs, 1)]
    Cm.free()
    Bm.free()
print(json.dumps(out))
