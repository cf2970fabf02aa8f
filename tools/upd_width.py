"""M4RM update efficiency vs width: C(n x 64w) ^= A(n x 64) * B(64 x 64w), HBM GB/s."""
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
a = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda")
out = []
for w in (1024, 255, 128, 64, 32, 16, 4, 1):
    Cm = f2.DeviceMatrix(n, 64 * w, ctx); Cm.random_dense(0.5, 1)
    Bm = f2.DeviceMatrix(64, 64 * w, ctx); Bm.random_dense(0.5, 2)

    def run():
        _lib.check(lib.f2gpu_mult_acc(ctx.handle, Cm.handle, 0, 0, w, C.c_void_p(a.data_ptr()), n, 64, Bm.handle, 0, 0))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(stream)
    for _ in range(reps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    out.append({"w": w, "us": round(us, 2), "GBs": round(2 * n * w * 8 / (us * 1e-6) / 1e9, 1)})
    Cm.free(); Bm.free()
print(json.dumps({"n": n, "widths": out}))
