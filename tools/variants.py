"""decompose_block vs decompose_recursive on BASELINE cfg3 / cfg5 shapes (device-resident, CUDA events)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

lib = _lib.load()
ctx = f2.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
which = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
if which == "cfg5":
    n, m = 262144, 131072
    A = f2.DeviceMatrix(n, m, ctx); A.random_dense(0.05, 7)
else:  # cfg3: X (16384 x 12000) * Y (12000 x 65536)
    n, k, m = 16384, 12000, 65536
    X = f2.DeviceMatrix(n, k, ctx); X.random_dense(0.5, 4)
    Y = f2.DeviceMatrix(k, m, ctx); Y.random_dense(0.5, 5)
    A = f2.DeviceMatrix(n, m, ctx)
    _lib.check(lib.f2gpu_strassen_mult(ctx.handle, X.handle, Y.handle, A.handle, 0))
    X.free(); Y.free()
W = f2.DeviceMatrix(n, m, ctx)
perm = np.zeros(n, np.uint32); rj = np.zeros((m + 63) // 64, np.uint32); rk = C.c_size_t()
res = {"cfg": which}
for v in ("block", "recursive"):
    def step():
        _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
        if v == "block":
            _lib.check(lib.f2gpu_decompose_block(ctx.handle, W.handle, perm.ctypes.data, rj.ctypes.data, C.byref(rk)))
        else:
            _lib.check(lib.f2gpu_decompose_recursive(ctx.handle, W.handle, 0, perm.ctypes.data, rj.ctypes.data,
                                                     C.byref(rk)))
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(2):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    res[v] = {"ms": round(ms, 2), "rank": int(rk.value), "Gbitop_s": round(n * m * min(n, m) / (ms * 1e-3) / 1e9, 1)}
print(json.dumps(res))
