"""Leaf-shaped block decomposition (n x w) timing, graphs on/off via F2GPU_GRAPHS."""
import ctypes as C
import json
import os
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
A = f2.DeviceMatrix(n, w, ctx); A.random_dense(0.5, 6)
W = f2.DeviceMatrix(n, w, ctx)
perm = np.zeros(n, np.uint32); rj = np.zeros(w // 64, np.uint32); rk = C.c_size_t()


def step():
    _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
    _lib.check(lib.f2gpu_decompose_block(ctx.handle, W.handle, perm.ctypes.data, rj.ctypes.data, C.byref(rk)))


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(5):
    step()
e1.record(stream)
torch.cuda.synchronize()
print(json.dumps({"n": n, "w": w, "graphs": os.environ.get("F2GPU_GRAPHS", "1"), "ms": round(e0.elapsed_time(e1) / 5, 3)}))
