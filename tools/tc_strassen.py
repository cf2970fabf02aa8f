"""Time f2gpu_strassen_mult (the paper's multiply) at n^3 on the current leaf
settings (F2GPU_TC, F2GPU_TC_CUT from the environment)."""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A, B, Cm = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
A.random_dense(0.5, 2)
B.random_dense(0.5, 3)


def run():
    _lib.check(lib.f2gpu_strassen_mult(ctx.handle, A.handle, B.handle, Cm.handle, 0))


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record(stream)
for _ in range(reps):
    run()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
from oracle import pyoracle as po  # noqa: E402
print(json.dumps({"n": n, "tc": os.environ.get("F2GPU_TC", "1"), "tc_cut": os.environ.get("F2GPU_TC_CUT", "none"),
                  "ms": round(ms, 3), "Gbitop_s": round(n ** 3 / (ms * 1e-3) / 1e9, 1),
                  "digest": po.digest(Cm.download().words, n, n)}))
