"""A/B timing of the fp4 product leaf: f2gpu_gemm_tc on n x k x m shapes
(CUDA events, mean of reps after warm-up).  Run twice with F2GPU_TC7=0/1."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

SHAPES = [(16384, 16384, 16384), (8192, 8192, 8192), (32768, 1024, 32768), (57344, 4096, 8192),
          (4096, 1024, 57344), (1024, 1024, 8192), (32768, 32768, 32768)]


def main():
    lib = _lib.load()
    ctx = f2.Context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    tag = os.environ.get("F2GPU_TC7", "1") + "/" + os.environ.get("F2GPU_TC7_MODE", "0")
    shapes = SHAPES
    if os.environ.get("SHAPES"):
        shapes = [tuple(int(x) for x in s.split("x")) for s in os.environ["SHAPES"].split(",")]
    for n, k, m in shapes:
        A, B, Cm = f2.DeviceMatrix(n, k, ctx), f2.DeviceMatrix(k, m, ctx), f2.DeviceMatrix(n, m, ctx)
        A.random_dense(0.5, 1)
        B.random_dense(0.5, 2)
        run = lambda: _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, Cm.handle, 0))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            run()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"tc7={tag} {n}x{k}x{m}: {ms * 1e3:9.1f} us  {2 * n * k * m / ms / 1e9:8.1f} TFLOP/s(fp4)", flush=True)
        A.free(); B.free(); Cm.free()


if __name__ == "__main__":
    main()
