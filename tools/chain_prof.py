"""k_panel_chain free-running (f2gpu_debug_panel_chain): its intrinsic per-panel cycle, and the launch ncu
captures (the chain cannot run under ncu inside the pipeline: it spins on kernels launched after it)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1209_5198_b200 as f2
from paper_1209_5198_b200 import _lib
lib = _lib.load(); ctx = f2.Context(0)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
A = f2.DeviceMatrix(n, w, ctx); W = f2.DeviceMatrix(n, w, ctx); A.random_dense(0.5, 6)
mu = w // 64
def run():
    _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
    _lib.check(lib.f2gpu_debug_panel_chain(ctx.handle, W.handle, mu))
for _ in range(2): run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); _lib.check(lib.f2gpu_debug_panel_chain(ctx.handle, W.handle, mu)); e1.record(stream)
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1000)
print(f"k_panel_chain free-running on {n} x {w}: {mu - 1} panels in {min(ts):.1f} us = {min(ts) / (mu - 1):.2f} us per panel")
