"""Device-trace one leaf-shaped block decomposition (n x w) and print the median
per-panel intervals of the lookahead chain (F2GPU_* env switches apply)."""
import ctypes as C
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
A = f2.DeviceMatrix(n, w, ctx); A.random_dense(0.5, 6)
W = f2.DeviceMatrix(n, w, ctx)
perm = np.zeros(n, np.uint32); rj = np.zeros(w // 64, np.uint32); rk = C.c_size_t()


def step():
    _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
    _lib.check(lib.f2gpu_decompose_block(ctx.handle, W.handle, perm.ctypes.data, rj.ctypes.data, C.byref(rk)))


cap = 1 << 20
_lib.check(lib.f2gpu_trace_enable(ctx.handle, cap))  # before warm-up: the captured graph carries it
buf = np.zeros(cap, np.uint64)
cnt = C.c_size_t()
for _ in range(3):
    step()
_lib.check(lib.f2gpu_trace_read(ctx.handle, buf.ctypes.data, cap, C.byref(cnt)))  # drop warm-up stamps
step()
_lib.check(lib.f2gpu_trace_read(ctx.handle, buf.ctypes.data, cap, C.byref(cnt)))
_lib.check(lib.f2gpu_trace_enable(ctx.handle, 0))
ev = buf[:cnt.value]
t = (ev >> np.uint64(16)).astype(np.int64)
code = ((ev >> np.uint64(12)) & np.uint64(15)).astype(int)
j = (ev & np.uint64(4095)).astype(int)
t0 = t.min()
names = {0: "P.w1end", 1: "P.begin", 2: "P.chain_end", 3: "P.end", 4: "post.begin", 5: "post.head", 6: "post.end",
         7: "U.begin", 8: "U.release", 9: "U.end", 10: "U0.tab0", 11: "U0.tile0", 12: "U0.end", 13: "P.done", 14: "U0.state", 15: "U0.barriers"}
mu = w // 64
T = {k: np.full(mu, np.nan) for k in names}
post_blk = []
# chain kernel (F2GPU_PANEL_CHAIN=1): helper stamps, code 0, panel | stage << 8
H = {st: np.full(mu, np.nan) for st in (1, 2, 3, 4, 5, 6, 7)}
for ti, ci, ji in zip(t, code, j):
    if ci == 0 and (ji >> 8) in H and (ji & 255) < mu and mu <= 256:
        H[ji >> 8][ji & 255] = (ti - t0) / 1000.0
for ti, ci, ji in zip(t, code, j):
    if ci == 0:
        continue
    if ci in T and ji < mu and np.isnan(T[ci][ji]):
        T[ci][ji] = (ti - t0) / 1000.0  # us


def med(x):
    x = x[~np.isnan(x)]
    return f"{np.median(x):7.2f} (p10 {np.percentile(x, 10):6.2f} p90 {np.percentile(x, 90):6.2f})" if x.size else "   n/a"


print(f"n={n} w={w} events={cnt.value} total {np.nanmax(T[6]) if not np.all(np.isnan(T[6])) else 0:.1f} us")
nx = lambda a: np.append(a[1:], np.nan)  # noqa: E731
rows = [
    ("panel chain (begin->chain end)", T[2] - T[1]),
    ("panel tail (chain end->end)", T[3] - T[2]),
    ("P end -> post begin", T[4] - T[3]),
    ("  P end -> P done (all warps)", T[13] - T[3]),
    ("  P done -> post begin", T[4] - T[13]),
    ("  P chain end -> warp 1 end", T[0] - T[2]),
    ("  P end (warp 2) -> warp 1 end", T[0] - T[3]),
    ("post begin -> head", T[5] - T[4]),
    ("post head -> next P begin", nx(T[1]) - T[5]),
    ("post begin -> post end", T[6] - T[4]),
    ("post end -> U begin", T[7] - T[6]),
    ("U begin -> release", T[8] - T[7]),
    ("  U0 begin -> state read", T[14] - T[7]),
    ("  U0 state -> barriers init", T[15] - T[14]),
    ("  U0 barriers -> first table", T[10] - T[15]),
    ("  U0 first table -> tile0 reduce", T[11] - T[10]),
    ("  U0 begin -> end (CTA 0)", T[12] - T[7]),
    ("  U0 end -> next post begin", nx(T[4]) - T[12]),
    ("next P chain end -> U release", nx(T[2]) - T[8]),
    ("cycle (P begin -> next P begin)", nx(T[1]) - T[1]),
]
rows += [
    ("chain: chain end -> warp 1 end", H[5] - T[2]),
    ("chain: chain end -> warp 2 replay end", H[6] - T[2]),
    ("chain: chain end -> helpers start", H[1] - T[2]),
    ("chain: helpers start -> col ready", H[2] - H[1]),
    ("chain:   U(j-1) release -> col ready", H[2] - np.append([np.nan], T[8][:-1])),
    ("chain: col ready -> gathered", H[3] - H[2]),
    ("chain: gathered -> hand-off", H[4] - H[3]),
    ("chain: hand-off -> next P begin", nx(T[1]) - H[4]),
]
for name, v in rows:
    print(f"{name:34s} {med(v)}")
if len(sys.argv) > 3:  # dump panels [a, a+k): event times relative to P(j) begin (us)
    a, k = int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 6
    cols = [(1, "P.beg"), (2, "P.chn"), (3, "P.end"), (13, "P.done"), (4, "po.beg"), (5, "po.head"), (6, "po.end"),
            (7, "U.beg"), (8, "U.rel"), (12, "U0.end")]
    print("panel " + " ".join(f"{nm:>8s}" for _, nm in cols) + "   (U(j-1).end0  U(j-1).beg)")
    for jj in range(a, min(mu, a + k)):
        b0 = T[1][jj]
        vals = " ".join(f"{T[c][jj] - b0:8.2f}" for c, _ in cols)
        prev = f"{T[12][jj - 1] - b0:8.2f} {T[7][jj - 1] - b0:8.2f}" if jj > 0 else ""
        print(f"{jj:5d} {vals}   ({prev})")
    if post_blk:
        jj = a + 1
        lo, hi = T[4][jj] - 0.5, T[6][jj] + 0.5
        sel = sorted(x for x in post_blk if lo <= x[0] <= hi)
        if sel:
            b0 = T[1][jj]
            ts = np.array([x[0] - b0 for x in sel])
            sms = np.array([x[1] for x in sel])
            print(f"post({jj}) block starts: {len(sel)} in [{ts.min():.2f}, {ts.max():.2f}] us after P({jj}) begin; "
                  f"{len(set(sms.tolist()))} distinct SMs; U({jj-1}) CTA0 end at {T[12][jj-1]-b0:.2f}")
            for q in (0.1, 0.25, 0.5, 0.75, 0.9):
                print(f"   {q:4.2f} quantile start {np.quantile(ts, q):7.2f}")
