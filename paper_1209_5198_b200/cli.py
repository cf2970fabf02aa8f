"""bench_cli-compatible command line, on the B200 path.

  python -m paper_1209_5198_b200.cli gen    --n N [--m M] [--density D] [--seed S] --out F [--format text|binary]
  python -m paper_1209_5198_b200.cli bench  --n N [N ...] [--variant block|recursive|both] [--reps R] [--seed S]
  python -m paper_1209_5198_b200.cli verify (--in F | --n N [--m M] [--density D] [--seed S])
  python -m paper_1209_5198_b200.cli rank   --in F

bench prints the reference CSV schema "n,b,c,variant,time_ms,rank":
time is the minimum over repetitions of the decomposition alone,
device-resident, CUDA events (generation and I/O excluded).  c is
the largest M4RM group width of the device tables (7x8 + 8 bits).
Exit codes: 0 success, 1 invariant violation, 2 usage error.
"""
from __future__ import annotations

import argparse
import ctypes as C
import sys

import numpy as np

from . import BitMatrix, Context, DeviceMatrix, _lib, decompose_block, m4rm_mult, rank
from .io import read_matrix, write_matrix


def _gen(args, ctx) -> BitMatrix:
    m = args.m or args.n
    return BitMatrix.random_dense(args.n, m, args.density, args.seed, ctx=ctx)


def cmd_gen(args, ctx) -> int:
    write_matrix(_gen(args, ctx), args.out, args.format)
    return 0


def cmd_bench(args, ctx) -> int:
    import torch

    lib = _lib.load()
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    variants = ["block", "recursive"] if args.variant == "both" else [args.variant]
    print("n,b,c,variant,time_ms,rank")
    for n in args.n:
        A = DeviceMatrix(n, n, ctx)
        A.random_dense(args.density, args.seed)
        W = DeviceMatrix(n, n, ctx)
        perm = np.zeros(n, np.uint32)
        rj = np.zeros((n + 63) // 64, np.uint32)
        rk = C.c_size_t()
        for v in variants:
            best = float("inf")
            for rep in range(args.reps + 1):
                _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                if v == "block":
                    _lib.check(lib.f2gpu_decompose_block(ctx.handle, W.handle, perm.ctypes.data,
                                                         rj.ctypes.data, C.byref(rk)))
                else:
                    _lib.check(lib.f2gpu_decompose_recursive(ctx.handle, W.handle, 0,
                                                             perm.ctypes.data, rj.ctypes.data,
                                                             C.byref(rk)))
                e1.record(stream)
                torch.cuda.synchronize()
                if rep:  # first run is a warm-up
                    best = min(best, e0.elapsed_time(e1))
            print(f"{n},64,7,{v},{best:.3f},{rk.value}", flush=True)
        A.free()
        W.free()
    return 0


def verify(a: BitMatrix, ctx) -> list[str]:
    """Recomposition P*A == L*U (GPU product), rank(A) == rank(A^T), L/U structure."""
    errs = []
    n, m = a.rows(), a.cols()
    f = decompose_block(a, ctx=ctx)
    if not f.P.is_bijection():
        errs.append("P is not a permutation")
    L, U = f.L, f.U
    pa = BitMatrix(n, m, a.words[:, f.P.perm]) if n else a
    lu = m4rm_mult(L, U, ctx=ctx) if f.rank else BitMatrix(n, m)
    if not (pa == lu):
        errs.append("recomposition P*A != L*U")
    at = BitMatrix(m, n)
    if n and m:
        da = DeviceMatrix.from_host(a, ctx)  # keep a reference: the handle must outlive the launch
        dt = DeviceMatrix(m, n, ctx)
        _lib.check(_lib.load().f2gpu_mat_transpose(ctx.handle, da.handle, dt.handle))
        at = dt.download()
        da.free()
        dt.free()
    if rank(at, ctx=ctx) != f.rank:
        errs.append("rank(A) != rank(A^T)")
    Ld = L.to_dense()
    for i in range(min(f.rank, n)):
        if Ld[i, i] != 1 or Ld[i, i + 1:].any():
            errs.append(f"L row {i} is not unit lower trapezoidal")
            break
    R = 0
    Ud = U.to_dense()
    for j, r in enumerate(f.block_ranks.tolist()):
        if r and Ud[R:R + r, :64 * j].any():
            errs.append(f"U block row {j} is not on the staircase")
            break
        R += r
    return errs


def cmd_verify(args, ctx) -> int:
    a = read_matrix(args.inp) if args.inp else _gen(args, ctx)
    errs = verify(a, ctx)
    for e in errs:
        print("FAIL:", e)
    if not errs:
        print(f"ok: {a.rows()}x{a.cols()} passes recomposition, rank and structure checks")
    return 1 if errs else 0


def cmd_rank(args, ctx) -> int:
    print(rank(read_matrix(args.inp), ctx=ctx))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1209_5198_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--m", type=int, default=0)
    g.add_argument("--density", type=float, default=0.5)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", required=True)
    g.add_argument("--format", choices=["text", "binary"], default="binary")
    b = sub.add_parser("bench")
    b.add_argument("--n", type=int, nargs="+", required=True)
    b.add_argument("--variant", choices=["block", "recursive", "both"], default="both")
    b.add_argument("--reps", type=int, default=10)
    b.add_argument("--density", type=float, default=0.5)
    b.add_argument("--seed", type=int, default=1)
    v = sub.add_parser("verify")
    v.add_argument("--in", dest="inp")
    v.add_argument("--n", type=int, default=256)
    v.add_argument("--m", type=int, default=0)
    v.add_argument("--density", type=float, default=0.5)
    v.add_argument("--seed", type=int, default=1)
    r = sub.add_parser("rank")
    r.add_argument("--in", dest="inp", required=True)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    ctx = Context(0)
    return {"gen": cmd_gen, "bench": cmd_bench, "verify": cmd_verify, "rank": cmd_rank}[args.cmd](args, ctx)


if __name__ == "__main__":
    sys.exit(main())
