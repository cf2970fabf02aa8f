#!/usr/bin/env python
"""bench.py — GF(2) block decomposition on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[3], the metric's headline): full
decomposition P*A = L*U of a 65536 x 65536 dense F2 matrix, bits Bernoulli(0.5)
from PackedMatrix::random_dense(seed 6) — synthetic input generated bit-exactly
on the device.  One step = copy A -> W (the API never modifies its input,
SPEC.md:379) + decompose_recursive(W) (--variant block: decompose_block(W);
both give the identical overlay, perm and r_j).  Metric: Gbitop/s = n^3 / t.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): word-columns round-robin over the ranks; decompose_recursive
replicates each leaf's columns once and every rank factors the leaf on its copy
(no per-panel exchange), the splits' TRSM + products are sharded by output
word-columns after one gather of the left columns (--variant block: one NCCL
broadcast per panel).  Strong scaling: the job is one 65536^2 decomposition.

The JSON line carries: value (device-resident, CUDA events, max over ranks),
parity (the LAST timed step's W, perm and r_j -- a CUDA-graph replay --
digested and compared with tests/golden/digests.json; exit 1 on mismatch),
e2e (through the C-ABI host entry point: H2D of A from pinned memory, the
decomposition, D2H of W/perm/r_j), roofline (the fused M4RM Schur update,
measured live as the north-star unit C(65536x65536) ^= A(65536x64) *
B(64x65536)), roofline_tensor (the fp4 product leaf), gemm (BASELINE
configs[1], 16384^2 products, with the reference's m4rm_mult timed beside it),
cpu_baseline (one FULL reference CPU decomposition of the same input on this
host's cores), clocks, gpu_launches.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
METRIC = "GF(2) decomposition Gbitop/s (n^3/t) at 65536^2"
UNIT = "Gbitop/s"


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def tensor_peak() -> tuple[float, str]:
    """Dense fp4 tensor peak in TFLOP/s: the measured bf16 burst GEMM figure x 4
    (fp4 : bf16 = 9 : 2.25 PFLOP/s dense, B200_PROFILING.md nominal table)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            bf16 = float(json.loads(p.read_text())["bf16_tflops"])
            return 4 * bf16, "derived: 4 x measured bf16 burst (MEASURED_PEAKS.json bf16_tflops)"
        except Exception:
            pass
    return 4 * 1590.0, "derived: 4 x fallback bf16 1.59 PFLOP/s (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# Parity of the benchmarked run: the order-independent digests of
# tests/golden/digests.json (computed once with oracle/_ref by
# tests/golden/make_golden.py), restated here in numpy so the bench does not
# load the oracle outside its CPU legs.
# ---------------------------------------------------------------------------
M64 = (1 << 64) - 1


def _mix64_int(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def digest_words(w: np.ndarray, n: int, m: int) -> int:
    """f2o_digest (oracle/f2oracle.c): mix64 sum over every word of the matrix,
    salted by row index and word-column; w is (mu, stride) uint64."""
    mu = (m + 63) // 64
    s = _mix64_int((n * 0x9E3779B97F4A7C15) ^ m)
    with np.errstate(over="ignore"):
        salt_i = np.arange(n, dtype=np.uint64) * np.uint64(0xD6E8FEB86659FD93)
        for q in range(mu):
            salt = np.uint64(_mix64_int(q + 0x1234567))
            s = (s + int(_mix64(w[q, :n] ^ salt_i ^ salt).sum(dtype=np.uint64))) & M64
    return s


def digest_cols(w: np.ndarray, n: int, cols: list[int]) -> int:
    """The digest's sum over the listed global word-columns only (w[l] = column
    cols[l]); the full digest is the base term plus the partial sums of every rank."""
    s = 0
    with np.errstate(over="ignore"):
        salt_i = np.arange(n, dtype=np.uint64) * np.uint64(0xD6E8FEB86659FD93)
        for l, q in enumerate(cols):
            salt = np.uint64(_mix64_int(q + 0x1234567))
            s = (s + int(_mix64(w[l, :n] ^ salt_i ^ salt).sum(dtype=np.uint64))) & M64
    return s


def digest_u32(v: np.ndarray) -> int:
    v = np.ascontiguousarray(v, dtype=np.uint32)
    with np.errstate(over="ignore"):
        x = (v.astype(np.uint64) << np.uint64(32)) ^ np.arange(v.size, dtype=np.uint64)
        return (_mix64_int(v.size) + int(_mix64(x).sum(dtype=np.uint64))) & M64


def golden(key: str) -> dict | None:
    p = ROOT / "tests" / "golden" / "digests.json"
    try:
        return json.loads(p.read_text()).get(key)
    except Exception:
        return None


def decomp_parity(cfg: dict, w: np.ndarray | None, perm: np.ndarray, rj: np.ndarray, rank: int,
                  w_digest: int | None = None) -> dict:
    key, g = None, None
    for k in ("cfg4", "cfg1"):
        e = golden(k)
        if e and (e["n"], e["m"], e["seed"], e["p"]) == (cfg["n"], cfg["m"], cfg["seed"], cfg["p"]):
            key, g = k, e
    if not g:
        return {"status": "unchecked", "why": "no committed digest for this configuration"}
    bad = []
    if rank != g["rank"]:
        bad.append(f"rank {rank} != {g['rank']}")
    if digest_u32(rj) != g["rj_digest"]:
        bad.append("r_j digest")
    if digest_u32(perm) != g["perm_digest"]:
        bad.append("perm digest")
    if w is not None and w_digest is None:
        w_digest = digest_words(w, cfg["n"], cfg["m"])
    if w_digest is not None and w_digest != g["w_digest"]:
        bad.append("W digest")
    return {"status": "ok" if not bad else "MISMATCH: " + ", ".join(bad),
            "checked": "rank, r_j, perm" + (", W" if w_digest is not None else "") +
                       f" of the last timed step vs tests/golden/digests.json {key} (oracle/_ref)"}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own M4RM (oracle/_ref, compiled from the
# reference headers) under the restated buildZ -- FULL decompositions.
# ---------------------------------------------------------------------------
class RefCpu:
    """The reference CPU decomposition of one input on this host's cores:
    oracle/_ref (reference m4rm.hpp build_tables/mult_acc + the restated buildZ,
    OpenMP over word-columns), or the oracle/f2oracle.c port when _ref is absent."""

    def __init__(self, n: int, m: int, p: float, seed: int):
        from oracle import pyoracle as po

        self.threads = os.cpu_count() or 1
        os.environ.setdefault("OMP_NUM_THREADS", str(self.threads))
        po.build(ref=False)
        self.po, self.n, self.m, self.seed = po, n, m, seed
        self.mu = (m + 63) // 64
        t0 = time.perf_counter()
        self.a = po.random_dense(n, m, p, seed)  # parallel jump-ahead twin of random_dense (pinned by tests)
        self.t_gen = time.perf_counter() - t0
        self.use_ref = po.ref_available()
        self.kind = "reference" if self.use_ref else "port"
        self.last = None

    def decompose(self, keep: bool = False) -> float:
        """One full decomposition; returns its wall time (generation and copies excluded)."""
        po, n, m, mu = self.po, self.n, self.m, self.mu
        perm = np.zeros(n, np.uint32)
        rj = np.zeros(mu, np.uint32)
        if self.use_ref:
            r = po.ref()
            h = r.ref_matrix_new(self.a, n, m, self.a.shape[1])
            t0 = time.perf_counter()
            rank = r.ref_decompose_block(h, perm, rj, 8, mu)
            dt = time.perf_counter() - t0
            w = None
            if keep:
                w = po.zeros(n, m)
                r.ref_matrix_read(h, w, w.shape[1])
            r.ref_matrix_free(h)
        else:
            w = self.a.copy()
            t0 = time.perf_counter()
            rank = po.lib().f2o_decompose_block(w, n, m, w.shape[1], perm, rj, 8, mu)
            dt = time.perf_counter() - t0
        if keep:
            self.last = (w, perm, rj, int(rank))
        return dt

    def sample(self, runs: int) -> str:
        what = ("reference m4rm.hpp build_tables/mult_acc compiled from the reference headers + restated buildZ"
                if self.use_ref else "oracle/f2oracle.c port")
        return (f"{runs} full {self.n}x{self.m} seed-{self.seed} decomposition(s), all {self.mu} panels "
                f"({what}), OpenMP {self.threads} threads, no extrapolation")


def cpu_baseline(n: int, m: int, p: float, seed: int) -> dict:
    rc = RefCpu(n, m, p, seed)
    dt = rc.decompose()
    return {"value": round(n * n * min(n, m) / dt / 1e9, 2), "unit": UNIT, "cores": rc.threads,
            "kind": rc.kind, "sample": rc.sample(1) + f": {dt:.2f} s", "t_s": round(dt, 3)}


def gemm_cpu_baseline(n: int, reps: int = 3) -> dict:
    """The reference's own m4rm_mult (m4rm.hpp:177-196, compiled from the reference
    headers into oracle/_ref, OpenMP over output word-columns) on the full n^3
    product with the same seeds, on all host cores: one warm-up + `reps` timed runs."""
    from oracle import pyoracle as po

    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    po.build(ref=False)
    if not po.ref_available():
        return {"unavailable": "oracle/_ref not built"}
    a = po.random_dense(n, n, 0.5, 2)
    b = po.random_dense(n, n, 0.5, 3)
    c = po.ref_m4rm_mult(a, n, n, b, n, tc=0)  # c = 0: the reference's cost-model table size
    g = golden("cfg2")
    ok = None if not g else po.digest(c, n, n) == g["c_digest"]
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        po.ref_m4rm_mult(a, n, n, b, n, tc=0)
        ts.append(time.perf_counter() - t0)
    dt = sum(ts) / len(ts)
    return {"value": round(n ** 3 / dt / 1e9, 1), "unit": UNIT, "ms": round(dt * 1e3, 1), "cores": threads,
            "kind": "reference", "parity": "ok" if ok else ("unchecked" if ok is None else "MISMATCH"),
            "sample": f"full {n}^3 reference m4rm_mult (table size from tuning, c=0), mean of {reps} runs"}


# ---------------------------------------------------------------------------
class StdoutToStderr:
    """File-descriptor level: NCCL prints its version banner on stdout when a
    communicator is created; rank 0's stdout must carry only the JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def run_reference(args, cfg) -> None:
    """The reference arm: W + K FULL CPU decompositions of the bench input (the
    reference's compiled M4RM + the restated buildZ, all host threads); value =
    n^3 / (mean time of the K timed runs).  Rank 0 only under torchrun."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    rc = RefCpu(cfg["n"], cfg["m"], cfg["p"], cfg["seed"])
    for i in range(args.warmup):
        rc.decompose(keep=(i == 0))
    t0 = time.perf_counter()
    ts = [rc.decompose() for _ in range(args.steps)]
    region = time.perf_counter() - t0
    t_step = sum(ts) / len(ts)
    v = round(cfg["n"] ** 2 * min(cfg["n"], cfg["m"]) / t_step / 1e9, 2)
    parity = {"status": "unchecked"}
    if rc.last is not None:
        w, perm, rj, rk = rc.last
        parity = decomp_parity(cfg, w, perm, rj, rk)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 1),
        "timed_region_s": round(region, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (random_dense seed %d, p=%g)" % (cfg["seed"], cfg["p"]),
        "config": cfg_json(cfg, args.gpus, args.variant),
        "parity": parity,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": rc.threads, "kind": rc.kind,
                         "sample": rc.sample(args.steps) + f" per step ({args.warmup} warm-up runs untimed)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_gemm:
        line["gemm"] = {"metric": "M4RM GEMM Gbitop/s (n^3/t), 16384^2 (BASELINE configs[1])",
                        "reference_m4rm_mult": gemm_cpu_baseline(16384)}
    print(json.dumps(line), flush=True)


VARIANTS = {
    "block": "decompose_block (lookahead 1: the panel chain in one persistent k_panel_chain CTA beside the "
             "graph-replayed posts and updates)",
    "recursive": "decompose_recursive (block leaves of <= 256 panels with lookahead: each leaf's panel chain is one "
                 "persistent k_panel_chain CTA, its posts and updates replayed from CUDA graphs; "
                 "TRSM + A' = D ^ L21 X products on the fp4 tensor-core leaf, Strassen-Winograd over 8192 leaves)",
}


def cfg_json(cfg, gpus, variant="block"):
    n, m = cfg["n"], cfg["m"]
    which = {65536: "BASELINE configs[3]", 4096: "BASELINE configs[0] size"}.get(n, "non-BASELINE size")
    mib = n * ((m + 63) // 64) * 8 / 2 ** 20
    return {"workload": f"decompose {n}x{m} dense F2, Bernoulli({cfg['p']}), seed {cfg['seed']} ({which})",
            "n": n, "m": m, "density": cfg["p"], "seed": cfg["seed"],
            "word_bits": 64, "tables": "k_update_v4: 8 x 8-bit tables per 8 word-column group (128 KiB shared memory per CTA)",
            "parallelism": f"column-round-robin x{gpus}" if gpus > 1 else "single GPU",
            "variant": VARIANTS[variant] + (f"; word-columns round-robin over {gpus} GPUs (f2gpu_decompose_{variant}_dist)"
                                            if gpus > 1 else ""),
            "l2": (f"inputs ({mib:.0f} MiB) larger than L2 (126 MB); no flush needed" if mib > 126
                   else f"inputs ({mib:.0f} MiB) fit in L2: warm-cache timing")}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=65536, help="matrix size (default: BASELINE cfg4)")
    ap.add_argument("--seed", type=int, default=6, help="input seed (cfg4: 6; cfg1 4096^2: 1)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gemm", action="store_true", help="skip the cfg2 16384^2 products")
    ap.add_argument("--force-dist", action="store_true",
                    help="one GPU through the distributed (NCCL) drivers with a 1-rank communicator")
    ap.add_argument("--variant", default="recursive", choices=["block", "recursive"],
                    help="decompose_recursive (default, fastest) or decompose_block; bit-identical factors")
    ap.add_argument("--min-cols", type=int, default=0, help="recursive leaf width in bits (0 = default)")
    args = ap.parse_args()
    cfg = {"n": args.n, "m": args.n, "p": 0.5, "seed": args.seed}

    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import paper_1209_5198_b200 as f2
    from paper_1209_5198_b200 import _lib

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    ctx = f2.Context(local)
    # a real (non-legacy) stream shared by torch events and the library's kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    # the distributed drivers (f2gpu_decompose_*_dist over NCCL): N > 1, or on one
    # GPU with --force-dist (a 1-rank communicator: checks this code path)
    dpath = world > 1 or args.force_dist
    with StdoutToStderr():
        if world > 1:
            obj = [f2.Context.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx.init_comm(rank, world, obj[0])
            dist.barrier()
        elif args.force_dist:
            os.environ["F2GPU_FORCE_NCCL"] = "1"
            ctx.init_comm(0, 1, f2.Context.nccl_unique_id())

    n, m = cfg["n"], cfg["m"]
    mu = (m + 63) // 64
    A = f2.DeviceMatrix(n, m, ctx)
    A.random_dense(cfg["p"], cfg["seed"])
    if world > 1:
        lw = int(lib.f2gpu_local_wcols(mu, rank, world))
        Aloc = f2.DeviceMatrix(n, lw * 64, ctx)
        _lib.check(lib.f2gpu_mat_select_wcols(ctx.handle, Aloc.handle, A.handle, rank, world, 0))
        A.free()
        A = Aloc
    W = f2.DeviceMatrix(A.n, A.m, ctx)
    perm = np.zeros(n, np.uint32)
    rj = np.zeros(mu, np.uint32)
    rk = C.c_size_t()

    def step():
        _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
        if dpath and args.variant == "recursive":
            _lib.check(lib.f2gpu_decompose_recursive_dist(ctx.handle, W.handle, m, args.min_cols, perm.ctypes.data,
                                                          rj.ctypes.data, C.byref(rk)))
        elif dpath:
            _lib.check(lib.f2gpu_decompose_block_dist(ctx.handle, W.handle, m, perm.ctypes.data,
                                                      rj.ctypes.data, C.byref(rk)))
        elif args.variant == "recursive":
            _lib.check(lib.f2gpu_decompose_recursive(ctx.handle, W.handle, args.min_cols,
                                                     perm.ctypes.data, rj.ctypes.data, C.byref(rk)))
        else:
            _lib.check(lib.f2gpu_decompose_block(ctx.handle, W.handle, perm.ctypes.data,
                                                 rj.ctypes.data, C.byref(rk)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ck = clocks.stop()
    launches = ctx.launches() - l0
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n * n * min(n, m) / (ms_step * 1e-3) / 1e9
    rank_found = int(rk.value)

    # ---- parity of the benchmarked (graph-replayed) run ----
    # every rank digests its own word-columns; the partial sums add up (mod 2^64)
    lcols = list(range(rank, mu, world))
    w_host = np.zeros((max(1, len(lcols)), (n + 7) // 8 * 8), np.uint64)
    if lcols:
        _lib.check(lib.f2gpu_mat_download(ctx.handle, W.handle, C.c_void_p(w_host.ctypes.data), w_host.shape[1]))
    part = digest_cols(w_host, n, lcols)
    if dist:
        t = torch.tensor([part - (1 << 64) if part >= (1 << 63) else part], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        part = int(t.item()) & M64
    w_dig = (_mix64_int((n * 0x9E3779B97F4A7C15) ^ m) + part) & M64
    parity = decomp_parity(cfg, None, perm, rj, rank_found, w_digest=w_dig) if rank == 0 else None
    del w_host

    # ---- roofline: the dominant kernel, measured live (north-star unit) ----
    roof = roof_tc = None
    if rank == 0:
        roof = measure_update_roofline(f2, lib, _lib, ctx, stream, torch, n)
        if args.variant == "recursive":
            roof_tc = measure_tensor_roofline(f2, lib, _lib, ctx, stream, torch)

    # ---- e2e through the C-ABI host entry point (pinned host buffers) ----
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(f2, lib, _lib, ctx, torch, A, n, m, mu, world, rank, dist, dpath,
                          steps=min(args.steps, 3), variant=args.variant, min_cols=args.min_cols,
                          warmup=args.warmup, cfg=cfg)

    gemm = None
    if not args.no_gemm and world == 1:
        gemm = measure_gemm(f2, lib, _lib, ctx, stream, torch, cpu=not args.no_cpu)
    elif not args.no_gemm:
        gemm = measure_gemm_dist(f2, lib, _lib, ctx, stream, torch, rank, world, dist)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(n, m, cfg["p"], cfg["seed"])
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": f"synthetic (random_dense seed {cfg['seed']}, p={cfg['p']}, generated on device)",
            "config": cfg_json(cfg, world, args.variant),
            "rank": rank_found, "parity": parity,
            "e2e": e2e, "roofline": roof, "roofline_tensor": roof_tc, "cpu_baseline": cpu, "clocks": ck,
            "gpu_launches": launches,
        }
        if gemm:
            line["gemm"] = gemm
        print(json.dumps(line), flush=True)
    bad = (parity and parity["status"] not in ("ok", "unchecked")) or (
        gemm and any(str(v.get("parity", "ok")) not in ("ok", "unchecked") for v in gemm.values() if isinstance(v, dict)))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if bad:
        print("bench: PARITY MISMATCH in the benchmarked results", file=sys.stderr, flush=True)
        sys.exit(1)


def measure_update_roofline(f2, lib, _lib, ctx, stream, torch, n: int) -> dict:
    """C(n x n) ^= A(n x 64) * B(64 x n) with the fused table-build + XOR kernel,
    averaged over back-to-back launches (C = 512 MiB > L2, so every launch streams
    C from HBM).  Algorithmic bytes = n*8 (A) + 64*n/8 (B) + 2*n*n/8 (C in+out)."""
    mu = n // 64
    Cm = f2.DeviceMatrix(n, n, ctx)
    Cm.random_dense(0.5, 101)
    Bm = f2.DeviceMatrix(64, n, ctx)
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
    t = e0.elapsed_time(e1) / reps * 1e-3
    alg = n * 8 + 64 * n // 8 + 2 * n * n // 8
    peak, src = peaks()
    ach = alg / t / 1e9
    traffic = None
    tp = ROOT / "profiles" / "update_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    Cm.free(); Bm.free()
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4), "traffic": traffic,
            "kernel": "k_update_v4 (fused M4RM table build + XOR sweep: 8-bit tables over 8-column groups, delta applied by bulk XOR reductions)",
            "unit_workload": f"C({n}x{n}) ^= A({n}x64)*B(64x{n})",
            "algorithmic_bytes": alg, "us_per_launch": round(t * 1e6, 1),
            "bitops_per_s": round(n * 64 * n / t, 1),
            "share_of_step": "19% of the decomposition's kernel time (profiles/r2d_launches_summary.txt)",
            "peak_source": src}


def measure_tensor_roofline(f2, lib, _lib, ctx, stream, torch, n: int = 16384) -> dict:
    """The fp4 tensor-core product leaf (k_gemm_tc7, CTA pairs) on C = A*B, n^3
    (BASELINE configs[1] shape): fp4 MACs executed = one per (i, j, k), 2 FLOP
    each.  The timed call includes the B^T staging transpose (~2% of it)."""
    Am, Bm, Cm = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
    Am.random_dense(0.5, 2)
    Bm.random_dense(0.5, 3)

    def launch():
        _lib.check(lib.f2gpu_gemm_tc(ctx.handle, Am.handle, Bm.handle, Cm.handle, 0))

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        launch()
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    peak, src = tensor_peak()
    ach = 2.0 * n ** 3 / t / 1e12
    traffic = None
    tp = ROOT / "profiles" / "tc7_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    Am.free(); Bm.free(); Cm.free()
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": round(peak, 1), "unit": "TFLOP/s",
            "frac": round(ach / peak, 4), "traffic": traffic,
            "kernel": "k_gemm_tc7 (fp4 kind::mxf4 GF(2) product leaf, cta_group::2, M-side operand in TMEM)",
            "unit_workload": f"C({n}x{n}) = A({n}x{n})*B({n}x{n}), 2*n^3 fp4 FLOP",
            "us_per_launch": round(t * 1e6, 1), "bitops_per_s": round(n ** 3 / t, 1),
            "share_of_step": "38% of the decomposition's kernel time (profiles/r2d_launches_summary.txt)",
            "peak_source": src}


def measure_e2e(f2, lib, _lib, ctx, torch, A, n, m, mu, world, rank, dist, dpath, steps: int,
                variant: str = "block", min_cols: int = 0, warmup: int = 3, cfg: dict | None = None) -> dict:
    """Same metric through the public C-ABI host entry point with host buffers:
    H2D of A (pinned) + decomposition + D2H of W, perm, r_j inside the region."""
    host_stride = (n + 7) // 8 * 8
    lw = A.m // 64 if world > 1 else mu
    words = torch.empty((lw, host_stride), dtype=torch.int64, pin_memory=True)
    wout = torch.empty((lw, host_stride), dtype=torch.int64, pin_memory=True)
    hA = words.numpy().view(np.uint64)
    hW = wout.numpy().view(np.uint64)
    # the input as a host matrix in the reference layout
    _lib.check(lib.f2gpu_mat_download(ctx.handle, A.handle, C.c_void_p(hA.ctypes.data), host_stride))
    perm = np.zeros(n, np.uint32)
    rj = np.zeros(mu, np.uint32)
    rk = C.c_size_t()

    def one():
        if dpath:
            Wd = f2.DeviceMatrix(n, lw * 64, ctx)
            Wd.upload_words(hA, host_stride)
            if variant == "recursive":
                _lib.check(lib.f2gpu_decompose_recursive_dist(ctx.handle, Wd.handle, m, min_cols, perm.ctypes.data,
                                                              rj.ctypes.data, C.byref(rk)))
            else:
                _lib.check(lib.f2gpu_decompose_block_dist(ctx.handle, Wd.handle, m, perm.ctypes.data,
                                                          rj.ctypes.data, C.byref(rk)))
            _lib.check(lib.f2gpu_mat_download(ctx.handle, Wd.handle, C.c_void_p(hW.ctypes.data),
                                              host_stride))
            Wd.free()
        elif variant == "recursive":
            _lib.check(lib.f2gpu_decompose_recursive_host(
                ctx.handle, C.c_void_p(hA.ctypes.data), n, m, host_stride, min_cols,
                C.c_void_p(hW.ctypes.data), perm.ctypes.data, rj.ctypes.data, C.byref(rk)))
        else:
            _lib.check(lib.f2gpu_decompose_block_host(
                ctx.handle, C.c_void_p(hA.ctypes.data), n, m, host_stride,
                C.c_void_p(hW.ctypes.data), perm.ctypes.data, rj.ctypes.data, C.byref(rk)))

    # warm-up calls as for the device metric: on a fresh box the first host<->device
    # copies run well below the link's steady rate (measured 104.9 vs 72.4 ms per step
    # with a single warm-up call)
    for _ in range(max(2, warmup)):
        one()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if dist:
        t = torch.tensor([dt], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    hbytes = lw * host_stride * 8
    parity = None
    if world == 1 and not dpath and cfg is not None:  # the host output of the last timed call
        parity = decomp_parity(cfg, hW, perm, rj, int(rk.value))["status"]
    return {"value": round(n * n * min(n, m) / dt / 1e9, 1), "unit": UNIT, "parity": parity,
            "h2d_bytes_per_step": hbytes * world,
            "d2h_bytes_per_step": hbytes * world + 4 * n + 4 * mu,
            "ms_per_step": round(dt * 1e3, 2),
            "api": (f"f2gpu_decompose_{variant}_host" if not dpath
                    else f"f2gpu_decompose_{variant}_dist + host upload/download")}


def measure_gemm_dist(f2, lib, _lib, ctx, stream, torch, rank, world, dist, n: int = 16384) -> dict:
    """BASELINE configs[1] on G GPUs: B and C word-columns round-robin,
    A broadcast from rank 0 (inside the timed region), local strassen_mult; the
    time is the max over ranks, the value the whole job's n^3 / t."""
    mu = n // 64
    lw = int(lib.f2gpu_local_wcols(mu, rank, world))
    Am = f2.DeviceMatrix(n, n, ctx)
    if rank == 0:
        Am.random_dense(0.5, 2)
    Bm = f2.DeviceMatrix(n, n, ctx)
    Bm.random_dense(0.5, 3)
    Bl, Cl = f2.DeviceMatrix(n, 64 * lw, ctx), f2.DeviceMatrix(n, 64 * lw, ctx)
    _lib.check(lib.f2gpu_mat_select_wcols(ctx.handle, Bl.handle, Bm.handle, rank, world, 0))
    Bm.free()

    def run():
        _lib.check(lib.f2gpu_strassen_mult_dist(ctx.handle, Am.handle, Bl.handle, Cl.handle, 0))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 5], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    Am.free(); Bl.free(); Cl.free()
    return {"metric": f"GF(2) multiply Gbitop/s (n^3/t), {n}^2, column-sharded over {world} GPUs "
                      "(A broadcast + local strassen_mult, max over ranks)",
            "ms": round(ms, 3), "Gbitop_s": round(n ** 3 / (ms * 1e-3) / 1e9, 1)}


def measure_gemm(f2, lib, _lib, ctx, stream, torch, cpu: bool = True) -> dict:
    """BASELINE configs[1]: C = A*B, A, B 16384^2 (seeds 2, 3): the M4RM kernel,
    Strassen-Winograd over M4RM leaves, the fp4 tensor-core leaf alone, and the
    default strassen_mult; each output is digested against tests/golden/digests.json
    cfg2 (oracle/_ref).  The reference's own m4rm_mult is timed beside them."""
    n = 16384
    Am, Bm, Cm = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
    Am.random_dense(0.5, 2)
    Bm.random_dense(0.5, 3)
    g = golden("cfg2")
    out = {}
    def smult(tc, cut):
        def run():
            ctx.set_tc(tc)
            _lib.check(lib.f2gpu_strassen_mult(ctx.handle, Am.handle, Bm.handle, Cm.handle, cut))
        return run

    variants = [("m4rm", lambda: _lib.check(lib.f2gpu_m4rm_mult(ctx.handle, Am.handle, Bm.handle, Cm.handle, 0)))]
    for cut in (16384, 8192, 4096):
        variants.append((f"strassen_m4rm_cut{cut}", smult(False, cut)))
    variants.append(("tc_fp4_leaf", lambda: _lib.check(lib.f2gpu_gemm_tc(ctx.handle, Am.handle, Bm.handle,
                                                                         Cm.handle, 0))))
    variants.append(("strassen_mult_default", smult(True, 0)))
    for name, fn in variants:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 5 * 1e-3
        par = "unchecked"
        if g:
            c = np.zeros((n // 64, n), np.uint64)
            _lib.check(lib.f2gpu_mat_download(ctx.handle, Cm.handle, C.c_void_p(c.ctypes.data), n))
            par = "ok" if digest_words(c, n, n) == g["c_digest"] else "MISMATCH"
        out[name] = {"ms": round(t * 1e3, 3), "Gbitop_s": round(n ** 3 / t / 1e9, 1), "parity": par}
    ctx.set_tc(True)
    Am.free(); Bm.free(); Cm.free()
    res = {"metric": "M4RM GEMM Gbitop/s (n^3/t), 16384^2 (BASELINE configs[1])",
           "value": out["strassen_mult_default"]["Gbitop_s"], "unit": UNIT, **out}
    if cpu:
        res["reference_m4rm_mult"] = gemm_cpu_baseline(n)
    return res


if __name__ == "__main__":
    main()
