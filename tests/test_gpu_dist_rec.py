"""decompose_recursive over word-column shards on one GPU.

f2gpu_decompose_recursive_sharded runs the distributed recursion's schedule
(f2gpu_dist_schedule: each leaf factored whole on a replicated copy, one left-column gather per
split, TRSM + A' product on each shard's own right-half columns) over G
logical shards with device-to-device exchanges; f2gpu_decompose_recursive_dist
runs it through NCCL (a 1-rank communicator here).  Every result must equal the
CPU oracle (or the committed oracle/_ref digests at full size) bit-for-bit.
"""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def _sharded(f2, ctx, a, n, m, G, min_cols):
    from paper_1209_5198_b200 import _lib

    W = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, a), ctx)
    perm = np.zeros(n, np.uint32)
    rj = np.zeros((m + 63) // 64, np.uint32)
    rk = C.c_size_t()
    _lib.check(_lib.load().f2gpu_decompose_recursive_sharded(ctx.handle, W.handle, G, min_cols, perm.ctypes.data,
                                                              rj.ctypes.data, C.byref(rk)))
    w = W.download()
    W.free()
    return w, perm, rj, int(rk.value)


@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("n,m,p,min_cols", [(1000, 1000, 0.5, 128), (2048, 4096, 0.5, 256), (3000, 1280, 0.1, 64),
                                            (700, 2000, 0.5, 64)])
def test_recursive_sharded_matches_oracle(f2, ctx, po, G, n, m, p, min_cols):
    a = po.random_dense(n, m, p, n + m + G)
    w0, p0, r0, k0 = po.decompose_block(a, n, m)
    w, perm, rj, rank = _sharded(f2, ctx, a, n, m, G, min_cols)
    assert rank == k0 and np.array_equal(rj, r0) and np.array_equal(perm, p0)
    assert np.array_equal(w.words[:, :n], w0[:, :n])


@pytest.mark.parametrize("G", [2, 5])
def test_recursive_sharded_rank_deficient(f2, ctx, po, G):
    n, k, m = 2500, 700, 3000
    a = po.m4rm_mult(po.random_dense(n, k, 0.5, 4), n, k, po.random_dense(k, m, 0.5, 5), m)
    w0, p0, r0, k0 = po.decompose_block(a, n, m)
    w, perm, rj, rank = _sharded(f2, ctx, a, n, m, G, 128)
    assert rank == k0 == k and np.array_equal(rj, r0) and np.array_equal(perm, p0)
    assert np.array_equal(w.words[:, :n], w0[:, :n])


def test_recursive_sharded_cfg4_digest(f2, ctx, po):
    """BASELINE configs[3] (65536^2, seed 6) over 8 logical shards, default leaves."""
    from paper_1209_5198_b200 import _lib

    g = json.loads((GOLD / "digests.json").read_text())["cfg4"]
    n = g["n"]
    A = f2.DeviceMatrix(n, n, ctx)
    A.random_dense(0.5, g["seed"])
    perm = np.zeros(n, np.uint32)
    rj = np.zeros(n // 64, np.uint32)
    rk = C.c_size_t()
    _lib.check(_lib.load().f2gpu_decompose_recursive_sharded(ctx.handle, A.handle, 8, 0, perm.ctypes.data,
                                                              rj.ctypes.data, C.byref(rk)))
    assert int(rk.value) == g["rank"]
    assert po.digest_u32(rj) == g["rj_digest"] and po.digest_u32(perm) == g["perm_digest"]
    assert po.digest(A.download().words, n, n) == g["w_digest"]
    A.free()


def test_recursive_dist_through_nccl_one_rank(f2, po, monkeypatch):
    import torch  # noqa: F401  (loads torch's libnccl.so.2 first, as in bench.py)

    from paper_1209_5198_b200 import _lib

    monkeypatch.setenv("F2GPU_FORCE_NCCL", "1")
    lib = _lib.load()
    ctx = f2.Context(0)
    ctx.init_comm(0, 1, f2.Context.nccl_unique_id())
    for n, m, mc in [(2000, 1500, 128), (3000, 4096, 256)]:
        a = po.random_dense(n, m, 0.5, 41 + n)
        W = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, a), ctx)
        perm = np.zeros(n, np.uint32)
        rj = np.zeros((m + 63) // 64, np.uint32)
        rk = C.c_size_t()
        _lib.check(lib.f2gpu_decompose_recursive_dist(ctx.handle, W.handle, m, mc, perm.ctypes.data,
                                                      rj.ctypes.data, C.byref(rk)))
        w, p0, r0, rank = po.decompose_block(a, n, m)
        assert rk.value == rank and np.array_equal(perm, p0) and np.array_equal(rj, r0)
        assert np.array_equal(W.download().words[:, :n], w[:, :n])
        W.free()
    ctx.close()


def test_recursive_sharded_cfg5_digest(f2, ctx, po):
    """BASELINE configs[4] (262144 x 131072, p = 0.05, 4 GiB) over 8 logical shards."""
    from paper_1209_5198_b200 import _lib

    p5 = GOLD / "digests_cfg5.json"
    if not p5.exists():
        pytest.skip("cfg5 digest not generated")
    g = json.loads(p5.read_text())["cfg5"]
    n, m = g["n"], g["m"]
    A = f2.DeviceMatrix(n, m, ctx)
    A.random_dense(g["p"], g["seed"])
    perm = np.zeros(n, np.uint32)
    rj = np.zeros(m // 64, np.uint32)
    rk = C.c_size_t()
    _lib.check(_lib.load().f2gpu_decompose_recursive_sharded(ctx.handle, A.handle, 8, 0, perm.ctypes.data,
                                                              rj.ctypes.data, C.byref(rk)))
    assert int(rk.value) == g["rank"]
    assert po.digest_u32(rj) == g["rj_digest"] and po.digest_u32(perm) == g["perm_digest"]
    assert po.digest(A.download().words, n, m) == g["w_digest"]
    A.free()


def test_recursive_dist_nccl_cfg4_digest(f2, po, monkeypatch):
    """The NCCL driver (1-rank communicator) on the bench configuration."""
    import torch  # noqa: F401

    from paper_1209_5198_b200 import _lib

    monkeypatch.setenv("F2GPU_FORCE_NCCL", "1")
    g = json.loads((GOLD / "digests.json").read_text())["cfg4"]
    n = g["n"]
    ctx = f2.Context(0)
    ctx.init_comm(0, 1, f2.Context.nccl_unique_id())
    A = f2.DeviceMatrix(n, n, ctx)
    A.random_dense(0.5, g["seed"])
    perm = np.zeros(n, np.uint32)
    rj = np.zeros(n // 64, np.uint32)
    rk = C.c_size_t()
    _lib.check(_lib.load().f2gpu_decompose_recursive_dist(ctx.handle, A.handle, n, 0, perm.ctypes.data,
                                                          rj.ctypes.data, C.byref(rk)))
    assert int(rk.value) == g["rank"]
    assert po.digest_u32(rj) == g["rj_digest"] and po.digest_u32(perm) == g["perm_digest"]
    assert po.digest(A.download().words, n, n) == g["w_digest"]
    A.free()
    ctx.close()


def test_recursive_sharded_leaf_graphs_replay(f2, ctx, po):
    """Whole-leaf mode replays each leaf from a captured CUDA graph from the third
    call with the same shape (the leaf runs on the context's persistent copy, so
    the graph does not depend on the caller's buffers or on G): eager, capture,
    replays -- with different inputs (full rank, rank-deficient, sparse) and
    different shard counts through the same graphs, every call against the oracle."""
    n, m, mc = 3000, 2560, 640   # 40 panels, leaves of 10
    inputs = [po.random_dense(n, m, 0.5, 91), po.random_dense(n, m, 0.5, 92),
              po.m4rm_mult(po.random_dense(n, 900, 0.5, 93), n, 900, po.random_dense(900, m, 0.5, 94), m),
              po.random_dense(n, m, 0.03, 95), po.random_dense(n, m, 0.5, 96)]
    for a, G in zip(inputs, [2, 2, 3, 8, 1]):
        w0, p0, r0, k0 = po.decompose_block(a, n, m)
        w, perm, rj, rank = _sharded(f2, ctx, a, n, m, G, mc)
        assert rank == k0 and np.array_equal(rj, r0) and np.array_equal(perm, p0), G
        assert np.array_equal(w.words[:, :n], w0[:, :n]), G


_CHILD_PER_PANEL = r"""
import sys
sys.path.insert(0, sys.argv[1])
import ctypes as C
import numpy as np
import paper_1209_5198_b200 as f2
from paper_1209_5198_b200 import _lib
from oracle import pyoracle as po

ctx = f2.Context(0)
lib = _lib.load()
for n, m, p, mc, G in [(1000, 1000, 0.5, 128, 2), (2048, 4096, 0.5, 256, 3), (3000, 1280, 0.1, 64, 8)]:
    a = po.random_dense(n, m, p, n + m + G)
    w0, p0, r0, k0 = po.decompose_block(a, n, m)
    W = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, a), ctx)
    perm = np.zeros(n, np.uint32)
    rj = np.zeros((m + 63) // 64, np.uint32)
    rk = C.c_size_t()
    _lib.check(lib.f2gpu_decompose_recursive_sharded(ctx.handle, W.handle, G, mc, perm.ctypes.data,
                                                     rj.ctypes.data, C.byref(rk)))
    assert rk.value == k0 and np.array_equal(rj, r0) and np.array_equal(perm, p0), (n, m, G)
    assert np.array_equal(W.download().words[:, :n], w0[:, :n]), (n, m, G)
    W.free()
print("OK")
"""


def test_recursive_sharded_per_panel_mode():
    """F2GPU_DIST_LEAF=0: the per-panel replication schedule (panel / apply callbacks)
    stays bit-exact.  Options are read once per process, hence the child."""
    import os
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, F2GPU_DIST_LEAF="0")
    r = subprocess.run([sys.executable, "-c", _CHILD_PER_PANEL, str(root)], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]
