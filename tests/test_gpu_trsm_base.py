"""decompose_recursive's TRSM base (k_trsm_block, csrc/kernels.cu) at every panel
count it takes: P <= 16 (128 threads), 17..32 (256 threads, the default base 32),
33..64 (F2GPU_REC_TBASE=64), each in both variants (F2GPU_TRSM_KERNEL=0/1),
against the CPU oracle.  The options are read once per process, so every setting
runs in a child process."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1209_5198_b200 as f2
from oracle import pyoracle as po

ctx = f2.Context(0)
cases = [
    # (rows, cols, min_cols, kind): the first split's left half is min_cols / 64 panels
    (8192, 8192, 4096, "dense"),      # left half 64 panels
    (6144, 6144, 3072, "dense"),      # 48 panels: P = 48 (base 64) / 24 (base 32)
    (6100, 6144, 3072, "deficient"),  # rank 3000: the rank-r_j fallback beside TRSM splits
    (7000, 5120, 2560, "dense"),      # 40 panels, tall
]
for n, m, mc, kind in cases:
    if kind == "dense":
        a = po.random_dense(n, m, 0.5, n + m)
    else:
        a = po.m4rm_mult(po.random_dense(n, 3000, 0.5, 3), n, 3000, po.random_dense(3000, m, 0.5, 4), m)
    w, perm, rj, rank = po.decompose_block(a, n, m)
    for rep in range(2):  # eager, then the captured leaf graphs
        lu = f2.decompose_recursive(f2.BitMatrix(n, m, a), min_cols=mc, ctx=ctx)
        assert lu.rank == rank, (n, m, mc, rep, lu.rank, rank)
        assert np.array_equal(lu.block_ranks, rj), (n, m, mc, rep)
        assert np.array_equal(lu.P.perm, perm), (n, m, mc, rep)
        assert np.array_equal(lu.overlay.words[:, :n], w[:, :n]), (n, m, mc, rep)
print("OK")
"""


@pytest.mark.parametrize("tbase,variant", [(16, 0), (32, 0), (32, 1), (64, 0), (64, 1)])
def test_trsm_base_panel_counts(tbase, variant):
    env = dict(os.environ, F2GPU_REC_TBASE=str(tbase), F2GPU_TRSM_KERNEL=str(variant))
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]
