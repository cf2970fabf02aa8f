"""Generate tests/golden/* from the REFERENCE compiled in place (oracle/_ref).

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py [--big]
The fixtures pin the plain-C oracle (tests/test_oracle.py) and, through it, the
GPU parity tests.  --big also computes full-size digests (cfg1..cfg4) with the
reference decomposition (minutes on 8 cores).
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from oracle import pyoracle as po  # noqa: E402

po.build(ref=True)
r = po.ref()

# PRNG outputs (prng.hpp:18-47)
prng = {}
for seed in [0, 1, 6, 0xDEADBEEF, 2**64 - 1]:
    out = np.zeros(16, np.uint64)
    r.ref_rng_outputs(seed, out, 16)
    prng[str(seed)] = [int(x) for x in out]
(HERE / "prng.json").write_text(json.dumps({"xorshift64star": prng}, indent=1))

# random_dense (bit_matrix.hpp:125-142)
rd_meta, rd = {}, {}
for (n, m, p, seed) in [(4, 5, 0.5, 1), (100, 130, 0.5, 7), (65, 64, 0.05, 3), (300, 1000, 0.3, 0),
                        (17, 1, 0.5, 9), (50, 70, 1.0, 2), (50, 70, 0.0, 2), (129, 4097, 0.5, 6),
                        (200, 300, 0.05, 7)]:
    k = f"rd_{n}_{m}_{p}_{seed}"
    rd_meta[k] = [n, m, p, seed]
    rd[k] = po.ref_random_dense(n, m, p, seed)
np.savez_compressed(HERE / "random_dense.npz", **rd)
(HERE / "random_dense.json").write_text(json.dumps(rd_meta, indent=1))

# m4rm_mult (m4rm.hpp:177-196)
mm_meta, mm = {}, {}
for (n, k, m) in [(1, 1, 1), (64, 64, 64), (300, 129, 200), (100, 1000, 65), (257, 63, 300)]:
    key = f"mm_{n}_{k}_{m}"
    sa, sb = n + k, k + m + 1
    a = po.random_dense(n, k, 0.5, sa)
    b = po.random_dense(k, m, 0.5, sb)
    mm[key] = po.ref_m4rm_mult(a, n, k, b, m, 0)  # c = 0 -> cost-model table size
    mm_meta[key] = [n, k, m, sa, sb]
np.savez_compressed(HERE / "m4rm.npz", **mm)
(HERE / "m4rm.json").write_text(json.dumps(mm_meta, indent=1))

# transposed (bit_matrix.hpp:220-238)
tr = {}
for (n, m) in [(64, 64), (100, 37), (37, 100), (130, 1)]:
    a = po.random_dense(n, m, 0.5, n + m)
    out = po.zeros(m, n)
    r.ref_transpose(a, n, m, a.shape[1], out, out.shape[1])
    tr[f"{n}x{m}"] = out
np.savez_compressed(HERE / "transpose.npz", **tr)

# decomposition via the reference's build_tables/mult_acc + restated buildZ
dc_meta, dc = {}, {}
for (n, m, p, seed) in [(4, 5, 0.5, 1), (64, 64, 0.5, 2), (200, 130, 0.1, 3), (130, 200, 0.5, 4),
                        (256, 256, 0.01, 5), (300, 64, 0.5, 6), (77, 500, 0.5, 8)]:
    key = f"dc_{n}_{m}_{p}_{seed}"
    a = po.random_dense(n, m, p, seed)
    w, perm, rj, rank = po.ref_decompose_block(a, n, m)
    dc[key + "_w"], dc[key + "_perm"], dc[key + "_rj"] = w, perm, rj
    dc[key + "_rank"] = np.array(rank)
    dc_meta[key] = [n, m, p, seed]
np.savez_compressed(HERE / "decompose.npz", **dc)
(HERE / "decompose.json").write_text(json.dumps(dc_meta, indent=1))

# full-size digests
dg_path = HERE / "digests.json"
dg = json.loads(dg_path.read_text()) if dg_path.exists() else {}
cfgs = {"cfg1": (4096, 4096, 0.5, 1)}
if "--big" in sys.argv:
    cfgs.update({"cfg4": (65536, 65536, 0.5, 6)})
for name, (n, m, p, seed) in cfgs.items():
    t = time.time()
    a = po.random_dense(n, m, p, seed)
    w, perm, rj, rank = po.ref_decompose_block(a, n, m)
    dg[name] = {"n": n, "m": m, "p": p, "seed": seed, "rank": rank,
                "input_digest": po.digest(a, n, m), "w_digest": po.digest(w, n, m),
                "perm_digest": po.digest_u32(perm), "rj_digest": po.digest_u32(rj),
                "source": "oracle/_ref (reference m4rm.hpp + restated buildZ)",
                "seconds": round(time.time() - t, 1)}
    print(name, dg[name], flush=True)
if "--big" in sys.argv:
    # cfg2 product digest, cfg3 (X*Y then decompose) digests
    t = time.time()
    n = 16384
    a, b = po.random_dense(n, n, 0.5, 2), po.random_dense(n, n, 0.5, 3)
    c = po.ref_m4rm_mult(a, n, n, b, n, 8)
    dg["cfg2"] = {"n": n, "seedA": 2, "seedB": 3, "c_digest": po.digest(c, n, n),
                  "seconds": round(time.time() - t, 1)}
    print("cfg2", dg["cfg2"], flush=True)
    t = time.time()
    x, y = po.random_dense(16384, 12000, 0.5, 4), po.random_dense(12000, 65536, 0.5, 5)
    a = po.m4rm_mult(x, 16384, 12000, y, 65536)
    w, perm, rj, rank = po.ref_decompose_block(a, 16384, 65536)
    dg["cfg3"] = {"n": 16384, "m": 65536, "k": 12000, "seedX": 4, "seedY": 5, "rank": rank,
                  "a_digest": po.digest(a, 16384, 65536), "w_digest": po.digest(w, 16384, 65536),
                  "perm_digest": po.digest_u32(perm), "rj_digest": po.digest_u32(rj),
                  "seconds": round(time.time() - t, 1)}
    print("cfg3", dg["cfg3"], flush=True)
dg_path.write_text(json.dumps(dg, indent=1))
