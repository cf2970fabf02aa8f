"""cfg5 digest (262144 x 131072, p=0.05, seed 7) from oracle/_ref — ~15 min on 8 cores.
Run in the build container: python tests/golden/make_golden_cfg5.py"""
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from oracle import pyoracle as po  # noqa: E402

n, m, p, seed = 262144, 131072, 0.05, 7
t = time.time()
a = po.random_dense(n, m, p, seed)
tg = time.time() - t
w, perm, rj, rank = po.ref_decompose_block(a, n, m)
out = {"cfg5": {"n": n, "m": m, "p": p, "seed": seed, "rank": rank,
                "input_digest": po.digest(a, n, m), "w_digest": po.digest(w, n, m),
                "perm_digest": po.digest_u32(perm), "rj_digest": po.digest_u32(rj),
                "source": "oracle/_ref (reference m4rm.hpp + restated buildZ)",
                "gen_seconds": round(tg, 1), "seconds": round(time.time() - t, 1)}}
(HERE / "digests_cfg5.json").write_text(json.dumps(out, indent=1))
print(out)
