"""bench.py's own legs at the BASELINE configs[0] size (4096^2, seed 1, the cfg1
digest): the reference arm on CPU (full oracle/_ref decompositions, digest-checked
output) and, on a B200, the device arm through the single-GPU and the distributed
(1-rank NCCL communicator) drivers with the parity check of the timed output."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout  # ONE JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_full_runs_cfg1():
    if not (ROOT / "oracle" / "_ref" / "libf2la_ref.so").exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    d = _run(["--impl", "reference", "--n", "4096", "--seed", "1", "--steps", "2", "--warmup", "1", "--no-gemm"])
    assert d["impl"] == "reference" and d["parity"]["status"] == "ok"
    assert d["cpu_baseline"]["kind"] == "reference" and "no extrapolation" in d["cpu_baseline"]["sample"]
    assert d["e2e"]["value"] == d["value"] and d["steps"] == 2
    assert abs(d["ms_per_step"] - 4096 ** 3 / (d["value"] * 1e9) * 1e3) < 0.1


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--variant", "block"], ["--force-dist"], ["--force-dist", "--variant", "block"]])
def test_device_arm_cfg1_parity(extra):
    d = _run(["--n", "4096", "--seed", "1", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-gemm", *extra])
    assert d["parity"]["status"] == "ok", d["parity"]
    assert d["e2e"]["parity"] in ("ok", None)
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_mhz"]
