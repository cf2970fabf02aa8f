"""In-tree build of libf2gpu.so (sm_100a) with nvcc.

The shared library is the product: hand-written CUDA kernels + the native
host drivers behind the C-ABI declared in include/f2gpu.h.  It is built in
place (paper_1209_5198_b200/libf2gpu.so) so it travels with the repo snapshot
to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libf2gpu.so"
SOURCES = [CSRC / "kernels.cu", CSRC / "tc_leaf.cu", CSRC / "tc_pair.cu", CSRC / "api.cu"]
HEADERS = [CSRC / "kernels.cuh", CSRC / "tc_common.cuh", CSRC / "options.h", ROOT / "include" / "f2gpu.h"]

# F2GPU_BUILD_EXPERIMENTAL=1 also compiles the evaluated-and-rejected variants
# (int8 leaves, single-CTA pair / persistent / double-buffered fp4 leaves, the
# tensor-core update); the default library carries only the kernels in use.
EXPERIMENTAL = os.environ.get("F2GPU_BUILD_EXPERIMENTAL", "0") == "1"
# csrc/experimental/: whole files of evaluated-and-rejected kernels (the tensor-core
# trailing update), compiled only into experimental builds
if EXPERIMENTAL:
    SOURCES.insert(3, CSRC / "experimental" / "tc_update.cu")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    f"-DF2GPU_EXPERIMENTAL={1 if EXPERIMENTAL else 0}",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-diag-suppress", "177",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libf2gpu.so")


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-shared", "-o", str(tmp), *map(str, SOURCES), "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
