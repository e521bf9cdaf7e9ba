"""Build libgs2b200.so in-tree with nvcc for sm_100a (no torch C++ ABI coupling).

    python -m paper_2104_01196_b200.build [--force] [--verbose]

Objects are compiled in parallel into paper_2104_01196_b200/_build/ and linked
into paper_2104_01196_b200/_build/libgs2b200.so, which travels to the GPU box
with the repo snapshot (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
LIB = OUT / "libgs2b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# host code: -ffp-contract=off keeps a*b + c as two roundings (the reference's numpy arithmetic)
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-ffp-contract=off",
         "--expt-relaxed-constexpr",
         f"-I{ROOT / 'include'}", "-Xptxas", "-v"]


def sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "gs2b200.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool) -> Path:
    obj = OUT / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src.name}")
    (OUT / (src.stem + ".ptxas.txt")).write_text(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    OUT.mkdir(exist_ok=True)
    if not force and not _stale(LIB, _deps()):
        return LIB
    srcs = sources()
    hdrs = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "gs2b200.h"]
    todo = [s for s in srcs if force or _stale(OUT / (s.stem + ".o"), [s, *hdrs])]
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(todo)))) as ex:
        list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [str(OUT / (s.stem + ".o")) for s in srcs]
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(p)
