"""Build the sm_100a C-ABI library ``libspecbatch_b200.so`` in-tree.

``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` over each of
``csrc/*.cu`` (in parallel, objects under ``build/``), then ``nvcc -shared``; the CUDA runtime is linked statically so the library carries no
dependency on torch's runtime (device pointers and streams cross the C-ABI as
plain integers).  Cross-compiles on a GPU-less host.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libspecbatch_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build specbatch_b200")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    built = LIB.stat().st_mtime
    deps = sources() + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h")) + [Path(__file__)]
    return any(p.stat().st_mtime > built for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """One object per translation unit, compiled in parallel, then one shared link."""
    if not force and not _stale():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
             f"-I{INCLUDE}", f"-I{CSRC}"]
    jobs = []
    for src in sources():
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *flags, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        jobs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    errs = []
    for src, _, proc in jobs:
        _, err = proc.communicate()
        if proc.returncode != 0:
            errs.append(f"{src.name}: nvcc failed ({proc.returncode}):\n{err[-4000:]}")
    if errs:
        raise RuntimeError("\n".join(errs))
    cmd = [nvcc(), *ARCH, "-shared", "-Xlinker", "-z,defs", *(str(o) for _, o, _ in jobs), "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
