"""Build libshorb200.so in-tree for sm_100a with nvcc (no JIT cache).

    python -m paper_1801_01434_b200.build          # or __graft_entry__.build()

The .so lands next to this file so it travels with the repo snapshot to the
GPU box; _native.py loads exactly that file.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libshorb200.so"
SOURCES = ["capi.cu", "modexp.cu", "collapse.cu", "dft.cu", "dft_tc05.cu", "dft_i8.cu", "sample.cu", "context.cu", "gates.cu"]
# extra objects: (object stem, source, defines)
EXTRA = []
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-O2", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / "shb_internal.cuh", PKG.parent / "include" / "shorb200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    objdir = PKG / "_obj"
    objdir.mkdir(exist_ok=True)
    objs = []
    units = [(Path(src).stem, src, []) for src in SOURCES] + EXTRA
    for stem, src, defs in units:
        obj = objdir / (stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, *defs, "-I", str(PKG.parent / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        (objdir / (stem + ".ptxas.txt")).write_text(r.stderr)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", str(tmp), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
