"""Compile the sm_100a CUDA core into an in-tree shared library.

    python -m paper_2502_18113_b200._build      # or __graft_entry__.build()

Every translation unit under csrc/ is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked into
``paper_2502_18113_b200/lib/libflashann_b200.so`` (git-ignored; it travels to
the GPU box with the repo snapshot).  Builds are incremental on mtimes.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# FLASHANN_B200_LIBDIR: build into another directory (A/B experiment variants)
LIBDIR = Path(os.environ.get("FLASHANN_B200_LIBDIR") or PKG / "lib")
OBJDIR = LIBDIR / "obj"
LIB = LIBDIR / "libflashann_b200.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
              "--extended-lambda", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v"]
# diagnostics build: per-phase SM cycles of the layer search in point_stats
if os.environ.get("FLASHANN_B200_PHASE_PROFILE") == "1":
    NVCC_FLAGS.append("-DFA_PHASE_PROFILE=1")
# experiment builds: extra -D flags (e.g. "-DFA_PIPE=0")
NVCC_FLAGS += os.environ.get("FLASHANN_B200_NVCC_DEFS", "").split()


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA core cannot be built")


def _deps_mtime() -> float:
    files = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return max((f.stat().st_mtime for f in files), default=0.0)


def _compile(src: Path, force: bool, verbose: bool) -> tuple[Path, str]:
    obj = OBJDIR / (src.stem + ".o")
    if (not force and obj.exists()
            and obj.stat().st_mtime >= max(src.stat().st_mtime, _deps_mtime())):
        return obj, ""
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{p.stderr}")
    return obj, p.stderr if verbose else ""


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJDIR.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
