"""Stage the reference package for the GPU box (TEST INFRASTRUCTURE ONLY).

    python oracle/stage_ref.py          # (make -C oracle ref runs it)

Packs the reference's Python package (/root/reference/pkg/src/flashann, *.py
only: the compiled core is oracle/_ref/_core*.so) and its test suite
(/root/reference/pkg/tests) into oracle/_ref/refpkg.zip.  oracle/_ref/ is
git-ignored (nothing of the reference enters the history) but not
gpurun-ignored, so the archive travels to the GPU box, where
tests/test_gpu_reference_suite.py extracts it into a temporary directory and
runs the reference's own tests with the sm100 core injected as the compiled
core.
"""

from __future__ import annotations

import sys
import zipfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")
OUT = HERE / "_ref" / "refpkg.zip"


def stage(ref: Path = REF, out: Path = OUT) -> Path:
    src = ref / "src" / "flashann"
    tests = ref / "tests"
    if not src.is_dir() or not tests.is_dir():
        raise FileNotFoundError(f"reference package not found under {ref}")
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".tmp")
    def put(z, f, name):
        # fixed timestamps (the read-only tree's mtimes predate what zip stores)
        z.writestr(zipfile.ZipInfo(name, (1980, 1, 1, 0, 0, 0)), f.read_bytes(),
                   zipfile.ZIP_DEFLATED)

    with zipfile.ZipFile(tmp, "w") as z:
        for f in sorted(src.rglob("*.py")):
            put(z, f, "src/" + str(f.relative_to(ref / "src")))
        for f in sorted(tests.glob("*.py")):
            put(z, f, "tests/" + f.name)
    tmp.replace(out)
    return out


if __name__ == "__main__":
    print(stage(Path(sys.argv[1]) if len(sys.argv) > 1 else REF))
