"""The reference's own test suite against the sm100 core.

oracle/_ref/refpkg.zip (built here by ``make -C oracle ref``; git-ignored, it
travels to the GPU box like the compiled reference core) holds the
reference's Python package and tests.  The test extracts it into a temporary
directory and runs, in a subprocess, the reference's tests/test_hnsw.py and
tests/test_flash.py with sm100 injected as the compiled core
(tests/refsuite/sm100_inject.py): every test parametrised over
``CORES = [_pycore, core.active_core()]`` (test_hnsw.py:13-15) and every
``EXT`` test (test_flash.py:23) runs on the GPU, and the reference's build()
and search_batch() route through sm100 as ``core_impl``.  A second file of
drop-in cases (tests/refsuite/dropin_cases.py) compares the public API's
results through sm100 with the reference's semantic core.
"""

import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET
import zipfile
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
ZIP = ROOT / "oracle" / "_ref" / "refpkg.zip"
HERE = Path(__file__).resolve().parent


def _run_suite(tmp_path, files, timeout=1500):
    assert ZIP.exists(), f"{ZIP} missing: run `make -C oracle ref` where /root/reference exists"
    with zipfile.ZipFile(ZIP) as z:
        z.extractall(tmp_path)
    shutil.copy(HERE / "refsuite" / "sm100_inject.py", tmp_path / "tests" / "sm100_inject.py")
    shutil.copy(HERE / "refsuite" / "dropin_cases.py", tmp_path / "tests" / "test_sm100_dropin.py")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(tmp_path / "src"), str(tmp_path / "tests"),
                                         str(ROOT)])
    env["FLASHANN_B200_REPO"] = str(ROOT)
    env.pop("FLASHANN_PURE_PYTHON", None)
    env.pop("FLASH_ANN_KERNEL", None)
    xml = tmp_path / "junit.xml"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "sm100_inject", "-p", "no:cacheprovider",
           f"--junitxml={xml}", "--rootdir", str(tmp_path / "tests"),
           *[str(tmp_path / "tests" / f) for f in files]]
    p = subprocess.run(cmd, cwd=tmp_path / "tests", env=env, capture_output=True, text=True,
                       timeout=timeout)
    cases = {}
    if xml.exists():
        for tc in ET.parse(xml).getroot().iter("testcase"):
            name = tc.get("classname", "") + "::" + tc.get("name", "")
            state = "passed"
            for child in tc:
                if child.tag in ("failure", "error"):
                    state = "failed"
                elif child.tag == "skipped":
                    state = "skipped"
            cases[name] = state
    return p, cases


def test_reference_suite_with_sm100_core(cuda, tmp_path):
    p, cases = _run_suite(tmp_path, ["test_hnsw.py", "test_flash.py", "test_sm100_dropin.py"])
    failed = sorted(k for k, v in cases.items() if v == "failed")
    sm100_cases = [k for k in cases if "sm100" in k]
    print(p.stdout[-3000:])
    assert cases, p.stdout[-3000:] + p.stderr[-3000:]
    assert not failed, "\n".join(failed) + "\n" + p.stdout[-6000:]
    # the CORES-parametrised tests ran on the GPU core, plus the drop-in cases
    assert len([k for k in sm100_cases if "[sm100]" in k]) == 7, sm100_cases
    assert len([k for k in cases if "test_sm100_dropin" in k]) == 5
    skipped = sorted(k for k, v in cases.items() if v == "skipped")
    assert not skipped, skipped
