"""Run the reference's own 141 tests against this package.

The reference suite (/root/reference/pkg/tests, read-only, this container only)
imports ``scalesim``; a pytest plugin (tests/scalesim_alias.py) maps
``scalesim`` and its submodules onto ``paper_2412_17246_b200`` before
collection, so every assertion in the reference suite runs against our code.
The reference sources are never put on ``sys.path``.
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference suite only exists in the build container")
def test_reference_suite_passes_against_our_package():
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=f"{ROOT}:{ROOT / 'tests'}")
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "scalesim_alias",
         "--rootdir", str(ROOT), "-c", os.devnull, str(REF_TESTS)],
        capture_output=True, text=True, env=env, cwd=str(ROOT), timeout=600)
    tail = proc.stdout[-3000:] + proc.stderr[-2000:]
    assert proc.returncode == 0, tail
    # 141 reference tests; the preset round-trip test is parametrized over PRESETS,
    # which here also holds the two B200 documents -> 143
    m = re.search(r"(\d+) passed", proc.stdout)
    assert m and int(m.group(1)) >= 141 and "failed" not in proc.stdout, tail
