"""GPU: every kernel family and edge case through the bounds-checked build
(libmatchb200_dbg.so, -DMB_BOUNDS_CHECK): each staged-smem window and global
text read is asserted in-kernel and traps on violation.  compute-sanitizer is
closed on this GPU pool; this is its stand-in."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checked_build_runs_all_families(cuda):
    lib = os.path.join(ROOT, "paper_1012_2547_b200", "libmatchb200_dbg.so")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1012_2547_b200", "csrc"), "debug"], check=True)
    env = dict(os.environ, MB_ENGINE_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize cases ok" in r.stdout
    assert "MB_CHECK failed" not in r.stdout + r.stderr
