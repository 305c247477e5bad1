"""The debug build (libv3db_debug.so, -DV3DB_DEBUG): every shared-memory candidate append, stage and
descriptor write whose bound rests on a protocol argument traps if the bound is ever violated,
and V3DB_SYNC_CHECK=1 synchronizes after each launch group.  compute-sanitizer is closed on this
pool, so this is the memory-safety check: the whole small workload (tools/sanitize_case.py: every
scan kernel and table geometry, the mma.sync coarse path, the fixed-point path on C0, the E2
shapes and c4_mini) must run without a trap and match the oracle bit for bit."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_library_runs_clean():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_03065_b200 import build as libbuild
    path = libbuild.build(variant="debug")
    assert path.endswith("libv3db_debug.so")
    env = dict(os.environ, V3DB_LIB="debug", V3DB_SYNC_CHECK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), "c0", "e2_basic",
                        "c4_mini", "e2_large"], env=env, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "libv3db_debug.so" in r.stdout
    for name in ("c0", "e2_basic", "c4_mini", "e2_large"):
        assert f"ok {name}" in r.stdout
