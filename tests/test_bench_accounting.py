"""bench.py's roofline arithmetic (SURVEY.md §8(d) algorithmic bytes) checked by hand on tiny
shapes -- CPU only (imports bench.py's helpers, runs nothing on a GPU)."""
import importlib.util
import os

import numpy as np

from synth import get_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_code_bytes_per_slot():
    b = _bench()
    assert b.code_bytes_per_slot(32, 256) == 32       # 8-bit codes
    assert b.code_bytes_per_slot(4, 16) == 2          # 4-bit codes (R16)
    assert b.code_bytes_per_slot(8, 1) == 0           # a single codeword carries no information


def test_algorithmic_scan_bytes_by_hand():
    """Two queries, nprobe 2, L 4, counts (3, 1, 4): per query D + valid*code + 4 nprobe + 8k
    (+ trace 4 nprobe L + 8 nprobe); the fixed-point variant has 4-byte coordinates and 8-byte
    distances."""
    b = _bench()
    cfg = get_config("c0").with_(D=16, M=4, Ks=256, nprobe=2, L=4, k=3)
    lists = np.array([[0, 1], [2, 0]])
    counts = np.array([3, 1, 4])
    valid = (3 + 1) + (4 + 3)
    ab = b.algorithmic_scan_bytes(cfg, lists, counts, trace=False)
    assert ab["valid_slots"] == valid
    assert ab["valid"] == 2 * 16 + valid * 4 + 2 * 4 * 2 + 2 * 8 * 3
    assert ab["padded"] == 2 * 16 + 2 * 2 * 4 * 4 + 2 * 4 * 2 + 2 * 8 * 3
    tr = b.algorithmic_scan_bytes(cfg, lists, counts, trace=True)
    assert tr["valid"] - ab["valid"] == 2 * (4 * 2 * 4 + 8 * 2)
    fx = b.algorithmic_scan_bytes(cfg, lists, counts, trace=True, fx=True)
    assert fx["valid"] == 2 * 16 * 4 + valid * 4 + 2 * 4 * 2 + 2 * 12 * 3 + 2 * (8 * 2 * 4 + 12 * 2)
