"""Workload shapes: BASELINE.json's five configs plus the paper's Experiment-2 shapes.

Shapes only (no arithmetic of the method).  Names follow BASELINE.json; the paper's
symbols are given beside them (SURVEY.md §0 notation map):
  N  = N_0 (raw vectors), D, nlist = n_list, L = n (per-list capacity,
  PAPER.md:142), M (sub-quantizers), Ks = K (codewords per sub-quantizer,
  PAPER.md:144), nprobe = n_probe, k (top-k size).
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Config:
    name: str
    cfg_id: int          # seed component (SeedSequence([20260303, cfg_id, stream, chunk]))
    gen: str             # generator family: "c0" | "sift" | "deep" | "text"
    N: int               # database vectors (paper N_0)
    D: int               # dimension
    Q: int               # query batch size
    nlist: int           # inverted lists (paper n_list)
    L: int               # per-list capacity (paper n)
    M: int               # PQ sub-quantizers
    Ks: int              # codewords per sub-quantizer (paper K)
    nprobe: int          # lists probed per query (paper n_probe)
    k: int               # top-k size

    @property
    def d(self) -> int:
        """Sub-block dimension d = D / M ('D = Md')."""
        return self.D // self.M

    @property
    def n_sel(self) -> int:
        """Scan budget N_sel = n_probe * n."""
        return self.nprobe * self.L

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


# BASELINE.json "configs" (indices 0..4).
C0 = Config("tiny", 0, "c0", N=4096, D=16, Q=64, nlist=8, L=640, M=4, Ks=16, nprobe=2, k=10)
C1 = Config("sift", 1, "sift", N=100_000, D=128, Q=10_000, nlist=256, L=512, M=16, Ks=256, nprobe=8, k=10)
C2 = Config("deep", 2, "deep", N=1_000_000, D=96, Q=16_384, nlist=1024, L=1280, M=24, Ks=256, nprobe=16, k=10)
C3 = Config("text", 3, "text", N=1_000_000, D=768, Q=4_096, nlist=4096, L=320, M=96, Ks=256, nprobe=32, k=100)
C4 = Config("scale", 4, "sift", N=10_000_000, D=128, Q=16_384, nlist=16_384, L=768, M=32, Ks=256, nprobe=64, k=100)

# Paper Experiment-2 shapes, tuple (N_pad, D, M, K, n_list, n_probe, k);
# N_pad = n_list * n is the padded capacity, so n = N_pad / n_list; we take N_0 = floor(0.8 N_pad)
# and the C1 ("sift") generator at that D.
E2_BASIC = Config("e2_basic", 10, "sift", N=6553, D=128, Q=1024, nlist=256, L=32, M=8, Ks=16, nprobe=16, k=64)
E2_LOWACC = Config("e2_lowacc", 11, "sift", N=6553, D=128, Q=1024, nlist=16, L=512, M=8, Ks=1, nprobe=1, k=1)
E2_LARGE = Config("e2_large", 12, "sift", N=52_428, D=256, Q=512, nlist=512, L=128, M=16, Ks=256, nprobe=64, k=128)

# C4's per-list and per-query shape (D, L, M, Ks, nprobe, k) at a size the oracle finishes in
# seconds: a parity / debugging stand-in for the scale config.
C4_MINI = Config("c4_mini", 20, "sift", N=200_000, D=128, Q=1024, nlist=512, L=768, M=32, Ks=256, nprobe=64, k=100)

CONFIGS = {c.name: c for c in (C0, C1, C2, C3, C4, E2_BASIC, E2_LOWACC, E2_LARGE, C4_MINI)}
BASELINE_CONFIGS = (C0, C1, C2, C3, C4)


def get_config(name: str) -> Config:
    if name in CONFIGS:
        return CONFIGS[name]
    if name.startswith("c") and name[1:].isdigit():
        return BASELINE_CONFIGS[int(name[1:])]
    raise KeyError(name)
