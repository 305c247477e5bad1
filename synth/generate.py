"""Seeded, chunked synthetic generators (SURVEY.md §8(d) "Synthetic inputs").

The paper evaluates on SIFT1M, GIST1M and MS MARCO; none
of them is available here, so these generators stand in for them, borrowing only
their shapes as BASELINE.json prescribes.  Seeds: SeedSequence([20260303, cfg_id,
stream, chunk]) with streams 0 = mixture parameters, 1 = database, 2 = queries,
3 = centroid rows, 4 = codeword rows (drawn in subspace order).  Rows are generated
in chunks of 2**20, each chunk with its own seed, so large configs never need
multi-GB float64 temporaries.

Nothing here is arithmetic of the V3DB method: these are the method's INPUTS.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .configs import Config

ROOT_SEED = 20260303
CHUNK = 1 << 20
STREAM_MIX, STREAM_DB, STREAM_Q, STREAM_CENT, STREAM_CODE = 0, 1, 2, 3, 4
STREAM_Q_RANK = 100  # + rank: the independent query batch of rank > 0 in a multi-GPU run


def _rng(cfg_id: int, stream: int, chunk: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([ROOT_SEED, cfg_id, stream, chunk]))


@dataclass
class Mixture:
    gen: str
    D: int
    centres: np.ndarray            # [ncomp, D] float64
    scale: np.ndarray | None       # [D] anisotropic per-dim scale ("text" only)
    sigma: float


def mixture(gen: str, D: int, cfg_id: int) -> Mixture:
    """Mixture parameters of BASELINE.json's generator families (stream 0)."""
    rng = _rng(cfg_id, STREAM_MIX)
    if gen == "c0":          # 8 components, centres U[-48,48]^D, sigma 8
        return Mixture(gen, D, rng.uniform(-48.0, 48.0, (8, D)), None, 8.0)
    if gen == "sift":        # 64 components, centres U[0,255]^D, sigma 20
        return Mixture(gen, D, rng.uniform(0.0, 255.0, (64, D)), None, 20.0)
    if gen == "deep":        # 256 unit-norm centres; noise 0.5/sqrt(D)
        c = rng.standard_normal((256, D))
        c /= np.linalg.norm(c, axis=1, keepdims=True)
        return Mixture(gen, D, c, None, 0.5 / np.sqrt(D))
    if gen == "text":        # 1024 unit-norm centres, anisotropic scale U[0.5,1.5]^D drawn first
        s = rng.uniform(0.5, 1.5, D)
        c = rng.standard_normal((1024, D))
        c /= np.linalg.norm(c, axis=1, keepdims=True)
        return Mixture(gen, D, c, s, 0.5 / np.sqrt(D))
    raise ValueError(f"unknown generator {gen!r}")


def _float_rows(mix: Mixture, rng: np.random.Generator, n: int) -> np.ndarray:
    """The real-valued vectors before BASELINE.json's int8 quantisation (used as they are by the
    16-bit fixed-point variant, NEXT-1): c0 / sift mixtures clipped to their value range, deep /
    text rows unit-normalised."""
    comp = rng.integers(0, mix.centres.shape[0], size=n)
    noise = rng.standard_normal((n, mix.D), dtype=np.float32)
    x = mix.centres[comp].astype(np.float32) + np.float32(mix.sigma) * noise
    if mix.gen == "c0":
        return np.clip(x, -127, 127)
    if mix.gen == "sift":
        return np.clip(x, 0, 255) - np.float32(128)
    if mix.scale is not None:
        x *= mix.scale.astype(np.float32)
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def _rows(mix: Mixture, rng: np.random.Generator, n: int) -> np.ndarray:
    comp = rng.integers(0, mix.centres.shape[0], size=n)
    noise = rng.standard_normal((n, mix.D), dtype=np.float32)
    x = mix.centres[comp].astype(np.float32) + np.float32(mix.sigma) * noise
    if mix.gen == "c0":
        return np.clip(np.rint(x), -127, 127).astype(np.int8)
    if mix.gen == "sift":    # uint8 0..255, stored shifted to int8 (distances are shift-invariant)
        return (np.clip(np.rint(x), 0, 255).astype(np.int16) - 128).astype(np.int8)
    if mix.scale is not None:
        x *= mix.scale.astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return np.clip(np.rint(127.0 * x), -127, 127).astype(np.int8)


def _chunked(fill, n: int) -> None:
    """fill(c, lo, hi) for every chunk [lo, hi) of CHUNK rows; chunks are independently seeded, so
    a thread pool (numpy's generators and arithmetic release the GIL) gives the same bytes."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    spans = [(c, lo, min(n, lo + CHUNK)) for c, lo in enumerate(range(0, n, CHUNK))]
    if len(spans) <= 1:
        for sp in spans:
            fill(*sp)
        return
    with ThreadPoolExecutor(max_workers=min(len(spans), os.cpu_count() or 4)) as ex:
        list(ex.map(lambda sp: fill(*sp), spans))


def gen_vectors(cfg: Config, stream: int, n: int) -> np.ndarray:
    """n int8 rows of dimension cfg.D from the config's mixture, chunk-seeded."""
    mix = mixture(cfg.gen, cfg.D, cfg.cfg_id)
    out = np.empty((n, cfg.D), dtype=np.int8)

    def fill(c, lo, hi):
        out[lo:hi] = _rows(mix, _rng(cfg.cfg_id, stream, c), hi - lo)
    _chunked(fill, n)
    return out


def sample_rows(cfg: Config) -> tuple[np.ndarray, np.ndarray]:
    """Seeded row samples: centroid rows [nlist] and codeword rows [M][Ks] (reading R3)."""
    cent = _rng(cfg.cfg_id, STREAM_CENT).choice(cfg.N, size=cfg.nlist, replace=False)
    rng = _rng(cfg.cfg_id, STREAM_CODE)
    code = np.stack([rng.choice(cfg.N, size=cfg.Ks, replace=False) for _ in range(cfg.M)])
    return cent.astype(np.int32), code.astype(np.int32).reshape(cfg.M, cfg.Ks)


@dataclass
class Inputs:
    cfg: Config
    db: np.ndarray              # int8 [N][D]
    queries: np.ndarray         # int8 [Q][D]
    centroid_rows: np.ndarray   # int32 [nlist]
    codeword_rows: np.ndarray   # int32 [M][Ks]


@lru_cache(maxsize=4)
def generate(cfg: Config) -> Inputs:
    db = gen_vectors(cfg, STREAM_DB, cfg.N)
    q = gen_vectors(cfg, STREAM_Q, cfg.Q)
    cent, code = sample_rows(cfg)
    return Inputs(cfg, db, q, cent, code)


def rank_queries(cfg: Config, rank: int) -> np.ndarray:
    """The query batch of rank `rank` of a multi-GPU (replica) run: rank 0 gets the config's own
    queries, rank r > 0 an independent draw from the same mixture (stream 100 + r)."""
    if rank == 0:
        return generate(cfg).queries
    return gen_vectors(cfg, STREAM_Q_RANK + rank, cfg.Q)


def gen_float_vectors(cfg: Config, stream: int, n: int) -> np.ndarray:
    """n float32 rows of the config's mixture (the same draws as gen_vectors, before int8)."""
    mix = mixture(cfg.gen, cfg.D, cfg.cfg_id)
    out = np.empty((n, cfg.D), dtype=np.float32)

    def fill(c, lo, hi):
        out[lo:hi] = _float_rows(mix, _rng(cfg.cfg_id, stream, c), hi - lo)
    _chunked(fill, n)
    return out


@dataclass
class FloatInputs:
    cfg: Config
    db: np.ndarray              # float32 [N][D]
    queries: np.ndarray         # float32 [Q][D]
    v_max: float                # max |coordinate| over db and queries (the public fixed-point scale input)
    centroid_rows: np.ndarray
    codeword_rows: np.ndarray


@lru_cache(maxsize=2)
def generate_float(cfg: Config) -> FloatInputs:
    """Real-valued inputs for the 16-bit fixed-point variant (NEXT-1)."""
    db = gen_float_vectors(cfg, STREAM_DB, cfg.N)
    q = gen_float_vectors(cfg, STREAM_Q, cfg.Q)
    v_max = float(max(np.abs(db).max(), np.abs(q).max()))
    cent, code = sample_rows(cfg)
    return FloatInputs(cfg, db, q, v_max, cent, code)


def rank_float_queries(cfg: Config, rank: int) -> np.ndarray:
    """Float32 counterpart of rank_queries (NEXT-1 replicas): rank 0 the config's own float queries,
    rank r > 0 an independent draw (stream 100 + r)."""
    if rank == 0:
        return generate_float(cfg).queries
    return gen_float_vectors(cfg, STREAM_Q_RANK + rank, cfg.Q)
