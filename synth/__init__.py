"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the V3DB method: it only draws the raw
database/query vectors and the seeded row samples that BASELINE.json's configs
prescribe ("nlist coarse centroids = seeded-sampled database vectors", "Ks
codewords per subspace = seeded-sampled residual subvectors").  The sampled row
indices are passed to both the oracle and the C-ABI, so no RNG is shared across
languages (SURVEY.md §8(c) reading R3).
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .generate import FloatInputs, Inputs, generate, generate_float, rank_float_queries, rank_queries  # noqa: F401
