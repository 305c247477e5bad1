"""V3DB CPU oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, literal CPU implementation of the fixed-shape IVF-PQ semantics of
V3DB (arxiv 2603.03065, §4.1-§4.2).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import it.  It shares no code with the CUDA path
(``paper_2603_03065_b200/``) and never imports it.
"""
from .v3db_oracle import (  # noqa: F401
    D_MAX,
    D_MAX_FX,
    encode_fixed_point,
    Snapshot,
    assign_rebalance,
    build_snapshot,
    dist,
    query,
    query_batch,
    step1_centroid_distances,
    step2_probe_select,
    step3_adc_tables,
    step4_candidate_distances,
    step5_topk,
    witness,
)
