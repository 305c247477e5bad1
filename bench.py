#!/usr/bin/env python
"""bench.py -- batched fixed-shape IVF-PQ query path (V3DB, arxiv 2603.03065) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--trace on|off]
  python bench.py --impl reference ...      (the CPU oracle on the host cores)
  python bench.py --precision fx16 ...      (NEXT-1: the paper's 16-bit fixed point)

One step = one v3db_query_batch over the config's whole query batch (Steps 1-5 of
PAPER.md §4.2, all on the GPU, witness trace on by default), inputs resident in HBM.
Multi-GPU (torchrun): every rank runs its own independent batch against its own snapshot
replica -- weak scaling, no data-path collective.
Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import generate, generate_float, get_config, rank_float_queries, rank_queries  # noqa: E402

METRIC = "queries/sec and scan HBM GB/s (fraction of roofline) at nprobe, k, 1 B200"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c4")
    p.add_argument("--trace", default="on", choices=["on", "off"])
    p.add_argument("--algo", type=int, default=0, help="V3DB_SCAN_* (0 = auto)")
    p.add_argument("--precision", default="int8", choices=["int8", "fx16"],
                   help="int8 (BASELINE.json) or fx16 (the paper's 16-bit fixed point, NEXT-1)")
    p.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


# ------------------------------------------------------------------------------- helpers

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def contraction_peak(kind: str, n: int = 8192, reps: int = 5) -> float:
    """Measured dense peak of the coarse step's contraction on this GPU: int8
    via torch._int_mm (cuBLASLt), fp64 via torch.mm (cuBLAS DGEMM) at n^3, best of `reps`, TOP/s or
    TFLOP/s.  Run after the timed region."""
    import torch
    if kind == "int8":
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
        fn = lambda: torch._int_mm(a, b)  # noqa: E731
    else:
        n = 4096
        a = torch.rand((n, n), dtype=torch.float64, device="cuda")
        b = torch.rand((n, n), dtype=torch.float64, device="cuda")
        fn = lambda: torch.mm(a, b)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        fn()
        e_.record()
        torch.cuda.synchronize()
        best = min(best, s_.elapsed_time(e_))
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def code_bytes_per_slot(M: int, Ks: int) -> int:
    """ceil(M * log2(Ks) / 8): the information content of one PQ code."""
    return math.ceil(M * max(1, math.ceil(math.log2(Ks))) / 8) if Ks > 1 else 0


def algorithmic_scan_bytes(cfg, lists: np.ndarray, counts: np.ndarray, trace: bool, fx: bool = False) -> dict:
    """Bytes the scan (Steps 3-5) must move per batch: per query the query
    vector, the codes of the VALID slots of its probed lists, the probed lists' counts, the
    top-k output, and with the trace the masked distance of every probed slot plus the probe
    list/distance -- no credit for cross-query reuse.  fx: int32 coordinates, int64 distances."""
    valid = int(counts[lists].sum())
    Q = lists.shape[0]
    cb = code_bytes_per_slot(cfg.M, cfg.Ks)
    qb, w = (4, 8) if fx else (1, 4)
    per_batch = Q * cfg.D * qb + valid * cb + Q * 4 * cfg.nprobe + Q * (4 + w) * cfg.k
    padded = Q * cfg.D * qb + Q * cfg.nprobe * cfg.L * cb + Q * 4 * cfg.nprobe + Q * (4 + w) * cfg.k
    if trace:
        tr = Q * (w * cfg.nprobe * cfg.L + (4 + w) * cfg.nprobe)
        per_batch += tr
        padded += tr
    return {"valid": per_batch, "padded": padded, "valid_slots": valid, "topk_out": Q * (4 + w) * cfg.k}


def resolved_algo(v3db, snap, algo: int, fx: bool) -> str:
    """The scan kernel V3DB_SCAN_AUTO (or the explicit algo) runs for this snapshot."""
    if fx:   # the fixed-point list-major scan where the snapshot holds its limb planes
        return "fx16_lm" if snap.dim % 16 == 0 and snap.dim <= 256 and snap.nlist <= 32768 else "fx16"
    names = {1: "generic", 2: "rotated", 3: "list_major"}
    if algo:
        return names[algo]
    return "list_major" if snap.dim % 16 == 0 else "rotated"


def algo_used_pre(algo: int, snap) -> str:
    return {1: "generic", 2: "rotated", 3: "list_major"}.get(algo) or ("list_major" if snap.dim % 16 == 0 else "rotated")


def main_kernel_name(algo: str) -> str:
    return {"list_major": "lm_kernel (Steps 3-4 + trace, tcgen05 int8 tiles per list)",
            "rotated": "scan_rot_kernel (Steps 3-5)", "generic": "scan_lut (Steps 3-5)",
            "fx16": "scan_fx_kernel (Steps 3-5)",
            "fx16_lm": "lm_fx_kernel (Steps 3-4 + trace, tcgen05 int8-limb tiles per list, int64 D)"}[algo]


def roofline_key(name: str, fx: bool, algo: str, trace: bool) -> str:
    return name + ("_fx16" if fx else "") + ("" if algo in ("list_major", "fx16", "fx16_lm") else "_" + algo) + \
        ("" if trace else "_traceoff")


def l2_label(cfg, algo: str, codes_mb: float) -> str:
    """What the 256 MiB write between timed steps leaves for the next step to fetch from HBM."""
    lm_mb = cfg.nlist * (-(-cfg.L // 128) * 128) * cfg.D / 1e6   # the list-major kernel's xhat
    data_mb = lm_mb if algo == "list_major" else 3 * lm_mb if algo == "fx16_lm" else codes_mb
    what = {"list_major": "xhat", "fx16_lm": "xhat limb planes"}.get(algo, "codes")
    if data_mb > 126:
        return f"flushed between timed steps (256 MiB write); the snapshot's {what} ({data_mb:.0f} MB) exceed L2"
    return (f"flushed between timed steps (256 MiB write); the snapshot's {what} ({data_mb:.0f} MB) fit in L2, "
            f"so within a step they are re-read from L2 after the first touch")


def load_traffic(cfg_name: str):
    """DRAM bytes per scan launch from the committed ncu --set full capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(cfg_name)
    except Exception:
        return None


# ------------------------------------------------------------------------------- CPU oracle

_OS = None
_OQ = None


def _oracle_init(snap, queries):
    global _OS, _OQ
    _OS, _OQ = snap, queries


def _oracle_work(args):
    import oracle
    rows, nprobe, k = args
    oracle.query_batch(_OS, _OQ, nprobe, k, rows=rows)
    return len(rows)


def time_oracle(snap, queries, cfg, seconds: float, workers: int):
    """Time the oracle's query (Steps 1-5, as it stands) on a bounded sample of the batch
    over `workers` processes.  Returns (qps, n_sampled, wall_s)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    import oracle
    t0 = time.perf_counter()
    oracle.query_batch(snap, queries, cfg.nprobe, cfg.k, rows=np.arange(2))
    per_q = (time.perf_counter() - t0) / 2
    n = int(min(cfg.Q, max(workers, round(seconds / max(per_q, 1e-6)))))
    rows = np.arange(n)
    shards = [s for s in np.array_split(rows, workers) if len(s)]
    with ProcessPoolExecutor(len(shards), mp_context=mp.get_context("fork"), initializer=_oracle_init,
                             initargs=(snap, queries)) as ex:
        list(ex.map(_oracle_work, [(shards[0][:1], cfg.nprobe, cfg.k)] * len(shards)))  # warm workers
        t0 = time.perf_counter()
        done = sum(ex.map(_oracle_work, [(s, cfg.nprobe, cfg.k) for s in shards]))
        wall = time.perf_counter() - t0
    return done / wall, done, wall


def oracle_snapshot_from_arrays(arr: dict):
    import oracle
    return oracle.Snapshot(arr["centroids"], arr["codebooks"], arr["ids"], arr["codes"], arr["counts"],
                           arr.get("list_of", np.zeros(0, np.int32)))


# ------------------------------------------------------------------------------- reference arm

def run_reference(args, rank: int, world: int):
    """--impl reference: the oracle (plain numpy, CPU) builds the snapshot and answers a
    bounded sample of the batch per step, on the host cores."""
    if rank != 0:
        return
    import oracle
    cfg = get_config(args.config)
    fx = args.precision == "fx16"
    inp = generate_float(cfg) if fx else generate(cfg)
    workers = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    db, queries = inp.db, inp.queries
    if fx:
        db = oracle.encode_fixed_point(db, inp.v_max)
        queries = oracle.encode_fixed_point(queries, inp.v_max)
    snap = oracle.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    build_s = time.perf_counter() - t0
    per_step = max(2.0, args.cpu_sample_seconds / max(1, args.steps + args.warmup) * workers)
    for _ in range(args.warmup):
        time_oracle(snap, queries, cfg, per_step, workers)
    tot_q, tot_t = 0, 0.0
    for _ in range(args.steps):
        _, n, wall = time_oracle(snap, queries, cfg, per_step, workers)
        tot_q += n
        tot_t += wall
    qps = tot_q / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": cfg.name, "Q": cfg.Q, "N": cfg.N, "D": cfg.D, "nlist": cfg.nlist, "L": cfg.L,
                   "M": cfg.M, "Ks": cfg.Ks, "nprobe": cfg.nprobe, "k": cfg.k, "trace": args.trace,
                   "precision": args.precision},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": workers, "kind": "oracle",
                         "sample": f"{tot_q} queries of the {cfg.name} batch over {args.steps} steps "
                                   f"(oracle snapshot build {build_s:.1f} s, not timed)"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- our arm

def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    from paper_2603_03065_b200 import dist as pdist
    from paper_2603_03065_b200 import v3db

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pdist.init(world, "nccl", dev)

    def barrier():
        pdist.barrier(world)

    cfg = get_config(args.config)
    trace = args.trace == "on"
    fx = args.precision == "fx16"
    inp = generate_float(cfg) if fx else generate(cfg)

    # Snapshot build (offline index shaping; timed separately, not part of a step).
    if fx:   # NEXT-1: float vectors -> 16-bit fixed point on the GPU (v_max over db and this rank's queries)
        queries = rank_float_queries(cfg, rank)
        v_max = float(max(np.abs(inp.db).max(), np.abs(queries).max()))
        db = v3db.encode_fixed_point(torch.from_numpy(inp.db).to(dev), v_max)
    else:
        queries = rank_queries(cfg, rank)    # replicas: an independent batch per rank (weak scaling)
        db = torch.from_numpy(inp.db).to(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    build = v3db.build_snapshot_fx if fx else v3db.build_snapshot
    snap = build(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    build_s = time.perf_counter() - t0
    del db
    counts = v3db.snapshot_export(snap, v3db.FIELD_COUNTS)

    if fx:
        q = v3db.encode_fixed_point(torch.from_numpy(queries).to(dev), v_max)
        out = v3db.alloc_outputs_fx(snap, cfg.Q, cfg.nprobe, cfg.k, trace=True, device=dev)

        def query(o):
            return v3db.query_batch_fx(snap, q, cfg.nprobe, cfg.k, out=o)
    else:
        q = torch.from_numpy(queries).to(dev)
        out = v3db.alloc_outputs(snap, cfg.Q, cfg.nprobe, cfg.k, trace=True, device=dev)

        def query(o):
            return v3db.query_batch(snap, q, cfg.nprobe, cfg.k, out=o, algo=args.algo)
    if not trace:
        for key in ("trace_cand_dist",):
            out.pop(key)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    v3db.profile_enable(True)
    torch.cuda.cudart().cudaProfilerStart()   # ncu --profile-from-start off sees only the query path
    for _ in range(args.warmup):
        query(out)
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kt = []
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        l0 = v3db.kernel_launches()
        for i in range(args.steps):
            flush.zero_()                                   # L2 flush between timed steps (not timed)
            starts[i].record(stream)
            query(out)
            ends[i].record(stream)
            kt.append(v3db.profile_read(detail=True))       # per-kernel CUDA-event times of this step
        launches = v3db.kernel_launches() - l0
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    tot_ms = pdist.max_over_ranks(float(np.sum(step_ms)), world, dev)

    # the same step with the witness trace off (qps with the trace on and off)
    out_off = {key: v for key, v in out.items() if key != "trace_cand_dist"}
    n_off = max(1, min(args.steps, 5))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_off)]
    query(out_off)
    for a_, b_ in ev:
        flush.zero_()
        a_.record(stream)
        query(out_off)
        b_.record(stream)
    torch.cuda.synchronize()
    off_ms = pdist.max_over_ranks(float(np.mean([a_.elapsed_time(b_) for a_, b_ in ev])), world, dev)
    # the literal-LUT alternative (V3DB_SCAN_ROTATED: per-query Step-3 table + Step-4 lookups), same
    # launch, timed beside the default for the record (int8 only)
    rot = None
    if not fx and algo_used_pre(args.algo, snap) == "list_major":
        try:
            ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
            v3db.query_batch(snap, q, cfg.nprobe, cfg.k, out=out, algo=v3db.SCAN_ROTATED)
            kr = []
            for a_, b_ in ev2:
                flush.zero_()
                a_.record(stream)
                v3db.query_batch(snap, q, cfg.nprobe, cfg.k, out=out, algo=v3db.SCAN_ROTATED)
                b_.record(stream)
                kr.append(v3db.profile_read(detail=True))
            torch.cuda.synchronize()
            rms = float(np.mean([a_.elapsed_time(b_) for a_, b_ in ev2]))
            rot = {"ms_per_step": rms, "value": cfg.Q / (rms / 1e3),
                   "scan_kernel_ms": float(np.mean([t[2] for t in kr])), "kernel": "scan_rot_kernel"}
        except Exception as exc:  # shapes the rotated scan does not support
            rot = {"error": str(exc)[:160]}
    ms_per_step = tot_ms / args.steps
    qps = cfg.Q * world / (ms_per_step / 1e3)
    coarse_ms = float(np.mean([t[0] for t in kt]))
    scan_ms = float(np.mean([t[1] for t in kt]))
    main_ms = float(np.mean([t[2] for t in kt]))      # the scan's main kernel alone
    pro_ms = float(np.mean([t[3] for t in kt]))
    sel_ms = float(np.mean([t[4] for t in kt]))
    algo_used = resolved_algo(v3db, snap, args.algo, fx)

    lists = out["trace_lists"].cpu().numpy()
    ab = algorithmic_scan_bytes(cfg, lists, counts, trace, fx)
    hbm, peak_src = peaks()
    traffic = load_traffic(roofline_key(cfg.name, fx, algo_used, trace))
    # dominant kernel: the scan's main kernel (list-major: Steps 3-4 + trace; query-major: Steps
    # 3-5).  Its algorithmic bytes: SURVEY.md §8(d) per query (no credit for cross-query reuse),
    # less the top-k output the list-major selection kernel writes.
    main_bytes = ab["valid"] - (ab["topk_out"] if algo_used in ("list_major", "fx16_lm") else 0)
    achieved = main_bytes / (main_ms / 1e3) / 1e9
    codes_mb = cfg.nlist * cfg.L * cfg.M / 1e6

    result = {
        "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64" if fx else "int32", "data": "synthetic",
        "config": {"workload": cfg.name, "Q": cfg.Q, "N": cfg.N, "D": cfg.D, "nlist": cfg.nlist, "L": cfg.L,
                   "M": cfg.M, "Ks": cfg.Ks, "nprobe": cfg.nprobe, "k": cfg.k, "trace": args.trace,
                   "precision": args.precision, "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": l2_label(cfg, algo_used, codes_mb),
                   "algo": algo_used, "snapshot_build_s": round(build_s, 3)},
        "ms_per_step_median": float(np.median(step_ms)), "ms_per_step_best": float(np.min(step_ms)),
        "value_trace_off": cfg.Q * world / (off_ms / 1e3),
        "scan_gbs": ab["valid"] / (scan_ms / 1e3) / 1e9,
        "scan_gbs_padded": ab["padded"] / (scan_ms / 1e3) / 1e9,
        "kernel_ms": {"coarse_steps12": coarse_ms, "scan_steps345": scan_ms, "scan_main_kernel": main_ms,
                      "scan_prologue": pro_ms, "scan_select": sel_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": main_kernel_name(algo_used), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": main_bytes,
                     "accounting": "SURVEY.md §8(d): per query its probed lists' valid codes, no credit for "
                                   "cross-query reuse" + (
                                       "; the list-major kernel reads each probed list ONCE per batch for all "
                                       "its queries (DRAM traffic = `traffic`), so frac > 1 is that reuse, "
                                       "see dram_roofline" if algo_used in ("list_major", "fx16_lm") else "")},
        "gpu_launches": int(launches),
    }
    if rot is not None:
        result["rotated_lut_scan"] = rot
    if traffic:
        dram = traffic / (main_ms / 1e3) / 1e9
        result["dram_roofline"] = {"bound": "hbm", "achieved": dram, "peak": hbm, "unit": "GB/s", "frac": dram / hbm,
                                   "bytes_per_launch": traffic, "source": "ncu dram__bytes_read.sum + "
                                   "dram__bytes_write.sum of the same kernel (profiles/ncu_traffic.json)"}

    # End-to-end through the C ABI with HOST buffers (H2D queries, D2H outputs inside).
    if not args.no_e2e and fx:
        # NEXT-1 through v3db_query_batch_fx_host: pinned float32 queries H2D, GPU encoding, Steps
        # 1-5, outputs D2H into pinned host buffers, all inside the C-ABI call.
        qh = torch.from_numpy(queries).pin_memory()
        oh = v3db.alloc_outputs_fx(snap, cfg.Q, cfg.nprobe, cfg.k, trace=trace, device="cpu", pin=True)

        def e2e_step():
            v3db.query_batch_fx_host(snap, qh, v_max, cfg.nprobe, cfg.k, oh)
        e2e_step()
        n_e2e = max(1, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        e2e_s = pdist.max_over_ranks((time.perf_counter() - t0) / n_e2e, world, dev)
        d2h = sum(v.numel() * v.element_size() for v in oh.values())
        result["e2e"] = {"value": cfg.Q * world / e2e_s, "unit": "queries/s",
                         "h2d_bytes_per_step": qh.numel() * 4, "d2h_bytes_per_step": d2h, "steps": n_e2e}
    elif not args.no_e2e:
        qh = torch.from_numpy(queries).pin_memory()
        oh = v3db.alloc_outputs(snap, cfg.Q, cfg.nprobe, cfg.k, trace=trace, device="cpu", pin=True)
        v3db.query_batch_host(snap, qh, cfg.nprobe, cfg.k, oh)
        n_e2e = max(1, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            v3db.query_batch_host(snap, qh, cfg.nprobe, cfg.k, oh)
        e2e_s = pdist.max_over_ranks((time.perf_counter() - t0) / n_e2e, world, dev)
        d2h = sum(v.numel() * 4 for v in oh.values())
        result["e2e"] = {"value": cfg.Q * world / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": qh.numel(),
                         "d2h_bytes_per_step": d2h, "steps": n_e2e}
        if trace:   # the same end-to-end call without the witness trace (top-k + probe lists only)
            oh2 = v3db.alloc_outputs(snap, cfg.Q, cfg.nprobe, cfg.k, trace=False, device="cpu", pin=True)
            v3db.query_batch_host(snap, qh, cfg.nprobe, cfg.k, oh2)
            barrier()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                v3db.query_batch_host(snap, qh, cfg.nprobe, cfg.k, oh2)
            e2 = pdist.max_over_ranks((time.perf_counter() - t0) / n_e2e, world, dev)
            result["e2e_trace_off"] = {"value": cfg.Q * world / e2, "unit": "queries/s",
                                       "h2d_bytes_per_step": qh.numel(),
                                       "d2h_bytes_per_step": sum(v.numel() * 4 for v in oh2.values()), "steps": n_e2e}

    result["clocks"] = clk.summary()

    # the coarse step's contraction against the measured peak of its arithmetic (int8 tensor
    # cores; fp64 for the fixed-point path): 2 Q nlist D ops per batch
    try:
        cpk = contraction_peak("fp64" if fx else "int8")
        cops = 2.0 * cfg.Q * cfg.nlist * cfg.D / (coarse_ms / 1e3) / 1e12
        result["coarse_roofline"] = {
            "bound": "fp64" if fx else "tensor", "achieved": cops, "peak": cpk, "unit": "TOP/s",
            "frac": cops / cpk, "kernel": "coarse (Steps 1-2, fused top-nprobe)",
            "peak_source": "measured now: torch.mm float64 4096^3" if fx else "measured now: torch._int_mm 8192^3"}
    except Exception as exc:  # never fail the bench line on the auxiliary peak
        result["coarse_roofline"] = {"error": str(exc)[:200]}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arr = {"centroids": v3db.snapshot_export(snap, v3db.FIELD_CENTROIDS),
               "codebooks": v3db.snapshot_export(snap, v3db.FIELD_CODEBOOKS),
               "ids": v3db.snapshot_export(snap, v3db.FIELD_IDS),
               "codes": v3db.snapshot_export(snap, v3db.FIELD_CODES), "counts": counts}
        workers = len(os.sched_getaffinity(0))
        oq = inp.queries
        if fx:
            import oracle
            oq = oracle.encode_fixed_point(queries, v_max)
        cq, n, wall = time_oracle(oracle_snapshot_from_arrays(arr), oq, cfg, args.cpu_sample_seconds, workers)
        result["cpu_baseline"] = {"value": cq, "unit": "queries/s", "cores": workers, "kind": "oracle",
                                  "sample": f"{n} of {cfg.Q} {cfg.name} queries, Steps 1-5 on this snapshot's "
                                            f"arrays, {wall:.1f} s wall on {workers} processes"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    snap.free()
    pdist.shutdown(world)


if __name__ == "__main__":
    main()
