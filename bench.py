#!/usr/bin/env python
"""bench.py — seconds per boosting round (and histogram GB/s vs HBM peak) of the B200 hot path
of "Out-of-Core GPU Gradient Boosting" (arXiv 2005.09148), BASELINE.json config 2:
1M rows x 500 features make_classification-style, 256 bins, depth 8, in-core, binary:logistic.

A step = one boosting round through the library's public API, exactly the north_star's calls:
  update margin with tree t-1 (Eq. 1) -> logistic gradients (Eq. 5) -> sample(NONE, f = 1)
  -> build_tree(depth 8, lambda 1, gamma 0)   (histograms, evaluation, partition, leaves)
Timing: W untimed warm-up rounds, then K rounds between CUDA events on the stream the library
launches on (torch's current stream is handed to the library), barrier + synchronize on both
sides, max over ranks.  Inputs (512 MB of ELLPACK) are larger than L2 (126 MB).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (row-sharded, weak scaling: 1M rows/GPU)

--impl reference times the CPU oracle (oracle/, as it stands) on a bounded sample of the same
workload and extrapolates to the config (it is the deliberately slow reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ROWS, N_FEAT, MAX_BIN, DEPTH = 1_000_000, 500, 256, 8
LAMBDA, GAMMA, MCW, ETA, QBITS = 1.0, 0.0, 1.0, 0.1, 16
METRIC = "sec/boosting round"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=N_ROWS, help="rows per GPU (config 2: 1M)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-link", action="store_true", help="skip the short out-of-core link leg")
    ap.add_argument("--nccl1", action="store_true",
                    help="N=1: run the sharded code path (NCCL exchanges) on a 1-rank communicator")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no JSON line)")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="2: 1M x 500 in-core f=1 (the driver's bench); 3: 20M x 500 out-of-core, "
                         "32 MiB pinned pages, MVS f=0.1")
    ap.add_argument("--rows3", type=int, default=20_000_000, help="config 3 rows")
    ap.add_argument("--stream-f1", action="store_true",
                    help="config 3 without sampling: Alg. 6 streamed build (one page pass per level)")
    ap.add_argument("--rows4", type=int, default=100_000_000, help="config 4 training rows")
    ap.add_argument("--rows5", type=int, default=400_000_000, help="config 5 global rows (sharded)")
    ap.add_argument("--strong-rows", type=int, default=0,
                    help="strong scaling: a fixed global row count sharded over the ranks (e.g. 100M)")
    ap.add_argument("--rounds4", type=int, default=50, help="config 4 boosting rounds per setting")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_GBps", "hbm"):
            if k in d:
                return float(d[k]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def pipe_roofline(row_features, hist_ms, clocks):
    """Shared-atomic pipe roofline of k_hist: algorithmic warp-wide ATOMS (2 per symbol / 32 lanes)
    per second against 1 per clock per SM at the SM clock measured during the timed region."""
    import torch

    n_sms = torch.cuda.get_device_properties(0).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    atoms = 2.0 * row_features / 32.0
    achieved = atoms / (hist_ms * 1e-3) / 1e9
    peak = n_sms * mhz * 1e6 / 1e9
    return {"bound": "shared-atomic pipe", "kernel": "k_hist", "achieved": achieved, "peak": peak,
            "unit": "G warp-ATOMS/s", "frac": achieved / peak, "ceiling_frac": 32.0 / 37.0,
            "sm_mhz": mhz, "sms": n_sms}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        self.path = f"/tmp/oocgb_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def hist_rows(nodes: np.ndarray):
    """(rows of built nodes summed over levels, number of built nodes) of one tree."""
    D = int(np.log2(len(nodes) + 1)) - 1
    rows, built = 0, 0
    for v in range((1 << D) - 1):
        if v == 0:
            rows += int(nodes["n_rows"][0])
            built += 1
            continue
        p = (v - 1) // 2
        if nodes["feature"][p] < 0 or v != 2 * p + 1:
            continue
        rows += min(int(nodes["n_rows"][v]), int(nodes["n_rows"][v + 1]))
        built += 1
    return rows, built


def hist_algorithmic_bytes(nodes: np.ndarray, m: int) -> float:
    """per built node, 1 B per (row, feature) symbol + 8 B (q_g, q_h int32)
    + 4 B row index per row, + the node's int64 histogram (m x 256 x 16 B) written.  Built nodes:
    the root, then the child with fewer rows of every split (ties: left), levels 0..D-1."""
    rows, built = hist_rows(nodes)
    return rows * (m + 8 + 4) + built * m * 256 * 16.0


def part_algorithmic_bytes(nodes: np.ndarray) -> float:
    """DESIGN.md §5 partition: per row of a split node and level, 4 B (row id) + 1 B (the split
    feature's symbol) + 8 B (q) read and 12 B written."""
    D = int(np.log2(len(nodes) + 1)) - 1
    rows = 0
    for v in range((1 << D) - 1):
        if nodes["feature"][v] >= 0:
            rows += int(nodes["n_rows"][v])
    return rows * 25.0


def measured_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per k_hist launch from the committed ncu
    --set full capture (profiles/k_hist_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "k_hist_traffic.json")) as f:
            return float(json.load(f)["traffic_bytes_per_launch"])
    except Exception:
        return None


def launches_per_round(D: int, world: int = 1) -> int:
    # update_margin 1 + logistic 1 + sample(NONE): absmax2, quantise (one rank; with W > 1 also
    # sstate_init, sstate_globalise around the all-reduces)
    # build_tree: init 1 + per level (k_hist, k_eval or k_eval_blk, k_eval_narrow, k_finalize,
    # k_part_fused) 5, at level 0 of an f = 1 build only the root's own list (4) (matches the ncu
    # launch list: 44 per depth-8 round at W = 1); W > 1 adds k_reduce_partials, k_part_counts and
    # k_part_plan per level
    return (4 if world == 1 else 6) + 1 + (5 if world == 1 else 8) * D - (1 if D > 0 else 0)


def make_data(rows, rank):
    import synth
    X, y = synth.fast_classification(rows, N_FEAT, seed=1000 + rank)
    return X, y


GEN_CHUNK = 1 << 21  # rows per generated chunk (global chunk grid: the data set is the same for every W)


def shard_chunks(n_global, rank, world, chunk=GEN_CHUNK):
    """This rank's rows [row0, row0 + n) (dist.shard_rows) as pieces of the GLOBAL generation grid:
    (global chunk start, chunk rows, slice begin, slice end) -- a chunk is generated whole and
    sliced, so the union of the ranks' rows is one data set whatever the world size."""
    from paper_2005_09148_b200.dist import shard_rows
    row0, n = shard_rows(n_global, rank, world)
    out = []
    r = row0
    while r < row0 + n:
        c0 = (r // chunk) * chunk
        cn = min(chunk, n_global - c0)
        b, e = r - c0, min(cn, row0 + n - c0)
        out.append((c0, cn, b, e))
        r = c0 + e
    return row0, n, out


def load_shard(ctx, n_global, rank, world, seed=5, device="cuda"):
    """Multi-GPU data path (config 2 weak scaling, config 5, strong scaling): every rank generates
    its own rows on its GPU (synth.torch_classification_chunk, never on the host) and streams
    them through the library's two-pass quantise (oocgb_sketch_push, the sketch all-gather in
    oocgb_cuts_finalize, oocgb_pages_push).  Returns (data, labels on the device, row0, n)."""
    import torch
    import synth
    row0, n, pieces = shard_chunks(n_global, rank, world)
    d = ctx.sketch_begin(N_FEAT, MAX_BIN, n_global, seed=2)
    for c0, cn, b, e in pieces:
        X, _ = synth.torch_classification_chunk(c0, cn, N_FEAT, seed=seed, device=device)
        d.sketch_push(X[b:e].contiguous(), c0 + b)
        del X
    d.cuts_finalize()
    ys = []
    for c0, cn, b, e in pieces:
        X, y = synth.torch_classification_chunk(c0, cn, N_FEAT, seed=seed, device=device)
        d.pages_push(X[b:e].contiguous(), c0 + b)
        ys.append(y[b:e])
        del X
    labels = torch.cat(ys) if ys else torch.zeros(0, device=device)
    return d, labels.contiguous(), row0, n


def _oracle_config2():
    """The oracle's setup of config 2 (1M x 500, bench.py's rank-0 data): cuts + bins (untimed)."""
    import oracle
    X, y = make_data(N_ROWS, 0)
    cv, cp = oracle.cuts(X, MAX_BIN)
    B = oracle.bins(X, cv, cp)
    return B, cv, cp, y


def _oracle_rounds(B, cv, cp, y, n_rounds, n_warm=0):
    """Boosting rounds of the oracle exactly as the product runs them (predict(t-1) -> logistic
    gradients -> sample(NONE) -> fixed point -> BuildTree at depth 8); sec/round of the timed ones."""
    import oracle
    margin = np.zeros(len(y), np.float32)
    prev = None
    ts = []
    for r in range(n_warm + n_rounds):
        t0 = time.perf_counter()
        prev, margin, _ = oracle.boosting_round(B, N_FEAT, cv, cp, margin, y, max_depth=DEPTH, lam=LAMBDA,
                                                gamma=GAMMA, mcw=MCW, eta=ETA, quant_bits=QBITS,
                                                prev_tree=prev, round_=r)
        if r >= n_warm:
            ts.append(time.perf_counter() - t0)
    return ts


def cpu_baseline_leg(rounds=2):
    """Oracle (as it stands, single thread) on the FULL config-2 workload: `rounds` boosting rounds
    on 1M x 500 at depth 8 (no extrapolation; about 20 s per round); setup (cuts, bins) untimed."""
    B, cv, cp, y = _oracle_config2()
    ts = _oracle_rounds(B, cv, cp, y, rounds)
    return {"value": statistics.mean(ts), "unit": "s", "cores": 1, "kind": "oracle",
            "sample": f"{rounds} full rounds of config 2 (1M x 500, depth 8), mean sec/round, no extrapolation; "
                      f"single thread, host {os.cpu_count()} cores",
            "rounds_s": ts}


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle as it stands (there is no reference code),
    on bench.py's own config-2 workload at full size: W untimed + K timed boosting rounds."""
    if rank != 0:
        return
    B, cv, cp, y = _oracle_config2()
    ts = _oracle_rounds(B, cv, cp, y, args.steps, args.warmup)
    v = sum(ts) / len(ts)
    sample = (f"each step = 1 full boosting round of config 2 (1M x 500, depth 8, f = 1) by the oracle; "
              f"single thread, host {os.cpu_count()} cores")
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64 fixed-point histograms (quant_bits 16), f64 gains", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "config 2: 1M x 500 make_classification, 256 bins, depth 8, in-core, f=1",
                       "rows_per_gpu": N_ROWS, "n_features": N_FEAT, "max_bin": MAX_BIN, "max_depth": DEPTH},
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_config3(args, rank, world, local):
    line = config3_measure(args, rank, world, local, args.rows3, args.steps, args.warmup)
    if rank == 0:
        print(json.dumps(line), flush=True)


def pinned_h2d_peak(local, gib=1, reps=5):
    """Measured host-link peak: pinned host -> device cudaMemcpyAsync of `gib` GiB, best of `reps`
    (CUDA events), one GPU (SURVEY §8(d) link roofline)."""
    import torch
    nb = gib << 30
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    dv = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{local}")
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dv.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del h, dv
    return nb / (best * 1e-3) / 1e9


def config3_measure(args, rank, world, local, n, steps, warmup):
    """Config 3 (BASELINE.json configs[2]): 20M x 500 streamed as 32 MiB ELLPACK pages from pinned
    host memory, gradient-based (MVS) sampling f = 0.1, depth 8.  Per round: predict(tree t-1)
    streams every page (Eq. 1), logistic gradients, sample(MVS) + Compact gathers the selected
    rows zero-copy from the pinned pages (Alg. 7), build_tree on the compacted device page.  Link busy = H2D copy time / round
    time; link GB/s = bytes copied / copy time (CUDA events on the copy stream)."""
    import torch
    import paper_2005_09148_b200 as ob
    import synth
    m = N_FEAT
    torch.cuda.set_device(local)
    link_peak = pinned_h2d_peak(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = ob.Context(local, rank, world, None, stream=stream.cuda_stream)
    chunk = 1 << 20
    d = ctx.sketch_begin(m, MAX_BIN, n, page_bytes=32 << 20, placement=ob.PLACE_PINNED_HOST, seed=2)
    t0 = time.perf_counter()
    for r0 in range(0, n, chunk):
        X, _ = synth.torch_classification_chunk(r0, min(chunk, n - r0), m, seed=3)
        d.sketch_push(X, r0)
    d.cuts_finalize()
    ys = []
    for r0 in range(0, n, chunk):
        X, y = synth.torch_classification_chunk(r0, min(chunk, n - r0), m, seed=3)
        d.pages_push(X, r0)
        ys.append(y)
    del X
    labels = torch.cat(ys)
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t0
    info = d.info()
    if args.stream_f1:
        d.set_streaming(True)
    margin = torch.zeros(n, dtype=torch.float32, device="cuda")
    tree = None
    sel = []

    def one_round(prev, r):
        if prev is not None:
            d.predict([prev], margin)     # streams all pages
            prev.close()
        d.set_logistic_gradients(margin, labels)
        if args.stream_f1:
            si = d.sample(ob.SAMPLE_NONE, 1.0, round=r, quant_bits=QBITS)
        else:
            si = d.sample(ob.SAMPLE_MVS, 0.1, 1.0, seed=1, round=r, quant_bits=QBITS)  # + Compact
        sel.append(si["n_selected_global"])
        return d.build_tree(DEPTH, LAMBDA, GAMMA, MCW, ETA)

    r = 0
    ctx.set_profiling(True)  # before the warm-up: the timed rounds replay an already-captured graph
    for _ in range(warmup):
        tree = one_round(tree, r)
        r += 1
    torch.cuda.synchronize()
    ctx.get_timings()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    e0.record(stream)
    for _ in range(steps):
        tree = one_round(tree, r)
        r += 1
    e1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / steps
    tm = ctx.get_timings()
    page_bytes_per_pass = n * info["row_stride"]
    # predict streams every page; Compact gathers only the selected rows (zero-copy, NEXT #2);
    # the Alg. 6 streamed build makes one more full pass per level plus the final leaf pass
    if args.stream_f1:
        copied = page_bytes_per_pass * (1 + DEPTH + 1)
    else:
        copied = page_bytes_per_pass + int(statistics.mean(sel[-steps:])) * info["row_stride"]
    h2d_ms = tm["h2d_ms"] / steps
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 symbols, int32/int64 fixed-point sums, f64 gains",
        "data": "synthetic (make_classification-style, generated on the GPU per chunk, seeded)",
        "config": {"workload": ("config 3 variant: 20M x 500 out-of-core, 32 MiB pinned-host pages, f=1, Alg. 6 "
                                "streamed build (one page pass per level)") if args.stream_f1 else
                               "config 3: 20M x 500 out-of-core, 32 MiB pinned-host ELLPACK pages, MVS f=0.1, depth 8",
                   "rows": n, "n_features": m, "n_pages": info["n_pages"], "rows_per_page": info["rows_per_page"],
                   "max_depth": DEPTH, "sample": "none" if args.stream_f1 else "MVS", "ratio": 1.0 if args.stream_f1 else 0.1},
        "link": {"bytes_per_round": copied, "h2d_ms_per_round": h2d_ms, "peak_gbps": link_peak,
                 "busy_frac_of_peak": copied / (ms * 1e-3) / 1e9 / link_peak,
                 "gbps_while_copying": copied / (h2d_ms * 1e-3) / 1e9 if h2d_ms > 0 else None,
                 "busy_frac": h2d_ms / ms, "effective_gbps": copied / (ms * 1e-3) / 1e9},
        "phases_ms_per_round": {k: v / steps for k, v in tm.items() if k.endswith("_ms")},
        "selected_rows_per_round": sel[-steps:],
        "prep_s": prep_s, "clocks": ck,
    }
    if tree is not None:
        tree.close()
    d.close()
    ctx.close()
    return line


def run_config4(args, rank, world, local):
    """Config 4 (BASELINE.json configs[3]): 100M x 500 in-core (51.2 GB of ELLPACK in HBM), 5M
    held-out rows (P:L460-461's 0.95/0.05 split analogue).  For f = 1 and for uniform (SGB), MVS
    and GOSS sampling at f in {0.1, 0.3, 0.5}: `rounds4` boosting rounds (depth 8, eta 0.1) from
    margin 0, then the held-out AUC (sklearn.metrics.roc_auc_score on the binned predict) and the
    median sec/round.  The paper's claim: MVS keeps accuracy at rates as low as 10% (P:L242-243,
    Fig. 1, Table 2)."""
    import torch
    from sklearn.metrics import roc_auc_score
    import paper_2005_09148_b200 as ob
    import synth
    n, m, n_eval = args.rows4, N_FEAT, 5_000_000
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = ob.Context(local, rank, world, None, stream=stream.cuda_stream)
    chunk = 1 << 21
    t0 = time.perf_counter()
    d = ctx.sketch_begin(m, MAX_BIN, n, seed=2)
    for r0 in range(0, n, chunk):
        X, _ = synth.torch_classification_chunk(r0, min(chunk, n - r0), m, seed=4)
        d.sketch_push(X, r0)
    d.cuts_finalize()
    ys = []
    for r0 in range(0, n, chunk):
        X, y = synth.torch_classification_chunk(r0, min(chunk, n - r0), m, seed=4)
        d.pages_push(X, r0)
        ys.append(y)
    labels = torch.cat(ys)
    del ys
    Xe, ye = synth.torch_classification_chunk(n, n_eval, m, seed=4)  # held-out rows n .. n + 5M
    de = d.quantise_like(Xe)
    del Xe, X
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t0
    settings = [("none", 1.0)] + [(mode, f) for mode in ("uniform", "mvs", "goss") for f in (0.1, 0.3, 0.5)]
    results = []
    for mode, f in settings:
        margin = torch.zeros(n, dtype=torch.float32, device="cuda")
        em = torch.zeros(n_eval, dtype=torch.float32, device="cuda")
        trees, times = [], []
        for r in range(args.rounds4):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            if trees:
                d.predict([trees[-1]], margin)   # every row gets the new tree (R18)
            d.set_logistic_gradients(margin, labels)
            if mode == "none":
                d.sample(ob.SAMPLE_NONE, 1.0, round=r, quant_bits=QBITS, want_info=False)
            elif mode == "uniform":
                d.sample(ob.SAMPLE_UNIFORM, f, seed=1, round=r, quant_bits=QBITS)
            elif mode == "mvs":
                d.sample(ob.SAMPLE_MVS, f, 1.0, seed=1, round=r, quant_bits=QBITS)
            else:  # GOSS with a = b = f / 2
                d.sample_goss(f / 2, f / 2, seed=1, round=r, quant_bits=QBITS)
            t = d.build_tree(DEPTH, LAMBDA, GAMMA, MCW, ETA)
            ev1.record(stream)
            torch.cuda.synchronize()
            times.append(ev0.elapsed_time(ev1))
            trees.append(t)
        de.predict(trees, em)
        auc = roc_auc_score(ye.cpu().numpy(), em.cpu().numpy())
        for t in trees:
            t.close()
        results.append({"mode": mode, "f": f, "auc": auc, "ms_per_round_median": statistics.median(times[1:]),
                        "rounds": args.rounds4})
        print(json.dumps(results[-1]), file=sys.stderr, flush=True)
    base = results[0]["auc"]
    for r_ in results:
        r_["auc_rel_diff_vs_f1"] = (r_["auc"] - base) / base
    line = {"config": {"workload": "config 4: 100M x 500 in-core (51.2 GB ELLPACK), 5M held-out rows, depth 8, "
                                   f"eta 0.1, {args.rounds4} rounds; GOSS a = b = f/2",
                       "rows": n, "held_out": n_eval, "n_features": m},
            "data": "synthetic (make_classification-style, generated on the GPU per chunk, seeded)",
            "prep_s": prep_s, "results": results}
    if rank == 0:
        print(json.dumps(line), flush=True)
    de.close()
    d.close()
    ctx.close()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.config == 4 and args.impl == "ours":
        run_config4(args, rank, world, local)
        return
    if args.config == 3 and args.impl == "ours":
        run_config3(args, rank, world, local)
        return
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import paper_2005_09148_b200 as ob
    from paper_2005_09148_b200 import build as obuild
    if rank == 0:
        obuild.build()
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
    torch.cuda.set_device(local)
    # one dedicated (non-default) stream shared by torch and the library: the library enqueues
    # on it, the CUDA events below are recorded on it, and the build_tree graph is captured on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nid = None
    if world > 1:
        import torch.distributed as tdist
        idl = [ob.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(idl, src=0)
        nid = idl[0]
    elif args.nccl1:  # the multi-GPU code path (every exchange through NCCL) on a 1-rank communicator
        nid = ob.nccl_unique_id()
    ctx = ob.Context(local, rank, world, nid, stream=stream.cuda_stream)
    if args.config == 5 or args.strong_rows:
        # config 5 (400M x 500 sharded) or strong scaling (a fixed global row count)
        n_global = args.strong_rows or args.rows5
        d, yd, _, rows = load_shard(ctx, n_global, rank, world)
        y = yd.cpu().numpy()
        workload = (f"config 5: {n_global} x {N_FEAT} row-sharded over {world} GPU(s)" if args.config == 5 else
                    f"strong scaling: {n_global} x {N_FEAT} row-sharded over {world} GPU(s)")
        scaling = "strong"
        rows_global = n_global
    elif world > 1:
        # config 2 weak scaling: 1M rows per GPU, generated on each rank's GPU
        d, yd, _, rows = load_shard(ctx, args.rows * world, rank, world)
        y = yd.cpu().numpy()
        workload = "config 2 weak scaling: 1M x 500 per GPU, 256 bins, depth 8, in-core, f=1"
        scaling = "weak"
        rows_global = args.rows * world
    else:
        rows = args.rows
        X, y = make_data(rows, rank)
        Xd = torch.from_numpy(X).cuda()
        yd = torch.from_numpy(y).cuda()
        d = ctx.quantise(Xd, MAX_BIN, row0_global=rank * rows, n_rows_global=world * rows)
        del Xd
        workload = "config 2: 1M x 500 make_classification, 256 bins, depth 8, in-core, f=1"
        scaling = "weak"
        rows_global = rows
    torch.cuda.synchronize()
    margin = torch.zeros(rows, dtype=torch.float32, device="cuda")

    def round_device(prev_tree, r, close_prev=True, via_predict=False):
        if prev_tree is not None:
            if via_predict:  # not the latest tree: binned traversal (same margins, R18)
                d.predict([prev_tree], margin)
            else:
                d.update_margin(prev_tree, margin)
            if close_prev:
                prev_tree.close()
        d.set_logistic_gradients(margin, yd)
        d.sample(ob.SAMPLE_NONE, 1.0, round=r, quant_bits=QBITS, want_info=False)
        return d.build_tree(DEPTH, LAMBDA, GAMMA, MCW, ETA)

    tree = None
    r = 0
    for _ in range(args.warmup):
        tree = round_device(tree, r)
        r += 1
    if args.profile_only:
        for _ in range(args.steps):
            tree = round_device(tree, r)
            r += 1
        torch.cuda.synchronize()
        return

    def timed_loop(replay=False):
        nonlocal tree, r
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        exported = []
        for i in range(args.steps):
            # the pending tree of the first round stays alive so region B can replay region A
            tree = round_device(tree, r, close_prev=i > 0, via_predict=replay and i == 0)
            exported.append(tree.export())   # the tree a user gets back (C call + copy)
            r += 1
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            ms = float(t[0])
        return ms, exported

    # timed region A (the reported value): the plain captured graph, no instrumentation
    tree_shape_state = (margin.clone(), r, tree)  # rounds differ (tree shapes evolve): B replays A's rounds
    clocks = ClockSampler(local)
    ms, _ = timed_loop()
    ck = clocks.stop()
    ms_step = ms / args.steps
    # timed region B (phase attribution + the k_hist roofline): the same rounds (margin and round
    # index restored) replaying the graph variant with CUDA event nodes around each phase; the
    # event nodes cost time per round, which is why region A is the reported value
    ctx.set_profiling(True)
    tree = round_device(tree, r)  # captures the instrumented graph variant
    torch.cuda.synchronize()
    ctx.get_timings()  # drain and reset
    tree.close()
    margin.copy_(tree_shape_state[0])
    r, tree = tree_shape_state[1], tree_shape_state[2]
    ms_prof, exported = timed_loop(replay=True)
    tree_shape_state[2].close()
    tm = ctx.get_timings()
    ctx.set_profiling(False)
    # per GPU: the exported tree counts global rows; each rank built 1/W of them (row-sharded)
    hist_bytes = sum(hist_algorithmic_bytes(nd, N_FEAT) for nd in exported) / world
    part_bytes = sum(part_algorithmic_bytes(nd) for nd in exported) / world
    hist_rowfeat = sum(hist_rows(nd)[0] * N_FEAT for nd in exported) / world
    hist_ms = tm["hist_ms"]
    n_hist = max(1, int(tm["hist_launches"]))
    achieved = (hist_bytes / n_hist) / (hist_ms / n_hist * 1e-3) / 1e9  # GB/s per launch average
    peak, peak_src = hbm_peak()

    # ---- e2e: the same round through the public API with HOST buffers (pinned), H2D/D2H inside
    m_host = torch.zeros(rows, dtype=torch.float32).pin_memory()
    y_host = torch.from_numpy(y).pin_memory()
    e2e_tree = None
    rr = r

    def round_host(prev_tree, r_):
        if prev_tree is not None:
            d.update_margin(prev_tree, m_host)      # H2D + D2H of the margin
            prev_tree.close()
        d.set_logistic_gradients(m_host, y_host)    # H2D of margin + labels
        d.sample(ob.SAMPLE_NONE, 1.0, round=r_, quant_bits=QBITS, want_info=False)
        t = d.build_tree(DEPTH, LAMBDA, GAMMA, MCW, ETA)
        t.export()                                  # D2H of the tree
        return t

    for _ in range(max(2, args.warmup)):
        e2e_tree = round_host(e2e_tree, rr)
        rr += 1
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_tree = round_host(e2e_tree, rr)
        rr += 1
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    e2e_wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    e2e_diag = ctx.get_timings()
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    n_nodes = (1 << (DEPTH + 1)) - 1
    h2d = rows * 4 * 3
    d2h = rows * 4 + n_nodes * 48

    d.close()
    # short out-of-core leg (config 3's path at 2M rows: 31 pinned 32 MiB pages, MVS f = 0.1):
    # link GB/s and busy fraction against the measured pinned H2D peak
    link = None
    if world == 1 and not args.no_link:
        lk = config3_measure(args, rank, world, local, 2_000_000, 3, 1)
        link = dict(lk["link"], rows=2_000_000, n_pages=lk["config"]["n_pages"], ms_per_round=lk["ms_per_step"],
                    phases_ms_per_round=lk["phases_ms_per_round"],
                    workload="config 3 path at 2M rows: 32 MiB pinned-host pages, MVS f=0.1, depth 8",
                    clocks=lk.get("clocks"))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg()
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": scaling,
            "vs_baseline": None, "dtype": "u8 symbols, int32/int64 fixed-point sums, f64 gains",
            "data": "synthetic (make_classification-style, seeded; W > 1: generated on each rank's GPU)",
            "config": {"workload": workload,
                       "rows_per_gpu": rows, "rows_global": rows_global, "n_features": N_FEAT,
                       "max_bin": MAX_BIN, "max_depth": DEPTH, "quant_bits": QBITS,
                       "parallelism": f"row-sharded dp{world}" + (" (NCCL 1-rank exchange path)" if args.nccl1 and world == 1 else ""),
                       "l2": f"inputs larger than L2 ({rows * 512 / 1e6:.0f} MB ELLPACK per GPU vs 126 MB L2), no flush"},
            "gpu_launches": launches_per_round(DEPTH, 2 if (world > 1 or args.nccl1) else 1) * args.steps,
            "rows_rounds_per_s": rows_global / (ms_step / 1e3),
            "histogram": {"row_features_per_s": hist_rowfeat / (hist_ms * 1e-3), "ms_per_round": hist_ms / args.steps,
                          "launches": n_hist, "algorithmic_bytes_per_round": hist_bytes / args.steps},
            "phases_ms_per_round": {k: v / args.steps for k, v in tm.items() if k.endswith("_ms")},
            "partition": {"ms_per_round": tm["partition_ms"] / args.steps,
                          "algorithmic_bytes_per_round": part_bytes / args.steps,
                          "GB_per_s": part_bytes / (tm["partition_ms"] * 1e-3) / 1e9,
                          "frac_of_hbm": part_bytes / (tm["partition_ms"] * 1e-3) / 1e9 / peak},
            "profiled_ms_per_step": ms_prof / args.steps,  # region B (event nodes in the graph)
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": measured_traffic(), "kernel": "k_hist",
                         "algorithmic_bytes_per_launch": hist_bytes / n_hist,
                         "peak_source": peak_src},
            # k_hist's binding on-chip resource: 2 shared atomics per symbol at <= 1
            # conflict-free warp-wide ATOMS per clock per SM; the symbol/q loads share the L1 data
            # pipe (4 + 1 wavefronts per 32 ATOMS at the root), so 32/37 of this peak is the ceiling
            "pipe_roofline": pipe_roofline(hist_rowfeat, hist_ms, ck),
            "e2e": {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "wall_ms_per_step": e2e_wall_ms, "graph_captures": e2e_diag.get("graph_captures")},
            "graph_captures_timed": tm.get("graph_captures"),
            "clocks": ck,
        }
        if link:
            line["link"] = link
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    for t in (tree, e2e_tree):
        if t is not None:
            t.close()
    ctx.close()
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
