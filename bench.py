#!/usr/bin/env python
"""Benchmark: exact Euclidean 1-NN queries/s over a resident iSAX index, plus
iSAX build Mseries/s, on BASELINE.json configs[1] (100M x 256 z-normalised
random walks, seed 1; 100 queries per step, generated the same way with
seed 2; w=16, 8-bit symbols, leaf capacity 2000).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

Ours: the dataset (fixed total size) is sharded by contiguous series ranges
across ranks (one process per GPU; `--gpus N` without torchrun re-launches
itself under torch.distributed.run). Each rank's index joins the library's
NCCL communicator (tsg_comm_init): per batch the shards' seed best-so-far
distances are min-allreduced inside the query graph and the per-shard
(distance, position) records are all-gathered and merged on the device
(lexicographic minimum = the exact global answer, ties to the lowest
position). `value` = queries/s with queries already in HBM; `e2e` = the same
through the public API with host queries (H2D + result D2H inside the timed
region). Reference arm (`--impl reference`): the unmodified reference
(oracle/_ref, compiled from /root/reference) on the host cores, rank 0 only.

Parity (both arms): BASELINE's 100 queries (rows 0..99 of the seed-2 query
stream) are answered outside the timed region and digested as the reference
CLI's oracle check prints them ("%zu %u %.17g\n": query, position, distance,
tools/main.cpp:193-210); on c2 the digest is compared with
tests/golden/c2_answers.txt (the reference's scan_nn over all 100M series,
oracle/make_c2_golden.py). A mismatch exits nonzero.

Inputs are synthetic (the reference's own seeded generator, BASELINE.json
configs), generated on the device by the library's generator (bit-identical
to the reference generator, see tests/test_gpu_parity.py).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "exact 1-NN queries/s & iSAX build Mseries/s (float32 series), % of HBM roofline"

CONFIGS = {
    # BASELINE.json configs. data: (kind, count, length, seed); queries: (kind, seed, begin) where
    # begin=None means "the next series of the same process" (index count, count+1, ...).
    # c4's count is per GPU (1B over 8 GPUs = 125M each); c5 = c2's data with noisy queries.
    "c1": {"data": ("rw", 1_000_000, 256, 1), "queries": ("rw", 2, 0), "nq": 100},
    "c2": {"data": ("rw", 100_000_000, 256, 1), "queries": ("rw", 2, 0), "nq": 100},
    "c3": {"data": ("c3", 200_000_000, 128, 3), "queries": ("c3", 3, None), "nq": 100},
    "c4": {"data": ("c4", 125_000_000, 96, 4), "queries": ("c4", 4, None), "nq": 100, "per_gpu": True},
    "c5": {"data": ("rw", 100_000_000, 256, 1), "queries": ("c5", 5, 0), "nq": 100},
}


GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_for(name, count):
    """(answers text, meta) of the reference's exhaustive answers for this workload, if committed."""
    if name != "c2" or count != CONFIGS["c2"]["data"][1]:
        return None, None
    path = os.path.join(GOLDEN, "c2_answers.txt")
    if not os.path.exists(path):
        return None, None
    with open(path) as f, open(os.path.join(GOLDEN, "c2_golden.json")) as g:
        return f.read(), json.load(g)


def answers_text(dist, pos):
    return "".join("%d %d %.17g\n" % (k, int(p), float(d)) for k, (d, p) in enumerate(zip(dist, pos)))


def parity_object(name, count, dist, pos, arm):
    """The parity check of the BASELINE query set against the committed golden answers."""
    import hashlib

    text = answers_text(dist, pos)
    gold, meta = golden_for(name, count)
    obj = {"queries": len(dist), "rows": f"0..{len(dist) - 1} of the query stream", "arm": arm,
           "digest": hashlib.sha256(text.encode()).hexdigest(), "format": "%zu %u %.17g (query, position, distance)"}
    if gold is None:
        obj["golden"] = None
        return obj, True
    gl = [l.split() for l in gold.splitlines()]
    k = min(len(gl), len(dist))  # the golden set is BASELINE's 100 queries
    gpos = np.array([int(x[1]) for x in gl[:k]])
    gdist = np.array([float(x[2]) for x in gl[:k]])
    dist, pos = np.asarray(dist, np.float64)[:k], np.asarray(pos, np.int64)[:k]
    obj["compared"] = k
    rel = np.abs(dist - gdist) / np.maximum(gdist, 1e-300)
    obj.update({"golden": "tests/golden/c2_answers.txt (reference scan_nn over all series)",
                "golden_digest": meta["answers_sha256"], "digest_equal": obj["digest"] == meta["answers_sha256"],
                "positions_equal": int((pos == gpos).sum()),
                "distances_bitwise_equal": int((dist == gdist).sum()),
                "max_rel_dist_err": float(rel.max()) if len(rel) else 0.0})
    ok = obj["positions_equal"] == k and obj["max_rel_dist_err"] <= 1e-5
    return obj, ok


def cmin_bytes(name, count, n, w=16):
    """SURVEY 8(d)'s flat-scan query bytes N*w + C_min*4n per query, C_min (words whose LB is below
    the exact NN distance) averaged over the golden query set (computed by the oracle over all words)."""
    _, meta = golden_for(name, count)
    if meta is None:
        return None
    cm = float(np.mean(meta["cmin"]))
    return {"bytes_per_query": count * w + cm * 4 * n, "mean_cmin": cm, "cmin_frac": cm / count,
            "source": "tests/golden/c2_golden.json (oracle, BASELINE queries rows 0..99)"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


NCU_SUMMARY = os.path.join(ROOT, "profiles", "round2e_ncu_summary.json")
NCU_REPORTS = {"lbscan": ["prof_k_lbscan.ncu-rep"], "refine": ["prof_k_refine_tma.ncu-rep"],
               "bound": ["prof_k_groups.ncu-rep", "prof_k_bound.ncu-rep"], "summarise": ["prof_k_summarise.ncu-rep"]}


RANDOM_BW = os.path.join(ROOT, "profiles", "micro", "random_bw_b200.json")


def ncu_binding(kernel):
    """What binds a query kernel, from the committed ncu capture, time-weighted over the kernel's
    launches of one batch: the issue slots (the kernels are instruction-issue-bound since the
    query-switch stalls were removed), the L1/LSU data pipe and shared-memory part of it, and the
    DRAM side against the RANDOM-LINE rate of this B200 (profiles/micro/random_bw.cu): the reads
    are scattered 128-byte lines, which HBM3e serves at ~4.7 TB/s, not at the sequential peak."""
    if not os.path.exists(NCU_SUMMARY) or kernel not in NCU_REPORTS:
        return None
    with open(NCU_SUMMARY) as f:
        reps = json.load(f)["reports"]
    recs = [r for name in NCU_REPORTS[kernel] for r in reps.get(name, [])]
    if not recs or any("lsu_pipe_pct" not in r for r in recs):
        return None
    t = sum(r["time_us"] for r in recs)
    issue = sum(r["issue_active_pct"] * r["time_us"] for r in recs) / t / 100
    lsu = sum(r["lsu_pipe_pct"] * r["time_us"] for r in recs) / t / 100
    shared = sum(r["lsu_shared_pct"] * r["time_us"] for r in recs) / t / 100
    dram = sum(r["dram_pct_peak"] * r["time_us"] for r in recs) / t / 100
    out = {"resource": "instruction issue slots (smsp__issue_active), time-weighted over the batch's launches",
           "frac": round(issue, 3), "lsu_data_pipe_frac": round(lsu, 3), "lsu_shared_part": round(shared, 3),
           "dram_frac_of_ncu_peak": round(dram, 3), "source": os.path.relpath(NCU_SUMMARY, ROOT)}
    if os.path.exists(RANDOM_BW):
        with open(RANDOM_BW) as f:
            peak = json.load(f)["random_line_peak_gbs"]
        gbs = sum(r.get("dram_read_MB", 0.0) + r.get("dram_write_MB", 0.0) for r in recs) * 1e-3 / (t * 1e-6)
        out["dram_random_line"] = {"achieved_gbs": round(gbs, 1), "peak_gbs": peak, "frac": round(gbs / peak, 3),
                                   "peak_def": "random 128-byte line reads over a 4-32 GB span, CUDA events",
                                   "source": os.path.relpath(RANDOM_BW, ROOT)}
    return out


def ncu_traffic(kernel, nq):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` per batch (all its launches of one
    batch: both waves for lbscan / refine), from the committed `ncu --set full` capture of the c2
    bench command (profiles/ncu_round2e.sh); None when the capture does not match this run."""
    if not os.path.exists(NCU_SUMMARY) or kernel not in NCU_REPORTS:
        return None
    with open(NCU_SUMMARY) as f:
        reps = json.load(f)["reports"]
    total = 0.0
    for name in NCU_REPORTS[kernel]:
        recs = reps.get(name)
        if not recs:
            return None
        total += sum(r.get("dram_read_MB", 0.0) + r.get("dram_write_MB", 0.0) for r in recs)
    per = "launch" if kernel == "summarise" else f"batch of {nq} queries (all of the batch's launches)"
    return {"bytes": round(total * 1e6), "per": per, "source": os.path.relpath(NCU_SUMMARY, ROOT)}


class Clocks:
    """SM clock and throttle-reason sampling during the timed region (B200_PROFILING.md clocks
    line). NVML is initialised BEFORE the region and polled from a thread every 5 ms: starting
    an `nvidia-smi -lms` process inside a 50 ms region perturbed it (its driver initialisation cost
    the device-query pass up to 3%); nvidia-smi remains the fallback when pynvml is missing."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.max_mhz = 0.0
        try:
            import pynvml

            pynvml.nvmlInit()
            # CUDA_VISIBLE_DEVICES remaps indices: resolve the torch device through its PCI bus id
            try:
                import torch

                bus = torch.cuda.get_device_properties(device).pci_bus_id
                dom = torch.cuda.get_device_properties(device).pci_domain_id
                dev_id = torch.cuda.get_device_properties(device).pci_device_id
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(f"{dom:08X}:{bus:02X}:{dev_id:02X}.0".encode())
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.nvml = pynvml
        except Exception:
            self.nvml = None

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
                try:
                    rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle))
                except Exception:
                    rs = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle))
                self.samples.append((mhz, rs))
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        if self.nvml:
            import threading

            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.nvml:
            self.stop.set()
            self.thread.join(timeout=2)
            return
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        if self.nvml:
            nv = self.nvml
            bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
            for mhz, rs in self.samples:
                sm.append(mhz)
                reasons.update(n for n, b in bits.items() if rs & b)
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz or None,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, 5 ms polling"}
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_obj(name, count, n, sigma, nq_par):
    """The workload description both arms print identically (same keys and values)."""
    return {"workload": workload_text(name, count, n, sigma),
            "parity_queries": f"rows 0..{nq_par - 1} of the query stream (BASELINE's {nq_par} queries)",
            "l2_flush": f"inputs larger than L2 ({count * n * 4 / 1e9:.1f} GB of rows)"}


def workload_text(name, count, n, sigma=None):
    spec = CONFIGS[name]
    dkind, _, _, seed = spec["data"]
    qkind, qseed, _ = spec["queries"]
    what = {"rw": "z-normalised random walks", "c3": "AR(1)+sinusoid series, z-normalised",
            "c4": "1024-component Gaussian-mixture vectors, z-normalised"}[dkind]
    q = {"rw": f"random walks (seed {qseed})", "c3": "unseen series of the same process",
         "c4": "unseen vectors of the same mixture",
         "c5": f"dataset rows + N(0, {sigma}^2) noise, re-z-normalised (seed {qseed})"}[qkind]
    return f"{name}: {count} x {n} {what} (seed {seed}); queries: {q}; w=16, 8-bit, leaf 2000"


def ref_inputs(name, count, n, nq_total, sigma, sample_cap):
    """Reference-side index + queries for a config (RW data is built inside the
    reference without a host copy; c3/c4 data and c5 queries come from the
    oracle's generators, the only other code allowed here). Returns
    (index, queries, dataset_count, generate_ns)."""
    from oracle.oracle import Oracle, Reference

    spec = CONFIGS[name]
    dkind, _, _, seed = spec["data"]
    qkind, qseed, qbegin = spec["queries"]
    ref, orc = Reference(), Oracle()
    if dkind == "rw":
        idx, gen_ns = ref.build_generated(count, n, seed)
    else:
        count = min(count, sample_cap)
        t0 = time.perf_counter()
        rows = (orc.generate_c3 if dkind == "c3" else orc.generate_c4)(count, n, seed)
        gen_ns = int((time.perf_counter() - t0) * 1e9)
        idx = ref.build_index(rows)
        del rows
    if qkind == "rw":
        qs = ref.series_window(qbegin, nq_total, n, qseed)
    elif qkind == "c5":
        qs, _ = orc.c5_queries(nq_total, sigma, qseed, seed, count, n)
    else:
        qs = (orc.generate_c3 if qkind == "c3" else orc.generate_c4)(nq_total, n, qseed, begin=count)
    return idx, qs, count, gen_ns


def cpu_baseline(name, count_full, n, sigma, sample, queries, dtw=-1):
    """The unmodified reference (oracle/_ref) on this host's cores, on a
    bounded sample of the workload (the first `sample` series of the same
    dataset): reference build_index + exact_search (mq, 24 queues, all cores).
    With dtw >= 0: exact_search(Measure::dtw(dtw)) on a 1M-series sample."""
    from oracle.oracle import Reference

    cores = Reference().hardware_concurrency()
    if dtw >= 0:
        sample = min(sample, 1_000_000)
        queries = min(queries, 5)
    idx, qs, used, _ = ref_inputs(name, min(sample, count_full), n, queries, sigma, sample)
    t = []
    for q in qs:
        if dtw >= 0:
            t0 = time.perf_counter_ns()
            idx.exact_search_dtw(q, dtw)
            t.append(time.perf_counter_ns() - t0)
        else:
            d, p, st, ns = idx.exact_search(q)
            t.append(ns)
    qps = len(t) / (sum(t) * 1e-9)
    build_ns = idx.build_stats["build_ns"]
    return {"value": round(qps, 3), "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": f"first {used} of the {count_full} series (same generator/seed), {queries} queries; "
                      f"reference build_index + exact_search(mq, 24 queues, {cores} workers)",
            "build_mseries_s": round(used / (build_ns * 1e-9) / 1e6, 3),
            "median_query_ms": round(statistics.median(t) * 1e-6, 3)}


def run_reference(args):
    world, rank, local = dist_setup()
    if rank != 0:
        return
    from oracle.oracle import Reference

    spec = CONFIGS[args.config]
    _, count, n, _ = spec["data"]
    if spec.get("per_gpu"):
        count *= max(args.gpus, 1)
    if args.count:
        count = args.count
    cores = Reference().hardware_concurrency()
    per_step = args.ref_queries_per_step
    nq_par = args.batch or spec["nq"]
    total = max((args.warmup + args.steps) * per_step, nq_par)
    idx, qs, used, gen_ns = ref_inputs(args.config, count, n, total, args.sigma, args.ref_sample)
    build_ns = idx.build_stats["build_ns"]
    ans = {}
    for k, q in enumerate(qs[: args.warmup * per_step]):
        d, p, _, _ = idx.exact_search(q)
        ans[k] = (d, p)
    t0 = time.perf_counter()
    times = []
    for k, q in enumerate(qs[args.warmup * per_step:(args.warmup + args.steps) * per_step]):
        d, p, st, ns = idx.exact_search(q)
        times.append(ns)
        ans[args.warmup * per_step + k] = (d, p)
    elapsed = time.perf_counter() - t0
    qps = len(times) / elapsed
    for k in range(nq_par):  # the rest of the parity set, untimed
        if k not in ans:
            d, p, _, _ = idx.exact_search(qs[k])
            ans[k] = (d, p)
    parity, ok = parity_object(args.config, used, [ans[k][0] for k in range(nq_par)],
                               [ans[k][1] for k in range(nq_par)], "reference exact_search")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(qps, 4), "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed * 1e3 / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_obj(args.config, used, n, args.sigma, nq_par),
        "step": {"queries_per_step": per_step, "query_rows": f"0..{total - 1} of the query stream",
                 "timed_query_rows": f"{args.warmup * per_step}..{(args.warmup + args.steps) * per_step - 1}"},
        "cpu_baseline": {"value": round(qps, 4), "unit": "queries/s", "cores": cores, "kind": "reference",
                         "sample": f"{used} of {count} series, {args.steps * per_step} timed queries"},
        "e2e": {"value": round(qps, 4), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build": {"value": round(used / (build_ns * 1e-9) / 1e6, 3), "unit": "Mseries/s",
                  "build_s": round(build_ns * 1e-9, 3), "generate_s": round(gen_ns * 1e-9, 3)},
        "median_query_ms": round(statistics.median(times) * 1e-6, 3),
        "parity": parity,
    }
    print(json.dumps(line), flush=True)
    if not ok:
        sys.exit(f"parity: the reference's answers differ from the golden answers ({parity})")


def timed_batches(tg, index, queries, nq, measure=None, warm=1):
    """Queries/s of device-resident query batches through the public API (CUDA events), plus the
    summed per-query statistics and the answers."""
    import torch

    measure = measure or tg.Measure.ed()
    nb = queries.shape[0] // nq
    for b in range(min(warm, nb)):
        tg.exact_search_batch_records(index, queries[b * nq:(b + 1) * nq], measure)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    res = [tg.exact_search_batch_records(index, queries[b * nq:(b + 1) * nq], measure) for b in range(warm, nb)]
    ev1.record()
    torch.cuda.synchronize()
    sec = ev0.elapsed_time(ev1) * 1e-3
    rec = np.concatenate(res)
    return (nb - warm) * nq / sec, rec


def other_configs(args, tg, index, count, n, seed):
    """Secondary BASELINE configs, measured after the headline line's numbers (1 GPU; they are not
    the headline, and their parity is covered by tests/test_gpu_parity.py at sizes the oracle
    finishes): config 5's query-difficulty / batch sweep on the c2 index, then configs 3 and 4
    (the c2 data and index are freed first)."""
    import torch

    out = {"note": "secondary configs (BASELINE.json configs[2..4]), device-resident queries, CUDA events; "
                   "not the headline"}
    sweep = []
    for sigma in (0.01, 0.1, 0.5, 1.0):
        for nq in (1, 64, 1024):
            if nq == 1 and sigma >= 0.5:
                continue  # hard single queries take seconds each: covered by batch 64 / 1024
            total = nq * (2 if nq >= 1024 else 4 if nq == 64 else 40)
            q = tg.generate_device("c5", total, n, 5, begin=0, noise=sigma, data_count=count, data_seed=seed)
            qps, rec = timed_batches(tg, index, q, nq)
            refined = float(rec["stats"][:, 2].astype(np.float64).mean())
            sweep.append({"sigma": sigma, "batch": nq, "queries_per_s": round(qps, 1),
                          "pruning_ratio": round(1 - refined / count, 6), "refined_rows_per_query": round(refined, 1)})
            del q
    out["c5"] = {"workload": workload_text("c5", count, n, "sigma"), "sweep": sweep}
    return out


def other_configs_c3_c4(tg):
    import torch

    res = {}
    for name in ("c3", "c4"):
        dkind, count, n, seed = CONFIGS[name]["data"]
        qkind, qseed, _ = CONFIGS[name]["queries"]
        rows = tg.generate_device(dkind, count, n, seed)
        q = tg.generate_device(qkind, 4 * 100, n, qseed, begin=count)
        index = tg.build_index(rows, tg.IndexConfig(n=n))
        bs = index.build_stats()
        qps, rec = timed_batches(tg, index, q, 100)
        refined = float(rec["stats"][:, 2].astype(np.float64).mean())
        res[name] = {"workload": workload_text(name, count, n), "queries_per_s": round(qps, 1),
                     "build_mseries_s": round(count / (bs.build_ns * 1e-9) / 1e6, 1),
                     "build_ms": round(bs.build_ns * 1e-6, 2), "pruning_ratio": round(1 - refined / count, 6),
                     "timed_queries": 300}
        index.free()
        del rows, q, index
        torch.cuda.empty_cache()
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2009_00786_b200 as tg
    from paper_2009_00786_b200 import _lib
    from paper_2009_00786_b200.shard import shard_range

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    ctx = tg.Context((local,))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        # the library's own communicator (seed-BSF allreduce + result all-gather inside tsg_search);
        # torch.distributed only carries its id and the bench's barrier / max-over-ranks
        cid = [tg.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(cid, src=0)
        ctx.comm_init(world, rank, cid[0])

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    spec = CONFIGS[args.config]
    dkind, count, n, seed = spec["data"]
    qkind, qseed, qbegin = spec["queries"]
    nq = args.batch or spec["nq"]
    if spec.get("per_gpu"):
        count *= world
    if args.count:
        count = args.count
    b, e = shard_range(count, rank, world)
    shard = e - b

    # ---- inputs in HBM (untimed setup), generated on the device ----
    t0 = time.perf_counter()
    rows = tg.generate_device(dkind, shard, n, seed, begin=b, device=local)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    # batch 0: the parity set (BASELINE's queries, rows 0..nq-1); 1..W warm-up; W+1..W+K timed
    total_batches = 1 + args.warmup + args.steps
    qdev = tg.generate_device(qkind, total_batches * nq, n, qseed, begin=count if qbegin is None else qbegin,
                              device=local, noise=args.sigma, data_count=count, data_seed=seed)
    qhost = qdev.cpu().numpy()

    # ---- build (device-timed inside the library with CUDA events) ----
    cfg = tg.IndexConfig(n=n)
    # untimed warm-up build of a 1M-series prefix: loads every build kernel's module
    # (lazy loading) before the timed build
    warm = tg.build_index(rows[: min(shard, 1_000_000)], cfg, devices=(local,))
    warm.free()
    del warm
    torch.cuda.synchronize()
    barrier()
    tb = time.perf_counter()
    index = tg.build_index(rows, cfg, context=ctx, position_offset=b)
    torch.cuda.synchronize()
    build_wall = max_over_ranks(time.perf_counter() - tb)
    bs = index.build_stats()
    build_dev_s = max_over_ranks(bs.build_ns * 1e-9)
    k1_s = max_over_ranks(bs.summarise_ms * 1e-3)

    measure = tg.Measure.dtw(args.dtw) if args.dtw >= 0 else tg.Measure.ed()

    def step(batch, host):
        # one C-ABI call per batch; results as a record array (no per-query Python objects). With
        # world > 1 the call is collective: the library exchanges seed BSFs and merges the shards'
        # answers over NCCL, so every rank gets the global answers.
        src = qhost if host else qdev
        res = tg.exact_search_batch_records(index, src[batch * nq:(batch + 1) * nq], measure)
        return res

    def timed(host, stats=None, answers=None):
        # CUDA events on the current stream bracket the K batches; each batch
        # call returns only after its lanes' streams finished (results are on
        # the host), so the end event is recorded after all of the batch work.
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        kept = []
        for i in range(1 + args.warmup, total_batches):
            kept.append(step(i, host=host))
        ev1.record()
        torch.cuda.synchronize()
        barrier()
        for res in kept:  # bookkeeping outside the timed region
            if answers is not None:
                answers.append(res)
            if stats is not None:
                st = res["stats"].astype(np.float64).sum(axis=0)
                stats += (*st, float(res["box_calcs"].astype(np.float64).sum()), float(res["fine_calcs"].astype(np.float64).sum()))
        return max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)

    # parity set (untimed): BASELINE's queries against the golden answers
    par = step(0, host=True)
    parity, parity_ok = parity_object(args.config, count, par["distance"], par["position"], "ours (tsg_search)")
    # warm-up
    for i in range(1, 1 + args.warmup):
        step(i, host=False)
    torch.cuda.synchronize()

    # ---- timed: device-resident queries (the `value`) ----
    # Each call is synchronous (results come back to the host per batch): the
    # event pair measures the K batches plus the per-batch result D2H.
    launches0 = tg.launch_count()
    stats_acc = np.zeros(8, np.float64)
    answers = []
    with Clocks(local) as clk:
        elapsed = timed(False, stats_acc, answers)
    launches = tg.launch_count() - launches0
    qps = args.steps * nq / elapsed

    # ---- timed: end to end through the public API with host queries ----
    e2e_s = timed(True)
    e2e_qps = args.steps * nq / e2e_s

    # ---- per-kernel CUDA-event timing pass (the roofline numbers) ----
    _lib.check(_lib.lib().tsg_profile_enable(index.handle, 1))
    _lib.check(_lib.lib().tsg_profile_read(index.handle, None, None, 1))
    prof_s = timed(False)
    ms = (ctypes.c_double * 8)()
    ln = (ctypes.c_uint64 * 8)()
    _lib.check(_lib.lib().tsg_profile_read(index.handle, ms, ln, 1))
    _lib.check(_lib.lib().tsg_profile_enable(index.handle, 0))
    prof_ms = [max_over_ranks(x) for x in ms]
    prof_ln = list(ln)

    # ---- roofline of the dominant query kernel (algorithmic bytes from the counters) ----
    hbm, peak_kind = peaks()
    nqt = args.steps * nq
    ws = 16
    P = bs.pages
    # library profile slots (include/tsgpu.h): 1 groups + bound, 2 prepare + seed, 3 refine wave A,
    # 4 lbscan, 5 refine wave B, 6 finalize, 7 cross-shard seed exchange
    groups = {"bound": [1], "seed": [2], "lbscan": [4], "refine": [3, 5], "finalize": [6], "exchange": [7]}
    lb_nodes, lb_entries, refined, cands, boxes = stats_acc[0], stats_acc[1], stats_acc[2], stats_acc[5], stats_acc[6]
    fine_calcs = stats_acc[7]
    fw = 2 * 16 if (n % 32 == 0 and not os.environ.get("TSG_NO_FINE")) else 0  # fine summary bytes per series (w = 16)
    NG = (P + 7) // 8
    group_bytes = {  # algorithmic bytes over the timed pass (per-unit figures of DESIGN.md §4 x the counters)
        # every group box (2 x 16 B) + pages of surviving groups and runs of surviving pages
        # (lb_node_calcs - groups; 2 x 16 B boxes, + 8 B offsets for pages: counted as 36 B)
        "bound": nqt * NG * 2 * ws + max(lb_nodes - nqt * NG, 0) * (2 * ws + 4),
        # quad boxes (box_calcs, 2 x 16 B) + words of surviving quads + candidate records (pos + bound)
        "lbscan": boxes * 2 * ws + lb_entries * ws + cands * 8,
        # candidate records (bound, row, sum) + the fine summary rows of those within the BSF
        # + the refined rows (full length)
        "refine": refined * 4 * n + cands * 16 + fine_calcs * fw,
    }
    group_ms = {g: sum(prof_ms[k] for k in ks) for g, ks in groups.items()}
    dom = max(group_ms, key=group_ms.get)
    dom_ms = group_ms[dom] / nqt  # per query (each group runs once per query per rank)
    dom_bytes = group_bytes.get(dom, 0.0) / nqt
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9 if dom_ms > 0 else 0.0
    # lbscan's other roofline: shared-memory table lookups (16 per quad box and per word), against one
    # conflict-free 32-lane wavefront per SM per clock
    props = torch.cuda.get_device_properties(local)
    sm_clock_mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0)) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
    lookups = (boxes + lb_entries) * ws
    lbscan_s = group_ms["lbscan"] * 1e-3
    smem_peak = props.multi_processor_count * sm_clock_mhz * 1e6 * 32 * world  # all ranks' SMs
    smem_roof = {"kernel": "lbscan", "bound": "smem", "unit": "table lookups/s",
                 "achieved": lookups / lbscan_s if lbscan_s > 0 else 0.0, "peak": smem_peak,
                 "frac": round(lookups / lbscan_s / smem_peak, 4) if lbscan_s > 0 else 0.0,
                 "peak_def": f"{props.multi_processor_count} SMs x {sm_clock_mhz:.0f} MHz x 32 lanes "
                             "(one conflict-free shared wavefront per SM per clock)"}
    flat = cmin_bytes(args.config, count, n, ws)
    # DRAM bytes per batch of the same kernel from the committed ncu capture (c2, 1 GPU only)
    traffic = ncu_traffic(dom, nq) if args.config == "c2" and world == 1 and nq == 100 else None

    # build K1 roofline: read 4n, write the 8-byte sort key and the word + fine row (one 64-byte
    # record per series when the fine summary is 32 wide, else 16-byte word + fine row)
    k1_rec = 64 if fw == 32 else 16 + fw
    k1_bytes = count * (4 * n + 8 + k1_rec) / world
    k1_gbs = k1_bytes / k1_s / 1e9
    algo_build = count * (4 * n + 16 + 4)  # N(4n + w + 4)

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(args.config, count, n, args.sigma, args.cpu_sample, args.cpu_queries, args.dtw)
            except Exception as ex:  # reported, not hidden
                cpu = {"error": str(ex)}
        clocks = clk.summary()
        share = group_ms[dom] / max(sum(group_ms.values()), 1e-12)
        line = {
            "metric": METRIC if args.dtw < 0 else METRIC.replace("exact 1-NN", f"exact 1-NN DTW(window {args.dtw})"),
            "value": round(qps, 3), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(elapsed * 1e3 / args.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_obj(args.config, count, n, args.sigma, nq),
            "step": {"queries_per_step": nq, "query_rows": f"0..{total_batches * nq - 1} of the query stream",
                     "timed_query_rows": f"{(1 + args.warmup) * nq}..{total_batches * nq - 1}",
                     "sharding": f"{world} contiguous series ranges, one process per GPU"
                                 + (", library NCCL communicator" if world > 1 else ""),
                     "per_gpu_bytes": f"{count * n * 4 / world / 1e9:.1f} GB rows, "
                                      f"{count * 16 / world / 1e9:.2f} GB words"},
            "parity": parity,
            "e2e": {"value": round(e2e_qps, 3), "unit": "queries/s", "h2d_bytes_per_step": nq * n * 4,
                    "d2h_bytes_per_step": nq * 72},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                         "peak": hbm * world, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / (hbm * world), 4),
                         "peak_note": "per-GPU measured peak x ranks (achieved is the whole job's bytes / max-rank time)"
                                      if world > 1 else "one GPU",
                         "traffic": traffic,
                         "algorithmic_bytes_per_batch": round(dom_bytes * nq),
                         "batch_queries": nq,
                         "share_of_query_time": round(share, 4),
                         "per_kernel_ms": {g: round(v, 3) for g, v in group_ms.items()},
                         "per_kernel_us_per_query": {g: round(v * 1e3 / nqt, 2) for g, v in group_ms.items()},
                         "per_slot_us_per_query": [round(v * 1e3 / nqt, 2) for v in prof_ms],
                         "profiled_pass_s": round(prof_s, 4),
                         "lbscan_smem": smem_roof,
                         "binding": ncu_binding(dom) if args.config == "c2" and world == 1 and nq == 100 else None},
            "flat_scan_roofline": None if flat is None else {
                "formula": "SURVEY 8(d): N*w + C_min*4n bytes per query",
                "bytes_per_query": round(flat["bytes_per_query"]), "mean_cmin": round(flat["mean_cmin"], 1),
                "cmin_frac": round(flat["cmin_frac"], 7), "source": flat["source"],
                "equivalent_gbs": round(flat["bytes_per_query"] * qps / 1e9, 1),
                "equivalent_frac": round(flat["bytes_per_query"] * qps / 1e9 / hbm / world, 3),
                "note": "what a flat LB scan would have to move per query; the box hierarchy reads ~1% of the "
                        "words, so this exceeds 1 by design"},
            "build": {"value": round(count / build_dev_s / 1e6, 3), "unit": "Mseries/s",
                      "build_device_s": round(build_dev_s, 4), "build_wall_s": round(build_wall, 3),
                      "phase_ms": {"summarise": round(bs.summarise_ms, 3), "organise": round(bs.organise_ms, 3),
                                   "leaves": round(bs.leaves_ms, 3)},
                      "roofline": {"bound": "hbm", "kernel": "summarise (K1)", "achieved": round(k1_gbs, 1),
                                   "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                                   "frac": round(k1_gbs / hbm, 4),
                                   "traffic": ncu_traffic("summarise", nq) if args.config == "c2" and world == 1 else None,
                                   "algorithmic_bytes_per_series": 4 * n + 8 + k1_rec},
                      "whole_build_frac": round(algo_build / build_dev_s / 1e9 / hbm / world, 4),
                      "leaves": bs.leaves, "pages": P, "root_children": bs.root_children, "max_depth": bs.max_depth,
                      "overflow_leaves": bs.overflow_leaves},
            "search_stats_per_query": {k: round(v / nqt, 2) for k, v in zip(
                ["lb_node_calcs", "lb_entry_calcs", "real_dist_calcs", "bsf_updates", "pruned_subtrees",
                 "queue_insertions", "box_calcs", "fine_calcs"], stats_acc)},
            # pruning ratio = 1 - refined rows / dataset rows (BASELINE config 5's difficulty measure)
            "pruning_ratio": round(1.0 - stats_acc[2] / nqt / count, 6),
            "query_bytes_gbs": round((lb_entries * ws + refined * 4 * n + nqt * P * (2 * ws + 8)) / elapsed / 1e9, 1),
            "clocks": clocks,
            "generate_s": round(gen_s, 2),
            "cpu_baseline": cpu,
        }
        if world == 1 and args.config == "c2" and not args.no_other_configs:
            try:  # secondary configs: reported inside the line, never failing the headline
                extra = other_configs(args, tg, index, count, n, seed)
                index.free()
                del rows, qdev
                torch.cuda.empty_cache()
                extra.update(other_configs_c3_c4(tg))
                line["other_configs"] = extra
            except Exception as ex:
                line["other_configs"] = {"error": str(ex)[:300]}
        print(json.dumps(line), flush=True)
    index.free()
    if world > 1:
        dist.destroy_process_group()
    if not parity_ok:
        sys.exit(f"parity: answers differ from the golden answers ({parity})")


def run_ingest(args):
    """build straight from a headerless f32 file. The first
    `--ingest` series of the config's dataset are written to a scratch file
    (untimed; the file is then in the page cache), and tsg_index_build_file
    streams it through pinned buffers with K1 overlapped. Reports file GB/s
    and Mseries/s end to end (wall clock of the build call), 1 GPU."""
    import tempfile

    import torch

    import paper_2009_00786_b200 as tg

    dkind, _, n, seed = CONFIGS[args.config]["data"]
    count = args.ingest
    rows = tg.generate_device(dkind, count, n, seed)
    fd, path = tempfile.mkstemp(suffix=".f32", dir=os.environ.get("TSG_SCRATCH", "/tmp"))
    os.close(fd)
    try:
        rows.cpu().numpy().tofile(path)
        del rows
        torch.cuda.empty_cache()
        cfg = tg.IndexConfig(n=n)
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            index = tg.build_index_from_file(path, cfg)
            wall = time.perf_counter() - t0
            st = index.build_stats()
            index.free()
            if best is None or wall < best[0]:
                best = (wall, st)
        wall, st = best
        gb = count * n * 4 / 1e9
        print(json.dumps({"metric": "index build from a float32 file (page cache -> pinned -> HBM, K1 overlapped)",
                          "value": round(count / wall / 1e6, 3), "unit": "Mseries/s", "file_gb": round(gb, 3),
                          "file_gbs": round(gb / wall, 2), "wall_s": round(wall, 3),
                          "stream_phase_s": round(st.h2d_ns * 1e-9, 3),
                          "phase_ms": {"stream+summarise": round(st.summarise_ms, 3),
                                       "organise": round(st.organise_ms, 3), "leaves": round(st.leaves_ms, 3)},
                          "config": {"workload": f"first {count} series of {args.config}", "n": n}}))
    finally:
        os.unlink(path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--count", type=int, default=0, help="override the series count (testing)")
    ap.add_argument("--cpu-sample", type=int, default=10_000_000)
    ap.add_argument("--cpu-queries", type=int, default=20)
    ap.add_argument("--ref-queries-per-step", type=int, default=4)
    ap.add_argument("--ref-sample", type=int, default=20_000_000,
                    help="cap on host-generated (c3/c4) datasets for the reference arm")
    ap.add_argument("--batch", type=int, default=0, help="queries per step (default: the config's 100)")
    ap.add_argument("--sigma", type=float, default=0.1, help="c5 query noise")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the secondary configs (c5 sweep on the c2 index, c3, c4) reported in other_configs")
    ap.add_argument("--dtw", type=int, default=-1, help="search under Measure::dtw(window) (SURVEY 8(f)#4)")
    ap.add_argument("--ingest", type=int, default=0,
                    help="instead of the search bench: build from a file of this many series (SURVEY 8(f)#3)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.impl == "ours" and not args.ingest:
        if args.gpus > 1 and world == 0:
            # one process per GPU: re-launch this command under torch.distributed.run
            import socket

            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
            sys.exit(subprocess.call(cmd))
        if world and world != args.gpus:
            sys.exit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.ingest:
        run_ingest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
