#!/usr/bin/env python
"""Benchmark: FMM particles/sec of the full adaptive FMM pipeline on B200.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c1|c2|c3|c4|c5] [--n N]
For N > 1 launch with torch.distributed.run (one rank per GPU, NCCL): the
distributed engine (paper_1205_4611_b200.distributed) evaluates
one problem of N_gpus x N points, subtrees partitioned across the ranks
(weak scaling).

A "step" is one full fmm_evaluate (tree build through P2P and un-permute) of
the configured point set.  `value` is measured with inputs resident in HBM
(device pointers) and CUDA events on the engine's stream; `e2e` goes through
the public drop-in API fmm_evaluate(ParticleSet(...)) with pinned host
buffers, host<->device copies inside the timed region.  L2 (126 MB) is
flushed between timed steps by writing a 512 MiB buffer.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[0..4]
    "c1": dict(kind="uniform", n=10_000, m=None, p=17, desc="uniform N=1e4, p=17 (CPU-runnable case)"),
    "c2": dict(kind="uniform", n=1_000_000, m=None, p=20, desc="uniform N=1e6, p=20, single B200"),
    "c3": dict(kind="normal", n=1_000_000, m=None, p=20, desc="normal sigma^2=0.01 N=1e6, p=20"),
    "c4": dict(kind="uniform", n=1_000_000, m=1_000_000, p=30,
               desc="uniform N=M=1e6 separate evaluation points, p=30"),
    "c5": dict(kind="uniform", n=10_000_000, m=None, p=20, desc="uniform N=1e7, p=20"),
}
METRIC = "FMM particles/sec (FP64, p≈20) at 1/2/4/8 B200; per-phase roofline fraction"
FP64_PEAK_FILE = ROOT / "profiles" / "r01_fp64_peak.json"


def m2l_flops_per_pair(p):          # 2p(p+1) + 18p
    return 2 * p * (p + 1) + 18 * p


def p2p_flops_per_interaction():
    return 11


HBM_FALLBACK_GBS = 6650.0   # B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)


def ncu_traffic(kernel, config):
    """dram__bytes_read + dram__bytes_write of one launch of `kernel` from the
    committed ncu capture (profiles/r01/ncu_traffic.json), or None."""
    try:
        d = json.loads((ROOT / "profiles" / "r01" / "ncu_traffic.json").read_text())
        t = d[kernel][config]
        return int(t["dram_read"] + t["dram_write"])
    except Exception:
        return None


def hbm_peak():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback copy bandwidth"


def phase_roofline(phase_ms, totals, n, m, levels, p, aliased, fp64_peak):
    """Per-phase roofline fractions (SURVEY 8(d) algorithmic work per unit).

    Compute phases count flops against the FP64 peak; the tree build counts
    bytes against HBM.  Interaction counts use the uniform leaf population
    n / 4^L (exact for the median-split tree up to +-1 per leaf)."""
    leaves = 4 ** levels
    per_leaf_src, per_leaf_ev = n / leaves, m / leaves
    k_children = sum(4 ** l for l in range(2, levels + 1))
    work = {
        "sort": ("bytes", 2 * levels * 2 * (28 * n + (0 if aliased else 20 * m))),
        "connect": ("bytes", 4 * sum(totals.values())),
        "p2m": ("flop", n * (8 * p + 2) + totals["p2l"] * per_leaf_src * (8 * (p + 1) + 11)),
        "m2m": ("flop", k_children * (p * (p - 1) + 18 * p)),
        "m2l": ("flop", totals["weak"] * (2 * p * (p + 1) + 18 * p)),
        "l2l": ("flop", k_children * (p * (p + 1) + 12 * p)),
        "l2p": ("flop", m * (8 * p + 2) + totals["m2p"] * per_leaf_ev * (8 * p + 10)),
        "p2p": ("flop", totals["p2p"] * per_leaf_ev * per_leaf_src * 11),
    }
    hbm, _ = hbm_peak()
    out = {}
    for k, (kind, w) in work.items():
        ms = phase_ms.get(k, 0.0)
        if ms <= 0:
            continue
        if kind == "flop":
            ach = w / (ms * 1e-3) / 1e12
            out[k] = {"bound": "fp64", "achieved": round(ach, 3), "unit": "TFLOP/s",
                      "frac": round(ach / fp64_peak, 4)}
        else:
            ach = w / (ms * 1e-3) / 1e9
            out[k] = {"bound": "hbm", "achieved": round(ach, 1), "unit": "GB/s",
                      "frac": round(ach / hbm, 4)}
    return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_points(cfg, seed):
    import paper_1205_4611_b200 as F
    pts = F.sample_points(F.DistributionSpec(cfg["kind"], 0.01, seed), cfg["n"])
    if cfg["m"] is None:
        return pts
    ev = F.sample_points(F.DistributionSpec(cfg["kind"], 0.01, seed + 1), cfg["m"]).positions
    return F.ParticleSet(pts.positions, pts.strengths, ev)


class ClockSampler:
    """SM clock and throttle reasons polled through NVML (about every 2 ms)
    while the timed region runs; nvidia-smi's 100 ms floor is longer than a
    whole timed region at C2."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.stop_flag = threading.Event()
        self.thread = None
        self.max_mhz = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv, h = self.nv, self.h
        while not self.stop_flag.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        self.stop_flag.set()
        if self.thread:
            self.thread.join(timeout=2)
        names = sorted(v for k, v in self.REASONS.items() if self.reasons & k)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples),
                "source": "NVML poll during the timed region"}


def run_ours(args, cfg, ws, rank, local):
    import torch
    import paper_1205_4611_b200 as F
    from paper_1205_4611_b200.engine import fmm_evaluate_device

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    tcfg = F.TreeConfig(35, 0.5, cfg["p"])
    pts = make_points(cfg, seed=rank)
    n, m = pts.n_sources, pts.n_evals
    alias = pts.evals_alias_sources

    # device-resident inputs (value) -------------------------------------------
    d_pos = torch.from_numpy(pts.positions.view(np.float64).reshape(-1, 2)).to(dev)
    d_g = torch.from_numpy(pts.strengths).to(dev)
    d_ev = None if alias else torch.from_numpy(pts.eval_positions.view(np.float64).reshape(-1, 2)).to(dev)
    d_out = torch.empty((m, 2), dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)

    def step_device(hist=False):
        return fmm_evaluate_device(n, d_pos.data_ptr(), d_g.data_ptr(), m,
                                   None if d_ev is None else d_ev.data_ptr(), d_out.data_ptr(),
                                   tcfg, device=local, histograms=hist)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step_device()
    clocks = ClockSampler(local)
    reps = []
    walls = []
    barrier()
    clocks.start()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = step_device()
        walls.append(time.perf_counter() - t0)
        reps.append(rep)
    barrier()
    clk = clocks.stop()
    dev_ms = [r.device_seconds * 1e3 for r in reps]
    ms_step = sum(dev_ms) / len(dev_ms)
    phase_ms = {k: 1e3 * sum(r.phase_seconds[k] for r in reps) / len(reps)
                for k in F.PHASE_NAMES[:-1]}

    # end to end through the public API with pinned host buffers ----------------
    h_pos = torch.empty(n, dtype=torch.complex128, pin_memory=True).numpy()
    h_pos[:] = pts.positions
    h_g = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    h_g[:] = pts.strengths
    if alias:
        ps = F.ParticleSet(h_pos, h_g)
    else:
        h_ev = torch.empty(m, dtype=torch.complex128, pin_memory=True).numpy()
        h_ev[:] = pts.eval_positions
        ps = F.ParticleSet(h_pos, h_g, h_ev)
    h_out = torch.empty(m, dtype=torch.complex128, pin_memory=True).numpy()
    for _ in range(max(1, args.warmup // 2)):
        F.fmm_evaluate(ps, tcfg, device=local, out=h_out)
    e2e_s = []
    h2d = d2h = 0
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        vals, rep_e2e = F.fmm_evaluate(ps, tcfg, device=local, out=h_out)
        e2e_s.append(time.perf_counter() - t0)
        h2d, d2h = rep_e2e.h2d_bytes, rep_e2e.d2h_bytes
    barrier()
    e2e_mean = sum(e2e_s) / len(e2e_s)

    # max over ranks
    if ws > 1:
        t = torch.tensor([ms_step, e2e_mean], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_step, e2e_mean = float(t[0]), float(t[1])

    last = reps[-1]
    pairs = last.list_totals.get("weak", 0)
    m2l_ms = phase_ms["m2l"]
    achieved = pairs * m2l_flops_per_pair(cfg["p"]) / (m2l_ms * 1e-3) / 1e12
    try:
        peak = json.loads(FP64_PEAK_FILE.read_text())["dfma_tflops"]
        peak_src = f"self-measured DFMA (= DMMA) FP64 peak, {FP64_PEAK_FILE.relative_to(ROOT)}"
    except Exception:
        peak, peak_src = 37.0, "nominal B200 FP64 (no measured FP64 peak found)"
    out = {
        "metric": METRIC,
        "value": ws * n / (ms_step * 1e-3),
        "unit": "particles/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference sample_points generator, Philox seed = rank)",
        "config": {"workload": cfg["desc"], "name": args.config, "n_sources": n, "n_evals": m,
                   "p": cfg["p"], "theta": 0.5, "n_desired": 35, "distribution": cfg["kind"],
                   "levels": int(last.n_levels), "parallelism": f"replicas x{ws}",
                   "l2": "flushed between timed steps (512 MiB write)"},
        "phase_ms": {k: round(v, 4) for k, v in phase_ms.items()},
        "e2e": {"value": ws * n / e2e_mean, "unit": "particles/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_mean * 1e3},
        # compute roof: on B200 the FP64 tensor (DMMA) peak equals the DFMA vector
        # peak (one shared FP64 pipe, profiles/r01_fp64_peak.json); the kernel
        # runs on the vector pipe
        "roofline": {"kernel": "m2l", "bound": "fp64", "pipe": "fp64 (DMMA = DFMA peak)",
                     "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": ncu_traffic("k_m2l_dense", args.config),
                     "algorithmic": f"{pairs} M2L pairs x {m2l_flops_per_pair(cfg['p'])} flop "
                                    "(SURVEY 8(d)) per launch / M2L phase event time",
                     "peak_source": peak_src},
        "phase_roofline": phase_roofline(phase_ms, last.list_totals, n, m, int(last.n_levels),
                                         cfg["p"], alias, peak),
        "clocks": clk,
        "gpu_launches": int(last.kernel_launches) * args.steps,
        "gpu_launches_per_step": int(last.kernel_launches),
        "host_wall_ms_per_step": 1e3 * sum(walls) / len(walls),
    }
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_n)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return out if rank == 0 else None


def run_dist(args, cfg, ws, rank, local):
    """N > 1 ranks (torchrun, one GPU each): the distributed engine on a weak-scaled
    problem of ws x N points; device time = CUDA events on the
    engine stream around one whole evaluation, max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_1205_4611_b200 as F
    from paper_1205_4611_b200 import _lib
    from paper_1205_4611_b200.distributed import (Comm, engine_stream, evaluate_shard,
                                                  fmm_evaluate_distributed, shard_bounds)

    backend = os.environ.get("FMM2D_DIST_BACKEND", "nccl")
    if backend != "nccl":              # test mode: several ranks may share one GPU
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    comm = Comm()
    tcfg = F.TreeConfig(35, 0.5, cfg["p"])
    n_total = ws * cfg["n"]
    pts = F.sample_points(F.DistributionSpec(cfg["kind"], 0.01, 0), n_total)
    m_total = n_total
    if cfg["m"] is not None:      # C4: separate evaluation points, weak-scaled too
        m_total = ws * cfg["m"]
        ev = F.sample_points(F.DistributionSpec(cfg["kind"], 0.01, 1), m_total).positions
        pts = F.ParticleSet(pts.positions, pts.strengths, ev)
    lo, hi = shard_bounds(n_total, ws, rank)
    st = engine_stream(local)
    ctx = _lib.default_context(local)
    evals = None
    with torch.cuda.stream(st):
        d_pos = torch.from_numpy(pts.positions[lo:hi].view(np.float64).reshape(-1, 2)).to(dev)
        d_g = torch.from_numpy(pts.strengths[lo:hi].copy()).to(dev)
        if cfg["m"] is not None:
            elo, ehi = shard_bounds(m_total, ws, rank)
            d_epos = torch.from_numpy(np.ascontiguousarray(pts.eval_positions[elo:ehi])
                                      .view(np.float64).reshape(-1, 2)).to(dev)
            evals = (m_total, d_epos, elo)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step():
        with torch.cuda.stream(st):
            e0.record(st)
            try:
                vals, idx, rep = evaluate_shard(ctx, comm, n_total, d_pos, d_g, lo, tcfg, evals)
            finally:
                ctx.lib.fmm2d_dist_end(ctx.h)
            e1.record(st)
        st.synchronize()
        return e0.elapsed_time(e1), rep

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(local)
    times, reps = [], []
    barrier()
    clocks.start()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ms, rep = step()
        times.append(ms)
        reps.append(rep)
    barrier()
    clk = clocks.stop()
    ms_step = sum(times) / len(times)
    phase = [sum(r.phase_ms[q] for r in reps) / len(reps) for q in range(8)]
    # end to end: the public SPMD API with the full host point set on every rank
    # (each rank uploads its shard, downloads the values it owns)
    for _ in range(max(1, args.warmup // 2)):
        fmm_evaluate_distributed(pts, tcfg, device=local, gather=False)
    e2e = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        (own, idx), _ = fmm_evaluate_distributed(pts, tcfg, device=local, gather=False)
        e2e.append(time.perf_counter() - t0)
    barrier()
    e2e_s = sum(e2e) / len(e2e)
    t = torch.tensor([ms_step, e2e_s] + phase, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, e2e_s, phase = float(t[0]), float(t[1]), [float(v) for v in t[2:]]
    last = reps[-1]
    pairs = int(last.list_totals[0])
    m2l_ms = phase[4]
    achieved = pairs * m2l_flops_per_pair(cfg["p"]) / (m2l_ms * 1e-3) / 1e12 if m2l_ms else 0.0
    peak = json.loads(FP64_PEAK_FILE.read_text())["dfma_tflops"] if FP64_PEAK_FILE.exists() else 37.0
    names = ["sort", "connect", "p2m", "m2m", "m2l", "l2l", "l2p", "p2p"]
    out = {
        "metric": METRIC, "value": n_total / (ms_step * 1e-3), "unit": "particles/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference sample_points generator, Philox seed 0), sharded by rank",
        "config": {"workload": cfg["desc"] + f", weak-scaled to {ws} x N", "name": args.config,
                   "n_sources": n_total, "n_per_gpu": cfg["n"], "p": cfg["p"], "theta": 0.5,
                   "n_desired": 35, "distribution": cfg["kind"], "levels": int(last.n_levels),
                   "parallelism": f"subtree domain decomposition x{ws} ({backend})",
                   "l2": "flushed between timed steps (512 MiB write)"},
        "phase_ms": {k: round(v, 4) for k, v in zip(names, phase)},
        "e2e": {"value": n_total / e2e_s, "unit": "particles/s",
                "h2d_bytes_per_step": 24 * (hi - lo) + (16 * int(evals[1].shape[0]) if evals else 0),
                "d2h_bytes_per_step": 24 * len(own),
                "ms_per_step": e2e_s * 1e3},
        "roofline": {"kernel": "m2l", "bound": "fp64", "pipe": "fp64 (DMMA = DFMA peak)",
                     "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                     "algorithmic": f"rank-0 M2L pairs {pairs} x {m2l_flops_per_pair(cfg['p'])} "
                                    "flop / slowest rank's M2L phase time"},
        "clocks": clk,
        "gpu_launches": int(last.kernel_launches) * args.steps,
        "gpu_launches_per_step": int(last.kernel_launches),
    }
    dist.destroy_process_group()
    return out if rank == 0 else None


REF_SITE = ROOT / "oracle" / "_ref" / "site"    # oracle/build_ref.sh (test/bench infrastructure)


def _import_reference():
    """The reference package itself (staged by oracle/build_ref.sh; travels to
    the GPU box with the snapshot).  None when it was not staged."""
    if not (REF_SITE / "fmm2d").is_dir():
        return None
    if str(REF_SITE) not in sys.path:
        sys.path.insert(0, str(REF_SITE))
    import fmm2d
    return fmm2d


def _reference_points(fmm2d, cfg, n):
    """The bench inputs from the reference's own generator (datasets.py:53-78):
    sources seed 0, separate evaluation points seed 1 (C4)."""
    from fmm2d.datasets import DistributionSpec, sample_points
    from fmm2d.tree import ParticleSet
    pts = sample_points(DistributionSpec(cfg["kind"], 0.01, 0), n)
    if cfg["m"] is not None:
        ev = sample_points(DistributionSpec(cfg["kind"], 0.01, 1), n).positions
        pts = ParticleSet(pts.positions, pts.strengths, ev)
    return pts


def _ref_single_core(job):
    """Subprocess body: the reference's fmm_evaluate, sequential
    (parallel=False), pinned to one host core with single-threaded BLAS."""
    cfg, n = job
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    fmm2d = _import_reference()
    from fmm2d.tree import TreeConfig
    pts = _reference_points(fmm2d, cfg, n)
    t0 = time.perf_counter()
    _, rep = fmm2d.fmm_evaluate(pts, TreeConfig(35, 0.5, cfg["p"]), parallel=False)
    return time.perf_counter() - t0, {k: round(v, 3) for k, v in rep.phase_seconds.items()}


CPU_FULL_MAX_N = 1_000_000    # the 1-core leg runs the full config up to C2-C4 size (~45-75 s)


def cpu_baseline(cfg, n_sample):
    """The reference's CPU path on one host core: its own
    fmm_evaluate, parallel=False, OPENBLAS_NUM_THREADS=1, same inputs and
    config as the GPU line when N <= 1e6 (C5: a 1e6-point sample).  Falls back
    to the oracle port when the reference was not staged."""
    import concurrent.futures as cf
    import multiprocessing as mp
    n = cfg["n"] if cfg["n"] <= CPU_FULL_MAX_N else min(n_sample, CPU_FULL_MAX_N)
    if _import_reference() is not None:
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        with cf.ProcessPoolExecutor(1, mp_context=mp.get_context("spawn")) as pool:
            dt, phases = pool.submit(_ref_single_core, (cfg, n)).result()
        same = n == cfg["n"]
        return {"value": n / dt, "unit": "particles/s", "cores": 1, "kind": "reference",
                "same_config": same,
                "sample": f"reference fmm2d.fmm_evaluate (oracle/_ref/site), parallel=False, "
                          f"1 core, OPENBLAS_NUM_THREADS=1, {cfg['kind']} N={n}"
                          f"{'' if cfg['m'] is None else ' M=N separate'}, p={cfg['p']}: "
                          f"one call, {dt:.1f} s"
                          + ("" if same else f" (bounded sample of N={cfg['n']})"),
                "phase_seconds": phases}
    from oracle import fmm2d_oracle as O
    import paper_1205_4611_b200 as F
    n = min(n_sample, cfg["n"])
    pts = F.sample_points(F.DistributionSpec(cfg["kind"], 0.01, 0), n)
    ev = None
    if cfg["m"] is not None:
        ev = F.sample_points(F.DistributionSpec(cfg["kind"], 0.01, 1), n).positions
    t0 = time.perf_counter()
    O.fmm(pts.positions, pts.strengths, ev, 35, 0.5, cfg["p"])
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "particles/s", "cores": 1, "kind": "port",
            "same_config": False,
            "sample": f"oracle port (reference not staged) on {cfg['kind']} N={n}, p={cfg['p']}, "
                      f"one call, {dt:.2f} s, numpy single-threaded"}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


REF_BUDGET_S = 150.0   # reference arm: seconds of timed full evaluations


def run_reference(args, cfg, ws, rank):
    """The reference arm: the UNMODIFIED reference package (oracle/_ref/site,
    staged from /root/reference/pkg by oracle/build_ref.sh) through its public
    API fmm2d.fmm_evaluate on the bench's own config and inputs, with every
    host core: parallel=True, n_workers = cores (the
    reference's thread pool, engine.py:50-64, 214-215).  Each timed step is one
    full evaluation (the same N as the GPU line).  Warm-up steps (imports,
    allocator) evaluate a 1e4-point problem of the same distribution.  Under
    torchrun only rank 0 runs."""
    if rank != 0:
        return None
    fmm2d = _import_reference()
    if fmm2d is None:
        return {"impl": "reference",
                "unavailable": "oracle/_ref/site not staged (run oracle/build_ref.sh)"}
    from fmm2d.tree import TreeConfig
    cores = max(1, min(host_cores(), args.ref_cores or host_cores()))
    n = cfg["n"]
    tcfg = TreeConfig(35, 0.5, cfg["p"])
    warm = _reference_points(fmm2d, cfg, min(n, 10_000))
    for _ in range(args.warmup):
        fmm2d.fmm_evaluate(warm, tcfg, parallel=True, n_workers=cores)
    pts = _reference_points(fmm2d, cfg, n)
    secs, phases = [], []
    # one full evaluation per step (~15 s at C2 on 16 cores); the arm stops
    # after REF_BUDGET_S of timed steps (at least two), so a --steps 20 run
    # still ends within a few minutes -- "steps" reports the steps timed
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, rep = fmm2d.fmm_evaluate(pts, tcfg, parallel=True, n_workers=cores)
        secs.append(time.perf_counter() - t0)
        phases.append(rep.phase_seconds)
        if len(secs) >= 2 and time.perf_counter() - t_start > REF_BUDGET_S:
            break
    ms = 1e3 * sum(secs) / len(secs)
    val = n / (ms * 1e-3)
    phase_mean = {k: round(sum(ph[k] for ph in phases) / len(phases), 3) for k in phases[0]}
    sample = (f"reference fmm2d.fmm_evaluate (oracle/_ref/site), parallel=True, "
              f"n_workers={cores}, full {args.config} problem ({cfg['kind']} N={n}"
              f"{'' if cfg['m'] is None else ' M=N separate'}, p={cfg['p']}) per step")
    return {"metric": METRIC, "value": val, "unit": "particles/s", "n_gpus": ws,
            "steps": len(secs), "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference sample_points, seed 0)", "impl": "reference",
            "config": {"workload": cfg["desc"], "name": args.config, "n_sources": n,
                       "n_evals": n if cfg["m"] is not None else n, "p": cfg["p"], "theta": 0.5,
                       "n_desired": 35, "distribution": cfg["kind"], "cores": cores,
                       "warmup_sample": "N=1e4 of the same distribution"},
            "phase_seconds": phase_mean,
            "cpu_baseline": {"value": val, "unit": "particles/s", "cores": cores,
                             "kind": "reference", "same_config": True, "sample": sample},
            "e2e": {"value": val, "unit": "particles/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--npoints", type=int, default=None, help="override N (and M)")
    ap.add_argument("--cpu-n", type=int, default=1_000_000,
                    help="CPU baseline sample size when the config exceeds 1e6 points")
    ap.add_argument("--ref-cores", type=int, default=0,
                    help="host cores for --impl reference (default: all available)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.npoints:
        cfg["n"] = args.npoints
        if cfg["m"] is not None:
            cfg["m"] = args.npoints
    ws, rank, local = dist_env()
    if args.impl == "reference":
        out = run_reference(args, cfg, ws, rank)
    elif ws > 1 or os.environ.get("FMM2D_FORCE_DIST") == "1":
        out = run_dist(args, cfg, ws, rank, local)
    else:
        out = run_ours(args, cfg, ws, rank, local)
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
