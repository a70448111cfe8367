"""Worker for the multi-rank tests: ``python tests/_dist_worker.py MODE OUT``
under torch.distributed.run (MASTER_ADDR=127.0.0.1).  MODE "comm" exercises
the collective layer with CPU tensors (gloo); MODE "engine:<kind>:<n>:<p>"
runs the distributed FMM with every rank on cuda:0 (gloo staging) and rank 0
saves values, indices and the report to OUT (npz)."""

import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def comm_checks(out):
    import torch
    import torch.distributed as dist
    from paper_1205_4611_b200.distributed import Comm, shard_bounds, top_split_steps
    c = Comm()
    G, r = c.size, c.rank
    res = {}
    t = torch.tensor([float(r + 1), -float(r)], dtype=torch.float64)
    c.allreduce(t, "min")
    res["min"] = t.tolist()
    t = torch.tensor([r + 1], dtype=torch.int32)
    c.allreduce(t, "sum")
    res["sum"] = t.tolist()
    g = torch.empty(2 * G, dtype=torch.int64)
    c.all_gather(g, torch.tensor([r, 10 * r], dtype=torch.int64))
    res["gather"] = g.tolist()
    # uneven all-to-all: rank r sends q+1 rows of value 100 r + q to rank q
    send_counts = [q + 1 for q in range(G)]
    send = torch.cat([torch.full((q + 1, 2), 100.0 * r + q, dtype=torch.float64) for q in range(G)])
    recv_counts = c.exchange_counts(send_counts)
    recv = torch.empty((sum(recv_counts), 2), dtype=torch.float64)
    c.all_to_all(recv, send, recv_counts, send_counts)
    res["recv_counts"] = recv_counts
    res["recv"] = recv[:, 0].tolist()
    res["shard"] = shard_bounds(1001, G, r)
    res["s0"] = top_split_steps(G)
    parts = [None] * G
    dist.all_gather_object(parts, res)
    if r == 0:
        Path(out).write_text(json.dumps(parts))


def engine_inputs(kind, n, m=None):
    """Sources (seed 7); with m, m separate evaluation points (uniform, seed 8)."""
    import paper_1205_4611_b200 as F
    pts = F.sample_points(F.DistributionSpec(kind, 0.01, 7), int(n))
    if m:
        ev = F.sample_points(F.DistributionSpec("uniform", 0.01, 8), int(m)).positions
        pts = F.ParticleSet(pts.positions, pts.strengths, ev)
    return pts


def engine_run(spec, out):
    import torch
    import paper_1205_4611_b200 as F
    from paper_1205_4611_b200.distributed import fmm_evaluate_distributed
    parts = spec.split(":")
    kind, n, p = parts[1], parts[2], parts[3]
    pts = engine_inputs(kind, n, parts[4] if len(parts) > 4 else None)
    cfg = F.TreeConfig(35, 0.5, int(p))
    vals, rep = fmm_evaluate_distributed(pts, cfg, device=0)
    (own, idx), _ = fmm_evaluate_distributed(pts, cfg, device=0, gather=False)
    if int(os.environ["RANK"]) == 0:
        np.savez(out, values=vals, own=own, idx=idx,
                 report=json.dumps({"levels": rep.n_levels, "totals": rep.list_totals,
                                    "skips": rep.coincident_skips,
                                    "hist": {k: {str(a): b for a, b in v.items()}
                                             for k, v in rep.list_histograms.items()}}))


def failure_inputs(case):
    """Inputs on which one rank (or every rank) must raise: 'degenerate' puts
    400 of 2000 sources on one point in the top-right corner (a level-2 box of
    one rank's subtree holds only that point; no top cut falls inside it);
    'ties' is a 39 x 40 lattice: the first median cut lies inside a column of
    40 equal x, so the quota sends only part of the column left."""
    import paper_1205_4611_b200 as F
    rng = np.random.default_rng(3)
    if case == "degenerate":
        z = rng.uniform(0.0, 1.0, 1600) + 1j * rng.uniform(0.0, 1.0, 1600)
        z = np.concatenate([z, np.full(400, 0.93 + 0.99j)])
    else:
        z = (np.arange(39)[:, None] / 39.0 + 1j * np.arange(40)[None, :] / 40.0).ravel()
    return F.ParticleSet(z, rng.uniform(-1.0, 1.0, z.size))


def raise_run(case, out):
    """Every rank must leave the evaluation with the same outcome (none may
    hang in a collective); rank 0 records all outcomes (and, on success, the
    gathered values)."""
    import torch.distributed as dist
    import paper_1205_4611_b200 as F
    from paper_1205_4611_b200.distributed import fmm_evaluate_distributed
    pts = failure_inputs(case)
    vals = None
    try:
        vals, _ = fmm_evaluate_distributed(pts, F.TreeConfig(35, 0.5, 12), device=0)
        res = None
    except Exception as e:     # noqa: BLE001 -- recorded for the test
        res = [type(e).__name__, str(e)]
    if vals is not None and int(os.environ["RANK"]) == 0:
        np.save(str(out) + ".npy", vals)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, res)
    if int(os.environ["RANK"]) == 0:
        Path(out).write_text(json.dumps(parts))


def main():
    import torch
    import torch.distributed as dist
    mode, out = sys.argv[1], sys.argv[2]
    if mode.startswith("engine-nccl"):
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
        mode = "engine" + mode[len("engine-nccl"):]
    else:
        if mode != "comm":
            torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    try:
        if mode == "comm":
            comm_checks(out)
        elif mode.startswith("raise:"):
            raise_run(mode.split(":")[1], out)
        else:
            engine_run(mode, out)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
