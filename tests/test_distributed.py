"""Multi-rank path.

CPU (no GPU needed): the collective layer of paper_1205_4611_b200.distributed
with world_size 2 and 4 on the gloo backend.  GPU: the full distributed FMM
with 2, 4 and 8 ranks sharing cuda:0 (gloo staging) against the single-GPU
engine -- same tree, same lists, same values to roundoff."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
WORKER = ROOT / "tests" / "_dist_worker.py"


def launch(nproc, mode, out, port, timeout=600):
    env = dict(os.environ, PYTHONPATH=str(ROOT), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(WORKER), mode, str(out)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]


@pytest.mark.parametrize("world", [2, 4])
def test_comm_layer_gloo(tmp_path, world):
    out = tmp_path / "comm.json"
    launch(world, "comm", out, 29561 + world)
    parts = json.loads(out.read_text())
    for r, res in enumerate(parts):
        assert res["min"] == [1.0, -float(world - 1)]
        assert res["sum"] == [world * (world + 1) // 2]
        assert res["gather"] == [v for q in range(world) for v in (q, 10 * q)]
        # rank r receives r+1 rows from every rank q, valued 100 q + r
        assert res["recv_counts"] == [r + 1] * world
        assert res["recv"] == [100.0 * q + r for q in range(world) for _ in range(r + 1)]
        lo, hi = res["shard"]
        assert (lo, hi) == ((1001 * r) // world, (1001 * (r + 1)) // world)
        assert res["s0"] == {2: 1, 4: 2}[world]


@pytest.mark.gpu
@pytest.mark.parametrize("world,kind,n,p", [(2, "uniform", 20000, 17), (4, "normal", 30000, 20),
                                            (8, "uniform", 40000, 20), (4, "layer", 25000, 12),
                                            # owned windows large enough for the split
                                            # connectivity kernels (>= 1024 parents per rank)
                                            (2, "uniform", 400000, 17)])
def test_distributed_matches_single_gpu(tmp_path, world, kind, n, p):
    import paper_1205_4611_b200 as F
    out = tmp_path / "dist.npz"
    launch(world, f"engine:{kind}:{n}:{p}", out, 29600 + world + n % 97)
    d = np.load(out)
    pts = F.sample_points(F.DistributionSpec(kind, 0.01, 7), n)
    cfg = F.TreeConfig(35, 0.5, p)
    ref, rep = F.fmm_evaluate(pts, cfg, device=0)
    vals = d["values"]
    err = np.max(np.abs(vals - ref) / np.abs(ref))
    assert err <= 1e-13, err
    # rank 0's owned points: its subtree, values consistent with the gathered ones
    np.testing.assert_array_equal(vals[d["idx"]], d["own"])
    drep = json.loads(str(d["report"]))
    assert drep["levels"] == rep.n_levels
    assert drep["totals"] == rep.list_totals, (drep["totals"], rep.list_totals)
    assert drep["skips"] == rep.coincident_skips
    assert drep["hist"] == {k: {str(a): b for a, b in v.items()}
                            for k, v in rep.list_histograms.items()}


@pytest.mark.gpu
def test_distributed_nccl_single_rank(tmp_path):
    """The NCCL (non-staged) collective path of the distributed engine, run
    with one rank (a single-GPU box cannot host two NCCL ranks)."""
    import paper_1205_4611_b200 as F
    out = tmp_path / "nccl.npz"
    env = dict(os.environ, PYTHONPATH=str(ROOT), FMM2D_DIST_BACKEND="nccl")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29677", str(WORKER),
           "engine-nccl:uniform:30000:20", str(out)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    d = np.load(out)
    pts = F.sample_points(F.DistributionSpec("uniform", 0.01, 7), 30000)
    ref, rep = F.fmm_evaluate(pts, F.TreeConfig(35, 0.5, 20), device=0)
    assert np.max(np.abs(d["values"] - ref) / np.abs(ref)) <= 1e-13
    assert json.loads(str(d["report"]))["totals"] == rep.list_totals


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_degenerate_raises_on_every_rank(tmp_path, world):
    """A degenerate box inside ONE rank's subtree ends the evaluation on EVERY
    rank with DegenerateInputError (dist.cu error agreement) -- no
    rank blocks in a collective -- as the single-GPU engine does."""
    sys.path.insert(0, str(ROOT / "tests"))
    import _dist_worker as W
    import paper_1205_4611_b200 as F
    out = tmp_path / "raise.json"
    launch(world, "raise:degenerate", out, 29700 + world, timeout=300)
    parts = json.loads(out.read_text())
    assert all(p is not None and p[0] == "DegenerateInputError" for p in parts), parts
    assert len({p[1] for p in parts}) == 1, parts
    with pytest.raises(F.DegenerateInputError):
        F.fmm_evaluate(W.failure_inputs("degenerate"), F.TreeConfig(35, 0.5, 12), device=0)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_ties_at_a_cut_match_single_gpu(tmp_path, world):
    """A 39 x 40 lattice: the first median cut falls inside a column of equal
    x, so the reference's evaluation split (coord <= cut) differs from the
    source split.  Every rank agrees on the tie and reruns with the points as
    separate evaluation points (dist.cu:198); values equal the
    single-GPU engine's (which re-splits the same way) to roundoff."""
    sys.path.insert(0, str(ROOT / "tests"))
    import _dist_worker as W
    import paper_1205_4611_b200 as F
    out = tmp_path / "ties.json"
    launch(world, "raise:ties", out, 29710 + world, timeout=300)
    parts = json.loads(out.read_text())
    assert all(p is None for p in parts), parts
    vals = np.load(str(out) + ".npy")
    pts = W.failure_inputs("ties")
    ref, _ = F.fmm_evaluate(pts, F.TreeConfig(35, 0.5, 12), device=0)
    assert np.max(np.abs(vals - ref) / np.abs(ref)) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("world,kind,n,m,p", [(2, "uniform", 20000, 15000, 20),
                                              (4, "normal", 30000, 24000, 30),
                                              (8, "uniform", 40000, 9000, 17)])
def test_distributed_separate_evaluation_points(tmp_path, world, kind, n, m, p):
    """Separate evaluation points (the C4 shape) across ranks: routed to the
    rank owning their top-split segment by coord <= cut, evaluated there, values
    gathered in input order -- equal to the single-GPU engine to roundoff, with
    the same list totals and coincident-skip count."""
    sys.path.insert(0, str(ROOT / "tests"))
    import _dist_worker as W
    import paper_1205_4611_b200 as F
    out = tmp_path / "sep.npz"
    launch(world, f"engine:{kind}:{n}:{p}:{m}", out, 29720 + world + n % 89)
    d = np.load(out)
    pts = W.engine_inputs(kind, n, m)
    ref, rep = F.fmm_evaluate(pts, F.TreeConfig(35, 0.5, p), device=0)
    vals = d["values"]
    assert vals.shape == (m,)
    assert np.max(np.abs(vals - ref) / np.abs(ref)) <= 1e-13
    np.testing.assert_array_equal(vals[d["idx"]], d["own"])
    drep = json.loads(str(d["report"]))
    assert drep["totals"] == rep.list_totals
    assert drep["skips"] == rep.coincident_skips


@pytest.mark.gpu
def test_distributed_matches_oracle(tmp_path):
    """4 ranks against the CPU oracle directly (not only against the GPU
    engine): potentials <= 1e-12 relative on normal inputs."""
    sys.path.insert(0, str(ROOT))
    from oracle import fmm2d_oracle as O
    out = tmp_path / "orc.npz"
    launch(4, "engine:normal:30000:20", out, 29740)
    d = np.load(out)
    sys.path.insert(0, str(ROOT / "tests"))
    import _dist_worker as W
    pts = W.engine_inputs("normal", 30000)
    ref, _, _, _ = O.fmm(pts.positions, pts.strengths, None, 35, 0.5, 20)
    assert O.max_rel(d["values"], ref) <= 1e-12
