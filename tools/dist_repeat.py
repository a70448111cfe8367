"""Repeat a distributed evaluation (gloo, all ranks on cuda:0) and report which
owned points differ from the single-GPU engine."""
import os, sys, subprocess, json
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_1205_4611_b200 as F
import _dist_worker as W
world, kind, n, p = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5])
pts = W.engine_inputs(kind, n)
ref, _ = F.fmm_evaluate(pts, F.TreeConfig(35, 0.5, p), device=0)
for r in range(reps):
    out = Path(f"/tmp/dbg_{r}.npz")
    env = dict(os.environ, PYTHONPATH=str(ROOT), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29800 + r}", str(ROOT / "tests/_dist_worker.py"),
           f"engine:{kind}:{n}:{p}", str(out)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    if res.returncode:
        print(r, "worker failed", res.stderr[-500:]); continue
    d = np.load(out)
    v = d["values"]
    rel = np.abs(v - ref) / np.abs(ref)
    bad = np.flatnonzero(rel > 1e-12)
    print(r, "max rel", float(rel.max()), "bad", bad.size, "first", bad[:10].tolist())
    if bad.size:
        own_idx = d["idx"]
        print("   rank0 owned bad:", np.isin(bad, own_idx).sum(), "of", bad.size)
