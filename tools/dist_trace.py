"""Where does the distributed engine's time go at one rank?  Runs
evaluate_shard at C2 (1 rank, NCCL) with every library call and collective
wrapped: the stream is synchronised after each and its wall time recorded.
Prints per-call totals (ms) over one evaluation, after warm-up, next to the
untraced CUDA-event time of the same evaluation."""
import collections
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1205_4611_b200 as F  # noqa: E402
from paper_1205_4611_b200 import _lib  # noqa: E402
from paper_1205_4611_b200 import distributed as D  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
pts = F.sample_points(F.DistributionSpec("uniform", 0.01, 0), n)
cfg = F.TreeConfig(35, 0.5, 20)
st = D.engine_stream(0)
ctx = _lib.default_context(0)
comm = D.Comm()
with torch.cuda.stream(st):
    d_pos = torch.from_numpy(pts.positions.view(np.float64).reshape(-1, 2)).to(dev)
    d_g = torch.from_numpy(pts.strengths.copy()).to(dev)
T = collections.defaultdict(float)
C = collections.Counter()


class LibProxy:
    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if not name.startswith("fmm2d_") or not TRACE[0]:
            return f

        def g(*a):
            t0 = time.perf_counter()
            r = f(*a)
            st.synchronize()
            T[name] += (time.perf_counter() - t0) * 1e3
            C[name] += 1
            return r
        return g


TRACE = [False]
for meth in ("exchange_counts", "all_to_all", "all_gather", "allreduce"):
    orig = getattr(comm, meth)

    def wrap(*a, _o=orig, _m=meth, **k):
        if not TRACE[0]:
            return _o(*a, **k)
        t0 = time.perf_counter()
        r = _o(*a, **k)
        st.synchronize()
        T["comm." + _m] += (time.perf_counter() - t0) * 1e3
        C["comm." + _m] += 1
        return r
    setattr(comm, meth, wrap)
real_lib = ctx.lib
ctx.lib = LibProxy(real_lib)


def once(trace):
    TRACE[0] = trace
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        t0 = time.perf_counter()
        e0.record(st)
        try:
            D.evaluate_shard(ctx, comm, n, d_pos, d_g, 0, cfg)
        finally:
            real_lib.fmm2d_dist_end(ctx.h)
        e1.record(st)
    st.synchronize()
    return e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3


for _ in range(3):
    once(False)
ev, wall = once(False)
print(f"untraced: event {ev:.3f} ms, wall {wall:.3f} ms")
T.clear(); C.clear()
ev, wall = once(True)
print(f"traced: wall {wall:.3f} ms, sum of traced calls {sum(T.values()):.3f} ms")
for k, v in sorted(T.items(), key=lambda kv: -kv[1]):
    print(f"  {k:32s} x{C[k]:3d} {v:8.3f} ms")
# single-GPU engine for comparison
vals, rep = F.fmm_evaluate(pts, cfg)
ts = []
for _ in range(5):
    vals, rep = F.fmm_evaluate(pts, cfg)
    ts.append(rep.device_seconds * 1e3)
print(f"single-GPU device ms: {min(ts):.3f}")
dist.destroy_process_group()
