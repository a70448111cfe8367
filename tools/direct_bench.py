"""Direct-sum timing on the GPU: asymmetric (IEEE 1/r2, thread per target)
vs symmetric (shared reciprocal, k_direct_sym + fold), end to end through
direct_evaluate, plus their agreement.  Usage: python tools/direct_bench.py [n ...]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1205_4611_b200 as F  # noqa: E402

sizes = [int(float(a)) for a in sys.argv[1:]] or [100_000, 300_000, 1_000_000]
for n in sizes:
    pts = F.sample_points(F.DistributionSpec("uniform", 0.01, 0), n)
    row = {"n": n}
    out = {}
    for sym in (False, True):
        F.direct_evaluate(pts, symmetric=sym)                 # warm (allocations)
        reps = 3 if n <= 300_000 else 1
        t0 = time.perf_counter()
        for _ in range(reps):
            out[sym] = F.direct_evaluate(pts, symmetric=sym)
        dt = (time.perf_counter() - t0) / reps
        key = "symmetric" if sym else "asymmetric"
        row[key + "_s"] = round(dt, 5)
        row[key + "_Ginteractions_per_s"] = round(n * n / dt / 1e9, 1)
    row["max_rel_sym_vs_asym"] = F.max_rel_error(out[True], out[False])
    row["speedup"] = round(row["asymmetric_s"] / row["symmetric_s"], 3)
    print(json.dumps(row), flush=True)
