"""The reference's four experiment studies (pkg/src/fmm2d/bench.py:65-165) run
on the B200 engine through paper_1205_4611_b200.experiments; CSVs in the
reference's 10-column schema go to OUT (default gpurun_out/exp), plus a
summary JSON with device times (EngineReport.device_seconds) next to the
reference protocol's wall-clock totals."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1205_4611_b200 as F  # noqa: E402
from paper_1205_4611_b200 import experiments as X, fileio  # noqa: E402

out = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/exp")
out.mkdir(parents=True, exist_ok=True)
summary = {}
t0 = time.time()

# accuracy (Fig. 3/5): FMM vs the GPU direct sum
rows = X.run_accuracy(n=100_000, p=17) + X.run_accuracy(n=100_000, p=30)
fileio.write_benchmark(rows, out / "accuracy.csv")
summary["accuracy"] = [(r.p, r.seconds, r.tol) for r in rows if r.phase == "total"]

# calibration (Fig. 6): N_d sweep at 1e6 uniform for p = 17, 20
nds = (8, 12, 20, 35, 45, 60, 80, 120, 160)
rows = X.run_calibration(nds, n=1_000_000, p_values=(17, 20), repeats=5)
fileio.write_benchmark(rows, out / "calibration.csv")
summary["calibration_optimal"] = [(r.p, r.nd, r.levels, r.seconds) for r in rows
                                  if r.phase == "optimal"]
# device-time view of the same sweep (no host copies)
pts = F.sample_points(F.DistributionSpec("uniform", 0.01, 0), 1_000_000)
dev = {}
for p in (17, 20):
    for nd in nds:
        cfg = F.TreeConfig(nd, 0.5, p)
        F.fmm_evaluate(pts, cfg)
        ms = sorted(F.fmm_evaluate(pts, cfg)[1].device_seconds * 1e3 for _ in range(5))
        dev[f"p{p}_nd{nd}"] = ms[2]
summary["calibration_device_ms_median"] = dev

# break-even (Fig. 8): FMM vs direct per N
rows = X.run_breakeven((500, 1000, 2000, 5000, 10_000, 20_000, 50_000, 100_000), p=17,
                       repeats=5)
fileio.write_benchmark(rows, out / "breakeven.csv")
summary["breakeven"] = [(r.n, r.phase, r.seconds) for r in rows]

# adaptivity (Fig. 9): equal N under uniform / normal / layer
rows = X.run_adaptivity(n=1_000_000, p=20, repeats=5)
fileio.write_benchmark(rows, out / "adaptivity.csv")
summary["adaptivity"] = [(r.experiment, r.phase, r.seconds, r.tol) for r in rows]
summary["wall_s"] = time.time() - t0
(out / "summary.json").write_text(json.dumps(summary, indent=1))
print(json.dumps(summary, indent=1))
