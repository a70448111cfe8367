"""Where does the C5 (1e7) deviation from the reference come from?
Prints the max relative error at the golden's sampled points, the number of
points above 1e-12, and the same for the reference's own ISA variant.
Run variants through FMM2D_LIBRARY / FMM2D_M2L."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1205_4611_b200 as F  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_uniform_1e7_p20"
rec = dict(np.load(ROOT / "tests/golden" / f"{name}.npz"))
isa = dict(np.load(ROOT / "tests/golden" / f"{name}_isa.npz"))
n = int(rec["n_sources"])
p = int(rec["cfg"][2])
pts = F.sample_points(F.DistributionSpec(str(rec["kind"]), 0.01, 0), n)
values, _ = F.fmm_evaluate(pts, F.TreeConfig(35, 0.5, p))
idx, want = rec["sample_idx"], rec["sample_values"]
rel = np.abs(values[idx] - want) / np.abs(want)
rel_isa = np.abs(isa["sample_values_isa"] - want) / np.abs(want)
tag = os.environ.get("FMM2D_LIBRARY", "base") + " M2L=" + os.environ.get("FMM2D_M2L", "dense")
print(f"{tag}: max {rel.max():.3e} (>1e-12: {(rel > 1e-12).sum()}, >5e-13: {(rel > 5e-13).sum()}) "
      f"| ISA floor {rel_isa.max():.3e} (>1e-12: {(rel_isa > 1e-12).sum()}, >5e-13: "
      f"{(rel_isa > 5e-13).sum()}) | worst idx {idx[rel.argmax()]} |phi|={abs(want[rel.argmax()]):.3g}")
# GPU vs ISA-variant reference at the same points
rel_gi = np.abs(values[idx] - isa["sample_values_isa"]) / np.abs(want)
print(f"   vs ISA-variant reference: max {rel_gi.max():.3e}")
