"""Golden vectors for the direct sum, symmetric and asymmetric modes, made by
running the REFERENCE's ``direct_evaluate`` (engine.py:282-323) read-only
from /root/reference/pkg/src in the build container:
    python tests/golden/make_golden_direct.py
Inputs are the reference's own generator draws (datasets.sample_points) plus
a set with coincident points (exact duplicates: the skip rule), stored with
the outputs so the GPU tests need nothing else.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent


def main() -> None:
    sys.path.insert(0, str(REF))
    import fmm2d as R

    cases = {}
    pts = R.sample_points(R.DistributionSpec("uniform", 0.01, 3), 3000)
    cases["uniform_3000"] = pts
    pts = R.sample_points(R.DistributionSpec("normal", 0.01, 4), 2500)
    # duplicates: 200 points repeated, one repeated three times
    pos = np.concatenate([pts.positions, pts.positions[:200], pts.positions[:1]])
    g = np.concatenate([pts.strengths, pts.strengths[:200] * 0.5, [0.25]])
    cases["normal_dup_2701"] = R.ParticleSet(pos, g)
    out = {}
    for name, p in cases.items():
        out[f"{name}_positions"] = p.positions
        out[f"{name}_strengths"] = p.strengths
        out[f"{name}_symmetric"] = R.direct_evaluate(p, symmetric=True)
        out[f"{name}_asymmetric"] = R.direct_evaluate(p)
    np.savez_compressed(HERE / "direct_sum.npz", **out)
    print("wrote", HERE / "direct_sum.npz")


if __name__ == "__main__":
    main()
