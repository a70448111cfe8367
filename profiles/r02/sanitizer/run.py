import sys
sys.path.insert(0, ".")
import os
os.environ.setdefault("FMM2D_GRAPHS", "0")
import paper_1205_4611_b200 as F
pts = F.sample_points(F.DistributionSpec("uniform", seed=0), 10_000)
for p in (17, 30):
    v, r = F.fmm_evaluate(pts, F.TreeConfig(35, 0.5, p))
ev = F.sample_points(F.DistributionSpec("normal", seed=3), 4_000)
sep = F.ParticleSet(pts.positions, pts.strengths, ev.positions)
v, r = F.fmm_evaluate(sep, F.TreeConfig(35, 0.5, 20))
print("ok", r.n_levels)
