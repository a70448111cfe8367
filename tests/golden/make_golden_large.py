"""Generate headline-config golden fixtures (C2-C5) by running the REFERENCE.

Run in the build container (where /root/reference exists), one config per
process so they can run side by side:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py c2
    ... c3 | c4 | c5

Each config runs the reference's public ``fmm2d.fmm_evaluate`` once
(sequential, ``parallel=False``) on the bench's exact inputs
(``sample_points`` Philox seed 0; C4 evals from seed 1), capturing the tree
and the interaction lists the engine builds internally (the reference's own
``build_tree`` / ``build_connectivity`` objects, engine.py:220-225).  A full
dump at 1e6-1e7 points is hundreds of MB, so the fixture stores:

* one SHA-256 per canonical tree field and per CSR list field (same
  canonicalisation as make_golden.py: per-level rects, offsets, eval_perm,
  src_perm with each finest box's members sorted),
* the list-length histograms, coincident_skips and n_boxes of the report,
* sampled potentials: 10,000 uniformly drawn evaluation points plus the
  2,000 points of smallest |phi| (the ill-conditioned, cancellation-heavy
  ones where a 1e-12 relative bound is hardest to meet).

The GPU tests (tests/test_gpu_headline.py) recompute the same hashes from
the GPU's exported tree/lists and compare the sampled potentials.
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent

CONFIGS = {
    # name: (kind, n, n_eval_separate (0 = alias), p, fixture name)
    "c2": ("uniform", 1_000_000, 0, 20, "c2_uniform_1e6_p20"),
    "c3": ("normal", 1_000_000, 0, 20, "c3_normal_1e6_p20"),
    "c4": ("uniform", 1_000_000, 1_000_000, 30, "c4_separate_1e6_p30"),
    "c5": ("uniform", 10_000_000, 0, 20, "c5_uniform_1e7_p20"),
}


def sha(a) -> str:
    h = hashlib.sha256()
    a = np.ascontiguousarray(a)
    h.update(str(a.dtype).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def canon_src_perm(src_off_finest, src_perm):
    """Sort every finest box's members ascending (vectorised)."""
    off = np.asarray(src_off_finest, np.int64)
    perm = np.asarray(src_perm, np.int64)
    box = np.repeat(np.arange(off.size - 1), np.diff(off))
    return perm[np.lexsort((perm, box))]


def tree_fields(tree):
    lv = tree.levels
    return dict(
        n_levels=np.int64(tree.n_levels),
        center=np.concatenate([l.center for l in lv]),
        half_width=np.concatenate([l.half_width for l in lv]),
        half_height=np.concatenate([l.half_height for l in lv]),
        src_offsets=np.concatenate([l.src_offsets for l in lv]).astype(np.int64),
        eval_offsets=np.concatenate([l.eval_offsets for l in lv]).astype(np.int64),
        eval_perm=np.asarray(tree.eval_perm, np.int64),
        src_perm_canon=canon_src_perm(lv[tree.n_levels].src_offsets, tree.src_perm),
    )


def csr(per_box):
    off = np.zeros(len(per_box) + 1, np.int64)
    off[1:] = np.cumsum([a.size for a in per_box])
    idx = np.concatenate(per_box).astype(np.int64) if len(per_box) else np.zeros(0, np.int64)
    return off, idx


def list_fields(lists):
    out = {}
    out["weak_off"], out["weak_idx"] = csr([a for per in lists.weak for a in per])
    for k in ("p2p", "p2l", "m2p"):
        out[k + "_off"], out[k + "_idx"] = csr(getattr(lists, k))
    return out


def inputs(name):
    sys.path.insert(0, str(REF))
    from fmm2d.datasets import DistributionSpec, sample_points
    from fmm2d.tree import ParticleSet
    kind, n, m, p, _ = CONFIGS[name]
    pts = sample_points(DistributionSpec(kind, 0.01, 0), n)
    if m:
        ev = sample_points(DistributionSpec("uniform", 0.01, 1), m).positions
        pts = ParticleSet(pts.positions, pts.strengths, ev)
    return pts, p


def main(name):
    sys.path.insert(0, str(REF))
    import fmm2d
    import fmm2d.engine as eng
    from fmm2d.tree import TreeConfig

    pts, p = inputs(name)
    cfg = TreeConfig(35, 0.5, p)
    captured = {}
    orig_tree, orig_conn = eng.build_tree, eng.build_connectivity

    def cap_tree(points, c):
        captured["tree"] = orig_tree(points, c)
        return captured["tree"]

    def cap_conn(tree, theta):
        captured["lists"] = orig_conn(tree, theta)
        return captured["lists"]

    eng.build_tree, eng.build_connectivity = cap_tree, cap_conn
    t0 = time.perf_counter()
    values, rep = fmm2d.fmm_evaluate(pts, cfg)
    wall = time.perf_counter() - t0
    eng.build_tree, eng.build_connectivity = orig_tree, orig_conn

    ft = tree_fields(captured["tree"])
    fl = list_fields(captured["lists"])
    rec = dict(cfg=np.array([35, 0.5, p]), aliased=np.bool_(pts.evals_alias_sources),
               kind=np.str_(CONFIGS[name][0]), n_sources=np.int64(pts.n_sources),
               n_evals=np.int64(pts.n_evals), ref_wall_s=np.float64(wall))
    for k, v in ft.items():
        rec["tree_sha_" + k] = np.str_(sha(v))
    for k, v in fl.items():
        rec["lists_sha_" + k] = np.str_(sha(v))
    rec["n_levels"] = ft["n_levels"]
    rec["coincident_skips"] = np.int64(rep.coincident_skips)
    rec["n_boxes"] = np.int64(rep.n_boxes)
    rec["finest_src_min"] = np.int64(rep.finest_src_min)
    rec["finest_src_max"] = np.int64(rep.finest_src_max)
    for k, h in rep.list_histograms.items():
        rec[f"hist_{k}"] = np.array(sorted(h.items()), dtype=np.int64).reshape(-1, 2)
    rng = np.random.default_rng(99)
    rand = rng.choice(values.size, 10_000, replace=False)
    small = np.argsort(np.abs(values), kind="stable")[:2000]
    sel = np.unique(np.concatenate([rand, small]))
    rec["sample_idx"] = sel.astype(np.int64)
    rec["sample_values"] = values[sel]
    rec["phase_seconds"] = np.array([rep.phase_seconds[k] for k in eng.PHASE_NAMES])
    fix = CONFIGS[name][4]
    np.savez_compressed(HERE / f"{fix}.npz", **rec)
    print(fix, "levels", int(ft["n_levels"]), "wall %.1f s" % wall,
          "tree", sha(np.concatenate([np.frombuffer(rec["tree_sha_" + k].item().encode(), np.uint8)
                                      for k in sorted(ft)]))[:12])


def isa_variant(name):
    """Re-run the reference on the same input with numpy's SIMD dispatch
    disabled (the caller sets NPY_DISABLE_CPU_FEATURES / OPENBLAS_CORETYPE as
    in SURVEY Appendix B) and store its potentials at the fixture's sampled
    points: the reference's own same-input ISA floor, point by point."""
    sys.path.insert(0, str(REF))
    import fmm2d
    from fmm2d.tree import TreeConfig
    fix = CONFIGS[name][4]
    rec = dict(np.load(HERE / f"{fix}.npz"))
    pts, p = inputs(name)
    values, _ = fmm2d.fmm_evaluate(pts, TreeConfig(35, 0.5, p))
    idx = rec["sample_idx"]
    np.savez_compressed(HERE / f"{fix}_isa.npz", sample_idx=idx, sample_values_isa=values[idx])
    rel = np.abs(values[idx] - rec["sample_values"]) / np.abs(rec["sample_values"])
    print(fix, "ISA floor at the sampled points: max rel %.3e" % rel.max())


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--isa-variant":
        for nm in args[1:]:
            isa_variant(nm)
    else:
        for nm in args or list(CONFIGS):
            main(nm)
