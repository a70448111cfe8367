"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference package read-only from /root/reference/pkg/src and
writes small .npz fixtures next to this script.  Nothing on the GPU box reads
/root/reference; the tests only read these committed files.

Canonical tree form (see oracle/fmm2d_oracle.py): per-level rectangles,
offsets and eval_perm exactly as the reference produced them, plus src_perm
with every finest box's members sorted ascending (the reference's in-box
order is an ISA-dependent artefact of np.argpartition).
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent


def canon_src_perm(tree):
    off = tree.levels[tree.n_levels].src_offsets
    out = np.array(tree.src_perm, dtype=np.int64, copy=True)
    for b in range(off.size - 1):
        out[off[b]:off[b + 1]].sort()
    return out


def flat_tree(tree):
    lv = tree.levels
    return dict(
        n_levels=np.int64(tree.n_levels),
        center=np.concatenate([l.center for l in lv]),
        half_width=np.concatenate([l.half_width for l in lv]),
        half_height=np.concatenate([l.half_height for l in lv]),
        src_offsets=np.concatenate([l.src_offsets for l in lv]),
        eval_offsets=np.concatenate([l.eval_offsets for l in lv]),
        eval_perm=np.asarray(tree.eval_perm, np.int64),
        src_perm_canon=canon_src_perm(tree),
    )


def flat_lists(lists):
    def csr(per_box):
        off = np.zeros(len(per_box) + 1, np.int64)
        off[1:] = np.cumsum([a.size for a in per_box])
        idx = np.concatenate(per_box) if per_box else np.zeros(0, np.int64)
        return off, idx.astype(np.int64)

    out = {}
    weak_all = [a for per in lists.weak for a in per]
    out["weak_off"], out["weak_idx"] = csr(weak_all)
    for k in ("p2p", "p2l", "m2p"):
        out[k + "_off"], out[k + "_idx"] = csr(getattr(lists, k))
    return out


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def main():
    sys.path.insert(0, str(REF))
    import fmm2d
    from fmm2d.datasets import DistributionSpec, sample_points
    from fmm2d.tree import ParticleSet, TreeConfig, build_tree
    from fmm2d.connectivity import build_connectivity

    cases = {}

    def pts_uniform(n, seed):
        return sample_points(DistributionSpec("uniform", seed=seed), n)

    rng12 = np.random.default_rng(12)
    sep = ParticleSet(rng12.uniform(size=4000) + 1j * rng12.uniform(size=4000),
                      rng12.uniform(-1, 1, 4000),
                      rng12.uniform(size=700) + 1j * rng12.uniform(size=700))
    rng10 = np.random.default_rng(10)
    base = rng10.uniform(size=600) + 1j * rng10.uniform(size=600)
    z = np.concatenate([base, base[:25]])
    coinc = ParticleSet(z, rng10.uniform(-1, 1, z.size))
    rng30 = np.random.default_rng(30)
    sep30 = ParticleSet(rng30.uniform(size=3000) + 1j * rng30.uniform(size=3000),
                        rng30.uniform(-1, 1, 3000),
                        rng30.uniform(size=2500) + 1j * rng30.uniform(size=2500))

    # name: (points, cfg, full)   full=False stores hashes + sampled values only
    spec = {
        "c1_uniform_1e4_p17": (pts_uniform(10_000, 0), TreeConfig(35, 0.5, 17), True),
        "normal_3000_nd40": (sample_points(DistributionSpec("normal", 0.001, 23), 3000),
                             TreeConfig(40, 0.5, 17), True),
        "separate_4000_700": (sep, TreeConfig(), True),
        "coincident_625_nd20": (coinc, TreeConfig(n_desired_per_box=20), True),
        "separate_p30_3000_2500": (sep30, TreeConfig(35, 0.5, 30), True),
        "layer_5000_p20": (sample_points(DistributionSpec("layer", 0.01, 4), 5000),
                           TreeConfig(35, 0.5, 20), True),
        "two_particles": (ParticleSet(np.array([0j, 1.0 + 0j]), np.ones(2)),
                          TreeConfig(), True),
        "four_corners_nd1": (ParticleSet(np.array([0, 1, 1j, 1 + 1j], dtype=complex),
                                         np.ones(4)), TreeConfig(n_desired_per_box=1), True),
        "uniform_1e5_p20": (pts_uniform(100_000, 0), TreeConfig(35, 0.5, 20), False),
        "normal_1e5_p20": (sample_points(DistributionSpec("normal", 0.01, 0), 100_000),
                           TreeConfig(35, 0.5, 20), False),
    }
    for name, (pts, cfg, full) in spec.items():
        tree = build_tree(pts, cfg)
        lists = build_connectivity(tree, cfg.theta)
        try:
            values, rep = fmm2d.fmm_evaluate(pts, cfg)
            error = ""
        except ValueError as exc:          # reference raises mid-pipeline
            values, rep, error = None, None, str(exc)
        ft = flat_tree(tree)
        fl = flat_lists(lists)
        rec = dict(cfg=np.array([cfg.n_desired_per_box, cfg.theta, cfg.p_terms]),
                   aliased=np.bool_(pts.evals_alias_sources),
                   error=np.str_(error),
                   tree_sha=np.str_(sha(*[ft[k] for k in sorted(ft)])),
                   lists_sha=np.str_(sha(*[fl[k] for k in sorted(fl)])))
        if rep is not None:
            rec["coincident_skips"] = np.int64(rep.coincident_skips)
            rec["n_boxes"] = np.int64(rep.n_boxes)
            for k, h in rep.list_histograms.items():
                rec[f"hist_{k}"] = np.array(sorted(h.items()), dtype=np.int64).reshape(-1, 2)
        if full:
            rec.update(ft)
            rec.update(fl)
            if values is not None:
                rec["values"] = values
            rec["positions"] = pts.positions
            rec["strengths"] = pts.strengths
            if not pts.evals_alias_sources:
                rec["eval_positions"] = pts.eval_positions
        else:
            sel = np.random.default_rng(99).choice(values.size, 2000, replace=False)
            rec["sample_idx"] = sel
            rec["sample_values"] = values[sel]
            rec["src_offsets"] = ft["src_offsets"]
            rec["n_levels"] = ft["n_levels"]
        np.savez_compressed(HERE / f"{name}.npz", **rec)
        print(name, "levels", tree.n_levels, "tree", rec["tree_sha"].item()[:12],
              "lists", rec["lists_sha"].item()[:12])

    # dataset generator fingerprints (restated in paper_1205_4611_b200.datasets)
    ds = {}
    for kind in ("uniform", "normal", "layer"):
        for seed in (0, 7):
            p = sample_points(DistributionSpec(kind, 0.01, seed), 5000)
            ds[f"{kind}_{seed}"] = sha(p.positions, p.strengths)
    np.savez(HERE / "datasets.npz", **{k: np.str_(v) for k, v in ds.items()})
    print("datasets", len(ds))


if __name__ == "__main__":
    main()
