"""Shared test helpers: canonical forms, fingerprints, fixtures loading."""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

FULL_CASES = ["c1_uniform_1e4_p17", "normal_3000_nd40", "separate_4000_700",
              "coincident_625_nd20", "separate_p30_3000_2500", "layer_5000_p20",
              "two_particles", "four_corners_nd1"]
SAMPLED_CASES = ["uniform_1e5_p20", "normal_1e5_p20"]
TIE_CASES = {"coincident_625_nd20"}   # ties at cuts: in-box membership is ISA dependent


def load(name):
    return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def canon_src_perm(src_off_finest, src_perm):
    out = np.array(src_perm, dtype=np.int64, copy=True)
    off = np.asarray(src_off_finest)
    for b in range(off.size - 1):
        out[off[b]:off[b + 1]].sort()
    return out


def flat_tree_pkg(tree):
    """Flatten an FmmTree (package or reference layout)."""
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


def flat_tree_oracle(T):
    return dict(
        n_levels=np.int64(T.n_levels),
        center=np.concatenate(T.center),
        half_width=np.concatenate(T.hw),
        half_height=np.concatenate(T.hh),
        src_offsets=np.concatenate(T.src_off).astype(np.int64),
        eval_offsets=np.concatenate(T.eval_off).astype(np.int64),
        eval_perm=np.asarray(T.eval_perm, np.int64),
        src_perm_canon=canon_src_perm(T.src_off[T.n_levels], T.src_perm),
    )


def _csr(per_box):
    off = np.zeros(len(per_box) + 1, np.int64)
    off[1:] = np.cumsum([a.size for a in per_box])
    idx = np.concatenate(per_box) if per_box else np.zeros(0, np.int64)
    return off, idx.astype(np.int64)


def flat_lists_pkg(lists):
    out = {}
    out["weak_off"], out["weak_idx"] = _csr([a for per in lists.weak for a in per])
    for k in ("p2p", "p2l", "m2p"):
        out[k + "_off"], out[k + "_idx"] = _csr(getattr(lists, k))
    return out


def flat_lists_oracle(Ls):
    weak = []
    for lev in range(Ls.n_levels + 1):
        off, idx = Ls.weak_off[lev], Ls.weak_idx[lev]
        weak += [idx[off[b]:off[b + 1]] for b in range(off.size - 1)]
    out = {}
    out["weak_off"], out["weak_idx"] = _csr(weak)
    for k in ("p2p", "p2l", "m2p"):
        off, idx = getattr(Ls, k + "_off"), getattr(Ls, k + "_idx")
        out[k + "_off"], out[k + "_idx"] = _csr([idx[off[b]:off[b + 1]]
                                                for b in range(off.size - 1)])
    return out


TREE_KEYS = ["center", "eval_offsets", "eval_perm", "half_height", "half_width", "n_levels",
             "src_offsets", "src_perm_canon"]
LIST_KEYS = ["m2p_idx", "m2p_off", "p2l_idx", "p2l_off", "p2p_idx", "p2p_off", "weak_idx",
             "weak_off"]


def tree_sha(flat):
    return sha(*[flat[k] for k in sorted(flat)])


def assert_tree_equal(got, want, ties=False):
    for k in TREE_KEYS:
        if ties and k == "src_perm_canon":
            continue
        g, w = np.asarray(got[k]), np.asarray(want[k])
        assert g.shape == w.shape, (k, g.shape, w.shape)
        assert np.array_equal(g, w), f"tree field {k} differs"


def assert_lists_equal(got, want):
    for k in LIST_KEYS:
        g, w = np.asarray(got[k]), np.asarray(want[k])
        assert g.shape == w.shape and np.array_equal(g, w), f"list field {k} differs"


def points_from(rec):
    from paper_1205_4611_b200 import ParticleSet
    ev = rec.get("eval_positions")
    return ParticleSet(rec["positions"], rec["strengths"], ev)


def cfg_from(rec):
    from paper_1205_4611_b200 import TreeConfig
    nd, theta, p = rec["cfg"]
    return TreeConfig(int(nd), float(theta), int(p))


def max_rel(a, e):
    a, e = np.asarray(a), np.asarray(e)
    ok = e != 0
    return float(np.max(np.abs(a[ok] - e[ok]) / np.abs(e[ok])))
