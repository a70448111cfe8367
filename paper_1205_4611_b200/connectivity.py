"""Interaction lists on the GPU (drop-in for ``fmm2d.connectivity``).

``build_connectivity`` uploads the tree's per-level geometry, runs the
θ-criterion classification on the B200 (csrc/connect.cu) and returns the
reference's :class:`InteractionLists` shape: directed lists, every one sorted
ascending by source box, bit-identical to connectivity.py:99-114.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np

from . import _lib
from .tree import FmmTree


@dataclass
class InteractionLists:
    """Directed interaction lists (connectivity.py:26-41)."""

    n_levels: int
    weak: list[list[np.ndarray]]
    p2p: list[np.ndarray]
    p2l: list[np.ndarray]
    m2p: list[np.ndarray]


def _split(off: np.ndarray, idx: np.ndarray) -> list[np.ndarray]:
    return np.split(idx, off[1:-1] - off[0]) if off.size > 1 else []


def export_lists(ctx: _lib.Context, n_levels: int) -> InteractionLists:
    tot = np.zeros(4, np.int64)
    ctx.check(ctx.lib.fmm2d_list_sizes(ctx.h, _lib.iptr(tot)))
    nbox = (4 ** (n_levels + 1) - 1) // 3
    nleaf = 4**n_levels
    woff = np.empty(nbox + 1, np.int64)
    widx = np.empty(tot[0], np.int64)
    arrs = []
    for q in range(1, 4):
        arrs += [np.empty(nleaf + 1, np.int64), np.empty(tot[q], np.int64)]
    ctx.check(ctx.lib.fmm2d_export_lists(ctx.h, _lib.iptr(woff), _lib.iptr(widx),
                                         *[_lib.iptr(a) for a in arrs]))
    weak = []
    base = 0
    for lev in range(n_levels + 1):
        nb = 4**lev
        off = woff[base:base + nb + 1]
        weak.append([w - base for w in _split(off, widx[off[0]:off[-1]])])
        base += nb
    p2p = _split(arrs[0], arrs[1])
    p2l = _split(arrs[2], arrs[3])
    m2p = _split(arrs[4], arrs[5])
    return InteractionLists(n_levels, weak, p2p, p2l, m2p)


def build_connectivity(tree: FmmTree, theta: float, *, device: int | None = None
                       ) -> InteractionLists:
    """Level-by-level weak/strong classification plus the finest
    reclassification, on the GPU (replaces connectivity.py:99-114)."""
    ctx = _lib.default_context(device)
    center = np.ascontiguousarray(np.concatenate([lv.center for lv in tree.levels]),
                                  dtype=np.complex128)
    hw = np.ascontiguousarray(np.concatenate([lv.half_width for lv in tree.levels]),
                              dtype=np.float64)
    hh = np.ascontiguousarray(np.concatenate([lv.half_height for lv in tree.levels]),
                              dtype=np.float64)
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_build_connectivity(
            ctx.h, int(tree.n_levels), _lib.dptr(center.view(np.float64)), _lib.dptr(hw),
            _lib.dptr(hh), float(theta)))
        return export_lists(ctx, tree.n_levels)


def write_lists_csv(lists: InteractionLists, path) -> None:
    """Dump all lists as ``level,target_box,kind,source_box`` rows
    (connectivity.py:117-131; debug I/O)."""
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["level", "target_box", "kind", "source_box"])
        for level, per_box in enumerate(lists.weak):
            for b, src in enumerate(per_box):
                out.writerows([level, b, "weak", int(a)] for a in src)
        for kind in ("p2p", "p2l", "m2p"):
            for b, src in enumerate(getattr(lists, kind)):
                out.writerows([lists.n_levels, b, kind, int(a)] for a in src)
