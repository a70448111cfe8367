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
    if off.size <= 1:
        return []
    if off.size == 2:
        return [idx]
    return np.split(idx, off[1:-1] - off[0])


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


def _csr_of(lists) -> tuple[np.ndarray, np.ndarray]:
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([np.size(a) for a in lists])
    idx = (np.concatenate([np.asarray(a, np.int64) for a in lists]) if len(lists)
           else np.zeros(0, np.int64))
    return off, np.ascontiguousarray(idx, np.int64)


def _level_geometry(lv):
    return (np.ascontiguousarray(lv.center, np.complex128),
            np.ascontiguousarray(lv.half_width, np.float64),
            np.ascontiguousarray(lv.half_height, np.float64))


def classify_level(tree: FmmTree, level: int, parent_strong: list[np.ndarray], theta: float,
                   *, device: int | None = None):
    """Split each box's inherited candidates into (strong, weak) lists
    (connectivity.py:47-68): candidates of box b are the children of the
    boxes in ``parent_strong[b // 4]``, ascending; the θ-criterion
    (bit-exact glibc hypot / numpy cabs restatement) runs on the GPU."""
    lv = tree.levels[level]
    c, hw, hh = _level_geometry(lv)
    poff, pidx = _csr_of(parent_strong)
    ncand = 16 * int(poff[-1])          # 4 children per parent, 4 candidates per entry
    woff = np.empty(lv.n_boxes + 1, np.int64)
    soff = np.empty(lv.n_boxes + 1, np.int64)
    widx = np.empty(ncand, np.int64)
    sidx = np.empty(ncand, np.int64)
    ctx = _lib.default_context(device)
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_classify_level(
            ctx.h, lv.n_boxes, _lib.dptr(c.view(np.float64)), _lib.dptr(hw), _lib.dptr(hh),
            _lib.iptr(poff), _lib.iptr(pidx), float(theta), _lib.iptr(woff), _lib.iptr(widx),
            _lib.iptr(soff), _lib.iptr(sidx)))
    strong = _split(soff, sidx[:soff[-1]])
    weak = _split(woff, widx[:woff[-1]])
    return strong, weak


def reclassify_finest(tree: FmmTree, strong: list[np.ndarray], theta: float, *,
                      device: int | None = None):
    """Refine finest strong pairs into (p2p, p2l, m2p) (connectivity.py:71-96):
    a non-self pair passing the swapped test with unequal radii moves to p2l
    (larger source) or m2p (smaller source); on the GPU."""
    lv = tree.levels[tree.n_levels]
    c, hw, hh = _level_geometry(lv)
    soff, sidx = _csr_of(strong)
    n = int(soff[-1])
    outs = [np.empty(lv.n_boxes + 1, np.int64) if k % 2 == 0 else np.empty(n, np.int64)
            for k in range(6)]
    ctx = _lib.default_context(device)
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_reclassify_finest(
            ctx.h, lv.n_boxes, _lib.dptr(c.view(np.float64)), _lib.dptr(hw), _lib.dptr(hh),
            _lib.iptr(soff), _lib.iptr(sidx), float(theta), *[_lib.iptr(a) for a in outs]))
    return tuple(_split(outs[k], outs[k + 1][:outs[k][-1]]) for k in (0, 2, 4))


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
