"""Tree types and the GPU tree build (drop-in for ``fmm2d.tree``).

The dataclasses keep the reference's names, fields and validation messages
(tree.py:20-334).  ``build_tree`` runs the median-split pyramid on the B200
(csrc/tree.cu) and returns the canonical tree: offsets, rectangles and
``eval_perm`` are bit-identical to the reference, and inside every finest box
the sources are in ascending original index (the reference's within-box order
is an ISA-dependent by-product of ``np.argpartition``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import Box


class DegenerateInputError(ValueError):
    """All points in a box coincide while further levels are still required
    (tree.py:20-21)."""


@dataclass
class ParticleSet:
    """Sources with real strengths plus evaluation points (tree.py:24-66).

    ``eval_positions=None`` makes the evaluation points alias the sources.
    """

    positions: np.ndarray
    strengths: np.ndarray
    eval_positions: np.ndarray | None = None

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.complex128)
        self.strengths = np.ascontiguousarray(self.strengths, dtype=np.float64)
        if self.eval_positions is None or self.eval_positions is self.positions:
            self.eval_positions = self.positions
        else:
            self.eval_positions = np.ascontiguousarray(self.eval_positions,
                                                       dtype=np.complex128)
        if self.positions.ndim != 1 or self.positions.size < 1:
            raise ValueError("positions must be a non-empty 1-d complex array")
        if self.strengths.shape != self.positions.shape:
            raise ValueError("strengths must be index-aligned with positions")
        if not np.isfinite(self.strengths).all():
            raise ValueError("strengths must be finite")
        for name in ("positions", "eval_positions"):
            arr = getattr(self, name)
            if not (np.isfinite(arr.real).all() and np.isfinite(arr.imag).all()):
                raise ValueError(f"{name} must be finite")

    @property
    def n_sources(self) -> int:
        return self.positions.size

    @property
    def n_evals(self) -> int:
        return self.eval_positions.size

    @property
    def evals_alias_sources(self) -> bool:
        return self.eval_positions is self.positions


@dataclass(frozen=True)
class TreeConfig:
    """N_d, θ and p (tree.py:69-83); defaults 35, 0.5, 17."""

    n_desired_per_box: int = 35
    theta: float = 0.5
    p_terms: int = 17

    def __post_init__(self):
        if self.n_desired_per_box < 1:
            raise ValueError("n_desired_per_box must be >= 1")
        if not 0.0 < self.theta < 1.0:
            raise ValueError("theta must lie in (0, 1)")
        if self.p_terms < 1:
            raise ValueError("p_terms must be >= 1")


def num_levels(n_sources: int, n_desired: int) -> int:
    """Eq. (6): max(0, ceil(0.5*log2((5/8)*n_sources/n_desired))) (tree.py:86-94)."""
    if n_sources < 1 or n_desired < 1:
        raise ValueError("n_sources and n_desired must be >= 1")
    return max(0, math.ceil(0.5 * math.log2(0.625 * n_sources / n_desired)))


def clamped_levels(n_sources: int, n_desired: int) -> int:
    """Depth actually built: Eq. (6) clamped so 4**L <= N (tree.py:186-192)."""
    lev = num_levels(n_sources, n_desired)
    while lev > 0 and 4**lev > n_sources:
        lev -= 1
    return lev


def partition_median(coords: np.ndarray, *companions: np.ndarray) -> int:
    """In-place median partition of a host array (tree.py:97-114).

    Same contract as the reference (left part holds ceil(n/2) elements, all
    <= the right part; companions follow), realised with the engine's
    canonical rule: a stable partition that keeps ties in input order.  Host
    utility; the GPU tree build does not call it.
    """
    n = coords.shape[0]
    if n < 1:
        raise ValueError("cannot partition an empty array")
    k = (n + 1) // 2
    if n > 1:
        order = np.argsort(coords, kind="stable")
        left = np.zeros(n, dtype=bool)
        left[order[:k]] = True
        perm = np.concatenate([np.flatnonzero(left), np.flatnonzero(~left)])
        coords[:] = coords[perm]
        for comp in companions:
            comp[:] = comp[perm]
    return k


@dataclass
class LevelBoxes:
    """Struct-of-arrays for one level, all of length 4**l (tree.py:117-140)."""

    center: np.ndarray
    half_width: np.ndarray
    half_height: np.ndarray
    src_offsets: np.ndarray
    eval_offsets: np.ndarray

    @property
    def n_boxes(self) -> int:
        return self.center.size

    def boxes(self) -> Box:
        return Box(self.center, self.half_width, self.half_height)

    def src_counts(self) -> np.ndarray:
        return np.diff(self.src_offsets)

    def eval_counts(self) -> np.ndarray:
        return np.diff(self.eval_offsets)


@dataclass(frozen=True)
class BoxNode:
    """Single-box view (tree.py:142-151)."""

    geometry: Box
    src_begin: int
    src_end: int
    eval_begin: int
    eval_end: int


@dataclass
class FmmTree:
    """Pyramid tree over permuted point arrays (tree.py:153-183)."""

    n_levels: int
    levels: list[LevelBoxes] = field(repr=False)
    src_pos: np.ndarray = field(repr=False)
    src_strength: np.ndarray = field(repr=False)
    eval_pos: np.ndarray = field(repr=False)
    src_perm: np.ndarray = field(repr=False)
    eval_perm: np.ndarray = field(repr=False)

    @property
    def finest(self) -> LevelBoxes:
        return self.levels[self.n_levels]

    def box(self, level: int, k: int) -> BoxNode:
        lv = self.levels[level]
        return BoxNode(
            geometry=Box(lv.center[k], float(lv.half_width[k]), float(lv.half_height[k])),
            src_begin=int(lv.src_offsets[k]),
            src_end=int(lv.src_offsets[k + 1]),
            eval_begin=int(lv.eval_offsets[k]),
            eval_end=int(lv.eval_offsets[k + 1]),
        )


def _level_slices(n_levels: int):
    box0 = 0
    off0 = 0
    for lev in range(n_levels + 1):
        nb = 4**lev
        yield lev, slice(box0, box0 + nb), slice(off0, off0 + nb + 1)
        box0 += nb
        off0 += nb + 1


def export_tree(ctx: _lib.Context, n_levels: int, n: int, m: int) -> FmmTree:
    """Copy the context's device tree into reference-shaped numpy arrays."""
    nbox = (4 ** (n_levels + 1) - 1) // 3
    noff = nbox + n_levels + 1
    center = np.empty(nbox, np.complex128)
    hw = np.empty(nbox)
    hh = np.empty(nbox)
    soff = np.empty(noff, np.int64)
    eoff = np.empty(noff, np.int64)
    sperm = np.empty(n, np.int64)
    eperm = np.empty(m, np.int64)
    spos = np.empty(n, np.complex128)
    sg = np.empty(n)
    epos = np.empty(m, np.complex128)
    ctx.check(ctx.lib.fmm2d_export_tree(
        ctx.h, _lib.dptr(center.view(np.float64)), _lib.dptr(hw), _lib.dptr(hh),
        _lib.iptr(soff), _lib.iptr(eoff), _lib.iptr(sperm), _lib.iptr(eperm),
        _lib.dptr(spos.view(np.float64)), _lib.dptr(sg), _lib.dptr(epos.view(np.float64))))
    levels = [LevelBoxes(center[bs].copy(), hw[bs].copy(), hh[bs].copy(), soff[os].copy(),
                         eoff[os].copy()) for _, bs, os in _level_slices(n_levels)]
    return FmmTree(n_levels, levels, spos, sg, epos, sperm, eperm)


def build_tree(points: ParticleSet, cfg: TreeConfig, *, device: int | None = None) -> FmmTree:
    """Build the pyramid tree on the GPU (replaces tree.py:230-334).

    Raises :class:`DegenerateInputError` when a box whose points all coincide
    must be split further.
    """
    ctx = _lib.default_context(device)
    pos = points.positions
    epos = None if points.evals_alias_sources else points.eval_positions
    lev = np.zeros(1, np.int32)
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_build_tree(
            ctx.h, pos.size, _lib.dptr(pos.view(np.float64)), _lib.dptr(points.strengths),
            points.n_evals, None if epos is None else _lib.dptr(epos.view(np.float64)),
            int(cfg.n_desired_per_box), lev.ctypes.data_as(_lib.C.POINTER(_lib.C.c_int32))))
        return export_tree(ctx, int(lev[0]), points.n_sources, points.n_evals)
