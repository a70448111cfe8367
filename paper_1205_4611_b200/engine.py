"""The FMM evaluation entry point (drop-in for ``fmm2d.engine``).

``fmm_evaluate`` keeps the reference signature and return shape
(engine.py:207-279): ``(values, EngineReport)`` with values in the original
input order.  Every phase -- tree build, connectivity, P2M/P2L, M2M, M2L,
L2L, L2P/M2P, P2P, un-permute -- runs as sm_100a kernels in libfmm2d.so on
one CUDA stream; ``phase_seconds`` are CUDA-event times of those phases and
``other`` holds the host<->device copies and call overhead.  ``parallel`` and
``n_workers`` are accepted for signature compatibility (the GPU grid replaces
the reference's thread pool, engine.py:50-64).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .tree import ParticleSet, TreeConfig

PHASE_NAMES = ("sort", "connect", "p2m", "m2m", "m2l", "l2l", "l2p", "p2p", "other")
_KINDS = ("weak", "p2p", "p2l", "m2p")


@dataclass
class EngineReport:
    """Per-phase times plus tree and list statistics (engine.py:34-47)."""

    phase_seconds: dict[str, float]
    total_seconds: float
    n_levels: int
    n_boxes: int
    finest_src_min: int
    finest_src_max: int
    finest_src_mean: float
    list_histograms: dict[str, dict[int, int]] = field(default_factory=dict)
    coincident_skips: int = 0
    parallel: bool = False
    # B200 extras
    device_seconds: float = 0.0
    list_totals: dict[str, int] = field(default_factory=dict)
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    retries: int = 0
    kernel_launches: int = 0


def _histograms(ctx: _lib.Context, rep: _lib.Report) -> dict[str, dict[int, int]]:
    out = {}
    for k, name in enumerate(_KINDS):
        nb = int(rep.max_len[k]) + 1
        h = np.zeros(nb, np.int64)
        ctx.check(ctx.lib.fmm2d_histogram(ctx.h, k, _lib.iptr(h), nb))
        nz = np.flatnonzero(h)
        out[name] = dict(zip(nz.tolist(), h[nz].tolist()))
    return out


def _report(ctx, rep: _lib.Report, wall: float, points_alias: bool, m: int, parallel: bool,
            histograms: bool = True) -> EngineReport:
    ms = list(rep.phase_ms)
    phases = {name: ms[i] * 1e-3 for i, name in enumerate(PHASE_NAMES[:-1])}
    phases["other"] = max(0.0, wall - sum(phases.values()))
    expected_self = m if points_alias else 0
    return EngineReport(
        phase_seconds=phases,
        total_seconds=wall,
        n_levels=int(rep.n_levels),
        n_boxes=int(rep.n_boxes),
        finest_src_min=int(rep.finest_src_min),
        finest_src_max=int(rep.finest_src_max),
        finest_src_mean=float(rep.finest_src_mean),
        list_histograms=_histograms(ctx, rep) if histograms else {},
        coincident_skips=max(0, int(rep.p2p_skips) - expected_self),
        parallel=bool(parallel),
        device_seconds=rep.device_ms * 1e-3,
        list_totals={name: int(rep.list_totals[k]) for k, name in enumerate(_KINDS)},
        h2d_bytes=int(rep.h2d_bytes),
        d2h_bytes=int(rep.d2h_bytes),
        retries=int(rep.retries),
        kernel_launches=int(rep.kernel_launches),
    )


def fmm_evaluate(points: ParticleSet, cfg: TreeConfig | None = None, *, parallel: bool = False,
                 n_workers: int | None = None, device: int | None = None,
                 out: np.ndarray | None = None):
    """Evaluate the potential at all evaluation points on the GPU.

    Returns ``(values, report)`` with values in the original input order.
    ``out`` may supply a preallocated complex128[M] (e.g. pinned) buffer.
    """
    t0 = time.perf_counter()
    cfg = cfg or TreeConfig()
    del n_workers
    ctx = _lib.default_context(device)
    pos = points.positions
    alias = points.evals_alias_sources
    epos = None if alias else points.eval_positions
    m = points.n_evals
    if out is None:
        out = np.empty(m, dtype=np.complex128)
    elif out.dtype != np.complex128 or out.shape != (m,) or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous complex128 array of length n_evals")
    rep = _lib.Report()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_evaluate(
            ctx.h, pos.size, _lib.dptr(pos.view(np.float64)), _lib.dptr(points.strengths), m,
            None if epos is None else _lib.dptr(epos.view(np.float64)), int(cfg.p_terms),
            float(cfg.theta), int(cfg.n_desired_per_box), _lib.dptr(out.view(np.float64)),
            _lib.C.byref(rep)))
        wall = time.perf_counter() - t0
        report = _report(ctx, rep, wall, alias, m, parallel)
    report.total_seconds = time.perf_counter() - t0
    return out, report


def fmm_evaluate_device(n: int, d_pos: int, d_gamma: int, m: int, d_eval: int | None,
                        d_out: int, cfg: TreeConfig | None = None, *, device: int | None = None,
                        histograms: bool = False):
    """Device-resident variant: raw CUDA pointers in and out (bench helper).

    ``d_eval=None`` aliases the evaluation points to the sources.
    """
    cfg = cfg or TreeConfig()
    ctx = _lib.default_context(device)
    rep = _lib.Report()
    t0 = time.perf_counter()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_evaluate_device(
            ctx.h, int(n), _lib.C.c_void_p(d_pos), _lib.C.c_void_p(d_gamma), int(m),
            None if d_eval is None else _lib.C.c_void_p(d_eval), int(cfg.p_terms),
            float(cfg.theta), int(cfg.n_desired_per_box), _lib.C.c_void_p(d_out),
            _lib.C.byref(rep)))
        wall = time.perf_counter() - t0
        return _report(ctx, rep, wall, d_eval is None, m if d_eval is not None else n, False,
                       histograms)


def export_expansions(p: int, n_levels: int, *, device: int | None = None):
    """Debug seam: (mult, local) of the last evaluation as lists per level of
    complex128[4**l, p+1] arrays (the reference's ``mult``/``local``)."""
    ctx = _lib.default_context(device)
    nbox = (4 ** (n_levels + 1) - 1) // 3
    mult = np.empty((nbox, p + 1), np.complex128)
    local = np.empty((nbox, p + 1), np.complex128)
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_export_expansions(ctx.h, _lib.dptr(mult.view(np.float64)),
                                                  _lib.dptr(local.view(np.float64))))
    ms, ls, b = [], [], 0
    for lev in range(n_levels + 1):
        ms.append(mult[b:b + 4**lev])
        ls.append(local[b:b + 4**lev])
        b += 4**lev
    return ms, ls


def export_phi(m: int, *, device: int | None = None) -> np.ndarray:
    """Debug seam: tree-ordered L2P+M2P potentials of the last evaluation."""
    ctx = _lib.default_context(device)
    phi = np.empty(m, np.complex128)
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_export_phi(ctx.h, _lib.dptr(phi.view(np.float64))))
    return phi


def direct_evaluate(points: ParticleSet, symmetric: bool = False, *,
                    device: int | None = None) -> np.ndarray:
    """All-pairs direct sum on the GPU (replaces engine.py:282-323).

    Asymmetric mode (engine.py:291-300): thread per evaluation point, IEEE
    ``1/r2`` as in ``reciprocal_parts`` (operators.py:258-277).  Symmetric
    mode (engine.py:302-323) requires aliased evaluation points, like the
    reference, and shares each pairwise reciprocal between both directions
    (``k_direct_sym``: super-tile pairs, deterministic fold); it matches the
    asymmetric mode to roundoff, as the reference's does.
    """
    if symmetric and not points.evals_alias_sources:
        raise ValueError("symmetric mode requires evaluation points to alias the sources")
    ctx = _lib.default_context(device)
    pos = points.positions
    out = np.empty(points.n_evals, np.complex128)
    with ctx.lock:
        if symmetric:
            ctx.check(ctx.lib.fmm2d_direct_symmetric(
                ctx.h, pos.size, _lib.dptr(pos.view(np.float64)), _lib.dptr(points.strengths),
                _lib.dptr(out.view(np.float64))))
            return out
        epos = None if points.evals_alias_sources else points.eval_positions
        ctx.check(ctx.lib.fmm2d_direct(
            ctx.h, pos.size, _lib.dptr(pos.view(np.float64)), _lib.dptr(points.strengths),
            points.n_evals, None if epos is None else _lib.dptr(epos.view(np.float64)),
            _lib.dptr(out.view(np.float64))))
    return out


def _p2m_all(tree, p: int) -> np.ndarray:
    """Batched P2M of every finest box (engine.py:67-82) on the GPU:
    complex128[4**L, p+1] about the box centers."""
    from .operators import p2m_boxes
    lv = tree.finest
    return p2m_boxes(tree.src_pos, tree.src_strength, lv.src_offsets, lv.center, p)


def max_rel_error(approx, exact) -> float:
    """max |a - e| / |e| over nonzero e (engine.py:326-341)."""
    approx = np.asarray(approx)
    exact = np.asarray(exact)
    if approx.shape != exact.shape:
        raise ValueError("field shapes differ")
    ok = exact != 0
    if not ok.any():
        raise ValueError("all reference values are zero; relative error undefined")
    return float(np.max(np.abs(approx[ok] - exact[ok]) / np.abs(exact[ok])))
