"""Expansion operators on the GPU (drop-in for ``fmm2d.operators``).

Same functions, signatures, batching rules and exceptions as the
reference's unit operators (operators.py:41-297); every one runs as a
batched sm_100a kernel in libfmm2d.so (csrc/operators.cu) with numpy's
element arithmetic (Smith complex division, no contraction) and the
reference's exact cascade order, for any order p >= 1.  The fused engine
does not call these: they serve callers that drive the algebra piecewise.

Conventions (operators.py:1-30): G(y; z, g) = g / (z - y); p2m gives
a[0] = 0, a[j] = -sum g (z - z0)**(j-1); p2l gives b[k] = sum g / (z - z0)**(k+1);
shifts are source center minus target center.
"""

from __future__ import annotations

import numpy as np

from . import _lib

_SCALED_MIN = 1e-12   # operators.py:37-38 (applied per row in the kernels)
_SCALED_MAX = 1e12


def _ctx():
    return _lib.default_context(None)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _as_batch(coeffs, shift):
    """Copy + broadcast exactly as operators.py:41-47."""
    a = np.array(coeffs, dtype=np.complex128, copy=True)
    if a.ndim < 1 or a.shape[-1] < 2:
        raise ValueError("coefficient arrays need at least 2 terms (p >= 1)")
    r = np.asarray(shift, dtype=np.complex128)
    r = np.ascontiguousarray(np.broadcast_to(r, a.shape[:-1]))
    return np.ascontiguousarray(a), r


def _dp(a):
    return _lib.dptr(a.view(np.float64))


def _points_call(fn, positions, strengths, center, p):
    pos = _c128(np.atleast_1d(positions)).ravel()
    g = np.ascontiguousarray(np.broadcast_to(np.asarray(strengths, np.float64), pos.shape))
    c = np.array([center], dtype=np.complex128)
    off = np.array([0, pos.size], np.int64)
    out = np.empty(p + 1, np.complex128)
    ctx = _ctx()
    with ctx.lock:
        ctx.check(fn(ctx.h, 1, _lib.iptr(off), _dp(pos), _lib.dptr(g), _dp(c), int(p), _dp(out)))
    return out


def p2m(positions, strengths, center, p: int) -> np.ndarray:
    """Outgoing coefficients of point sources about ``center`` (operators.py:63-75)."""
    return _points_call(_ctx().lib.fmm2d_op_p2m, positions, strengths, center, p)


def p2l(positions, strengths, center, p: int) -> np.ndarray:
    """Incoming coefficients of far point sources about ``center``
    (operators.py:78-93); raises if a source sits on the center."""
    return _points_call(_ctx().lib.fmm2d_op_p2l, positions, strengths, center, p)


def p2m_boxes(positions, strengths, offsets, centers, p: int) -> np.ndarray:
    """Batched P2M over boxes ``offsets[b]:offsets[b+1]`` -> complex128[nbox, p+1]
    (the engine's ``_p2m_all`` layout, engine.py:67-82)."""
    pos = _c128(positions)
    g = np.ascontiguousarray(strengths, np.float64)
    off = np.ascontiguousarray(offsets, np.int64)
    c = _c128(centers)
    out = np.empty((c.size, p + 1), np.complex128)
    ctx = _ctx()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_op_p2m(ctx.h, c.size, _lib.iptr(off), _dp(pos), _lib.dptr(g),
                                       _dp(c), int(p), _dp(out)))
    return out


def m2m(coeffs, shift, variant: str = "scaled") -> np.ndarray:
    """Re-center outgoing coefficients; ``shift`` = old center - new center
    (operators.py:127-148)."""
    a, r = _as_batch(coeffs, shift)
    if variant not in ("scaled", "unscaled"):
        raise ValueError(f"unknown m2m variant: {variant!r}")
    p = a.shape[-1] - 1
    ctx = _ctx()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_op_m2m(ctx.h, r.size, p, _dp(a), _dp(r),
                                       0 if variant == "scaled" else 1))
    return a


def l2l(coeffs, shift) -> np.ndarray:
    """Re-center incoming coefficients; ``shift`` = old center - new center
    (operators.py:171-186)."""
    b, r = _as_batch(coeffs, shift)
    p = b.shape[-1] - 1
    ctx = _ctx()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_op_l2l(ctx.h, r.size, p, _dp(b), _dp(r)))
    return b


def m2l(coeffs, shift) -> np.ndarray:
    """Outgoing -> incoming across a separated pair; ``shift`` = outgoing
    center minus incoming center, nonzero (operators.py:189-220)."""
    a, rho = _as_batch(coeffs, shift)
    p = a.shape[-1] - 1
    out = np.empty_like(a)
    ctx = _ctx()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_op_m2l(ctx.h, rho.size, p, _dp(a), _dp(rho), _dp(out)))
    return out


def _eval_call(fn, coeffs, center, targets):
    a = _c128(coeffs)
    t = np.asarray(targets, dtype=np.complex128)
    shape = t.shape
    t = np.ascontiguousarray(t).ravel()
    c = np.array([center], dtype=np.complex128)
    out = np.empty(t.size, np.complex128)
    ctx = _ctx()
    with ctx.lock:
        ctx.check(fn(ctx.h, a.size - 1, _dp(a), _dp(c), t.size, _dp(t), _dp(out)))
    return out.reshape(shape)


def l2p(coeffs, center, targets) -> np.ndarray:
    """Evaluate an incoming expansion at targets (Horner; operators.py:227-234)."""
    return _eval_call(_ctx().lib.fmm2d_op_l2p, coeffs, center, targets)


def m2p(coeffs, center, targets) -> np.ndarray:
    """Evaluate an outgoing expansion at targets away from its center
    (operators.py:237-255)."""
    return _eval_call(_ctx().lib.fmm2d_op_m2p, coeffs, center, targets)


def reciprocal_parts(src, tgt):
    """Real and imaginary parts of 1/(z_s - y) for a source/target block,
    zero for coincident pairs, plus their count (operators.py:258-277)."""
    s = _c128(np.atleast_1d(src)).ravel()
    t = _c128(np.atleast_1d(tgt)).ravel()
    re = np.empty((t.size, s.size))
    im = np.empty((t.size, s.size))
    nskip = np.zeros(1, np.int64)
    ctx = _ctx()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_op_reciprocal_parts(ctx.h, s.size, _dp(s), t.size, _dp(t),
                                                    _lib.dptr(re), _lib.dptr(im),
                                                    _lib.iptr(nskip)))
    return re, im, int(nskip[0])


def kernel_block(src_pos, strengths, targets):
    """Dense kernel evaluation of one source block at one target block:
    (potential increments, coincident pairs skipped) (operators.py:280-292)."""
    s = _c128(np.atleast_1d(src_pos)).ravel()
    g = np.ascontiguousarray(np.broadcast_to(np.asarray(strengths, np.float64), s.shape))
    t = _c128(np.atleast_1d(targets)).ravel()
    out = np.empty(t.size, np.complex128)
    nskip = np.zeros(1, np.int64)
    ctx = _ctx()
    with ctx.lock:
        ctx.check(ctx.lib.fmm2d_op_kernel_block(ctx.h, s.size, _dp(s), _lib.dptr(g), t.size,
                                                _dp(t), _dp(out), _lib.iptr(nskip)))
    return out, int(nskip[0])


def p2p_pair(src_pos, strengths, targets):
    """Direct near-field evaluation of one box pair (operators.py:295-297)."""
    return kernel_block(src_pos, strengths, targets)
