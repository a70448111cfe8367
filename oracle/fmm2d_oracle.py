"""CPU ORACLE for the adaptive 2-D FMM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``fmm2d`` pipeline
(/root/reference/pkg/src/fmm2d, "the reference" below).  It is the checker
for the CUDA engine in ``paper_1205_4611_b200``: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path never calls it.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``): canonical trees and interaction lists
bit-exact, potentials to 1e-13 relative.

Canonical tree.  The reference median split uses ``np.argpartition``
(tree.py:97-114) whose order *within* each half is ISA dependent; the
member sets, offsets, cuts and rectangles are not.  This restatement uses
the deterministic rule the GPU engine implements: a stable partition that
sends the k = ceil(n/2) smallest coordinates left, ties broken by position
(which is always ascending original index, because every partition is
stable starting from the identity).  Hence inside every finest box the
sources are in ascending original index order -- the canonical form.

Every function cites the reference lines it restates.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

PHASES = ("sort", "connect", "p2m", "m2m", "m2l", "l2l", "l2p", "p2p", "other")
SCALED_LO, SCALED_HI = 1e-12, 1e12          # operators.py:37-38


class OracleDegenerate(ValueError):
    """Mirror of tree.DegenerateInputError (tree.py:20-21)."""


# ---------------------------------------------------------------------------
# tree  (tree.py:86-334)

def levels_for(n: int, nd: int) -> int:
    """Eq. (6) depth, clamped so that 4**L <= n (tree.py:86-94, 249-255)."""
    if n < 1 or nd < 1:
        raise ValueError("n_sources and n_desired must be >= 1")
    lev = max(0, math.ceil(0.5 * math.log2(0.625 * n / nd)))
    while lev > 0 and 4**lev > n:
        lev -= 1
    return lev


@dataclass
class OTree:
    n_levels: int
    # per level l: arrays of length 4**l
    x0: list
    x1: list
    y0: list
    y1: list
    center: list
    hw: list
    hh: list
    src_off: list          # length 4**l + 1
    eval_off: list
    src_perm: np.ndarray
    eval_perm: np.ndarray
    src_pos: np.ndarray
    src_g: np.ndarray
    eval_pos: np.ndarray
    aliased: bool = False


def _rect_geometry(x0, x1, y0, y1):
    """Center / half extents from rectangle corners (tree.py:225-227, 375-377)."""
    center = (x0 + x1) / 2 + 1j * ((y0 + y1) / 2)
    return center, (x1 - x0) / 2, (y1 - y0) / 2


def _seg_ids(off):
    counts = np.diff(off)
    return np.repeat(np.arange(counts.size), counts), counts


def _split_step(coords_x, coords_y, perm_arrays, off, rect, eval_state):
    """One successive-split step over every segment at once.

    Per segment: axis from the rectangle (geometry.py:57-63 on
    tree.py:225-227), k = ceil(n/2) (tree.py:108), cut = k-th smallest
    coordinate (tree.py:202), sources stable-partitioned (canonical rule),
    evaluation points stable-partitioned by ``coord <= cut``
    (tree.py:205-215), rectangles cut at ``cut`` (tree.py:218-222).
    """
    x0, x1, y0, y1 = rect
    along_y = (y1 - y0) / 2 > (x1 - x0) / 2
    seg, counts = _seg_ids(off)
    n_seg = counts.size
    coords = np.where(along_y[seg], coords_y, coords_x)
    # stable order inside each segment by coordinate (ties keep position)
    order = np.lexsort((coords, seg))
    kk = (counts + 1) // 2
    pos_in_seg = np.empty(coords.size, dtype=np.int64)
    pos_in_seg[order] = np.arange(coords.size) - np.repeat(off[:-1], counts)
    left = pos_in_seg < np.repeat(kk, counts)
    cut = coords[order[off[:-1] + kk - 1]]
    new_order = np.lexsort((~left, seg))  # stable: left block then right block
    for a in perm_arrays:
        a[:] = a[new_order]
    new_off = np.empty(2 * n_seg + 1, dtype=np.int64)
    new_off[0] = 0
    new_off[1::2] = off[:-1] + kk
    new_off[2::2] = off[1:]

    ex, ey, eperm, eoff = eval_state
    eseg, ecounts = _seg_ids(eoff)
    ecoords = np.where(along_y[eseg], ey, ex)
    eleft = ecoords <= cut[eseg]
    eorder = np.lexsort((~eleft, eseg))
    ex[:] = ex[eorder]
    ey[:] = ey[eorder]
    eperm[:] = eperm[eorder]
    nleft = np.bincount(eseg[eleft], minlength=n_seg) if eseg.size else np.zeros(n_seg, np.int64)
    new_eoff = np.empty(2 * n_seg + 1, dtype=np.int64)
    new_eoff[0] = 0
    new_eoff[1::2] = eoff[:-1] + nleft
    new_eoff[2::2] = eoff[1:]

    # child rectangles, left child first
    nx0 = np.empty(2 * n_seg); nx1 = np.empty(2 * n_seg)
    ny0 = np.empty(2 * n_seg); ny1 = np.empty(2 * n_seg)
    nx0[0::2] = x0; nx0[1::2] = np.where(along_y, x0, cut)
    nx1[0::2] = np.where(along_y, x1, cut); nx1[1::2] = x1
    ny0[0::2] = y0; ny0[1::2] = np.where(along_y, cut, y0)
    ny1[0::2] = np.where(along_y, cut, y1); ny1[1::2] = y1
    return new_off, new_eoff, (nx0, nx1, ny0, ny1)


def build_tree(positions, strengths, eval_positions=None, nd=35) -> OTree:
    """Canonical pyramid tree (restates tree.py:230-334)."""
    pos = np.ascontiguousarray(positions, dtype=np.complex128)
    g = np.ascontiguousarray(strengths, dtype=np.float64)
    aliased = eval_positions is None or eval_positions is positions
    epos = pos if aliased else np.ascontiguousarray(eval_positions, dtype=np.complex128)
    n, m = pos.size, epos.size
    n_lev = levels_for(n, nd)
    xs, ys, gs = pos.real.copy(), pos.imag.copy(), g.copy()
    ex, ey = epos.real.copy(), epos.imag.copy()
    sperm = np.arange(n, dtype=np.int64)
    eperm = np.arange(m, dtype=np.int64)
    rect = tuple(np.array([v]) for v in (min(xs.min(), ex.min()), max(xs.max(), ex.max()),
                                          min(ys.min(), ey.min()), max(ys.max(), ey.max())))
    off = np.array([0, n], dtype=np.int64)
    eoff = np.array([0, m], dtype=np.int64)
    T = OTree(n_lev, [], [], [], [], [], [], [], [], [], sperm, eperm, None, None, None, aliased)

    def record(rect, off, eoff):
        c, hw, hh = _rect_geometry(*rect)
        for lst, v in ((T.x0, rect[0]), (T.x1, rect[1]), (T.y0, rect[2]), (T.y1, rect[3]),
                       (T.center, c), (T.hw, hw), (T.hh, hh), (T.src_off, off), (T.eval_off, eoff)):
            lst.append(v.copy())

    record(rect, off, eoff)
    for lev in range(n_lev):
        # degenerate boxes (tree.py:285-291): first offending box in order
        seg, counts = _seg_ids(off)
        starts = off[:-1]
        same_x = np.minimum.reduceat(xs, starts) == np.maximum.reduceat(xs, starts)
        same_y = np.minimum.reduceat(ys, starts) == np.maximum.reduceat(ys, starts)
        bad = np.flatnonzero(same_x & same_y)
        if bad.size:
            k = int(bad[0]); s0 = int(starts[k])
            raise OracleDegenerate(
                f"all {int(counts[k])} source points in box {k} at level {lev} "
                f"coincide at ({xs[s0]}, {ys[s0]}) but {n_lev - lev} more "
                "level(s) are required; reduce the level count or perturb "
                "the input")
        for _ in range(2):
            off, eoff, rect = _split_step(xs, ys, (xs, ys, gs, sperm), off, rect,
                                          (ex, ey, eperm, eoff))
        record(rect, off, eoff)
    T.src_pos = xs + 1j * ys
    T.src_g = gs
    T.eval_pos = ex + 1j * ey
    return T


# ---------------------------------------------------------------------------
# connectivity  (geometry.py:27-54, connectivity.py:47-114)

def _radius(hw, hh):
    return np.hypot(hw, hh)                       # geometry.py:27-29


def _separated(rt, rs, ct, cs, theta, swapped=False):
    """θ-criterion, geometry.py:32-41 (normal) and 44-54 (swapped)."""
    d = np.abs(ct - cs)
    big, small = np.maximum(rt, rs), np.minimum(rt, rs)
    if swapped:
        big, small = small, big
    return big + theta * small <= theta * d


@dataclass
class OLists:
    n_levels: int
    weak_off: list      # per level l: int64[4**l + 1]
    weak_idx: list      # per level l: int64[...]
    p2p_off: np.ndarray
    p2p_idx: np.ndarray
    p2l_off: np.ndarray
    p2l_idx: np.ndarray
    m2p_off: np.ndarray
    m2p_idx: np.ndarray


def _csr_split(owner, values, mask, n_owner):
    sel_owner = owner[mask]
    counts = np.bincount(sel_owner, minlength=n_owner)
    off = np.zeros(n_owner + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off, values[mask]


def build_connectivity(T: OTree, theta=0.5) -> OLists:
    """Level-by-level weak/strong classification (connectivity.py:47-68,
    99-114) and the finest reclassification (connectivity.py:71-96)."""
    s_off = np.array([0, 1], dtype=np.int64)
    s_idx = np.array([0], dtype=np.int64)
    weak_off = [np.zeros(2, dtype=np.int64)]
    weak_idx = [np.empty(0, dtype=np.int64)]
    for lev in range(1, T.n_levels + 1):
        nb = 4**lev
        r = _radius(T.hw[lev], T.hh[lev])
        c = T.center[lev]
        par = np.arange(nb) // 4
        pcount = np.diff(s_off)[par]
        tgt = np.repeat(np.arange(nb), 4 * pcount)
        # candidates: children of the parent's strong boxes, ascending
        starts = np.repeat(s_off[par], pcount)
        within = np.arange(pcount.sum()) - np.repeat(np.cumsum(pcount) - pcount, pcount)
        parents_strong = s_idx[starts + within]
        cand = (parents_strong[:, None] * 4 + np.arange(4)).ravel()
        far = _separated(r[tgt], r[cand], c[tgt], c[cand], theta)
        wo, wi = _csr_split(tgt, cand, far, nb)
        s_off, s_idx = _csr_split(tgt, cand, ~far, nb)
        weak_off.append(wo)
        weak_idx.append(wi)
    lev = T.n_levels
    nb = 4**lev
    r = _radius(T.hw[lev], T.hh[lev])
    c = T.center[lev]
    tgt = np.repeat(np.arange(nb), np.diff(s_off))
    src = s_idx
    sw = _separated(r[tgt], r[src], c[tgt], c[src], theta, swapped=True)
    moved = sw & (src != tgt) & (r[src] != r[tgt])
    larger = moved & (r[src] > r[tgt])
    smaller = moved & (r[src] < r[tgt])
    p2p = _csr_split(tgt, src, ~moved, nb)
    p2l = _csr_split(tgt, src, larger, nb)
    m2p = _csr_split(tgt, src, smaller, nb)
    return OLists(T.n_levels, weak_off, weak_idx, *p2p, *p2l, *m2p)


# ---------------------------------------------------------------------------
# operators  (operators.py:41-297), batched over a leading axis

def _pow_table(r, p):
    out = np.empty(r.shape + (p + 1,), dtype=np.complex128)
    out[..., 0] = 1.0
    for j in range(1, p + 1):
        out[..., j] = out[..., j - 1] * r
    return out


def op_m2m(a, r):
    """Outgoing re-centering, shift = child - parent (operators.py:100-148).
    a[...,0] is zero throughout the harmonic pipeline (p2m sets it)."""
    a = np.array(a, dtype=np.complex128)
    p = a.shape[-1] - 1
    mag = np.abs(r)
    ok = (mag >= SCALED_LO) & (mag <= SCALED_HI)
    rr = np.where(ok, r, 1.0)
    pw = _pow_table(rr, p)
    s = a.copy()
    s[..., 1:] /= pw[..., 1:]
    for k in range(p, 1, -1):                       # new-value cascade
        for j in range(k, p + 1):
            s[..., j] += s[..., j - 1]
    s[..., 1:] = (s[..., 1:] - s[..., :1] / np.arange(1, p + 1)) * pw[..., 1:]
    if np.all(ok):
        return s
    u = a.copy()                                     # unscaled fallback
    for k in range(p, 1, -1):
        for j in range(k, p + 1):
            u[..., j] += r * u[..., j - 1]
    return np.where(ok[..., None], s, u)


def op_l2l(b, r):
    """Incoming re-centering, shift = parent - child (operators.py:151-186)."""
    b = np.array(b, dtype=np.complex128)
    p = b.shape[-1] - 1
    mag = np.abs(r)
    ok = (mag >= SCALED_LO) & (mag <= SCALED_HI)
    rr = np.where(ok, r, 1.0)
    pw = _pow_table(rr, p)
    s = b.copy()
    s[..., 1:] *= pw[..., 1:]
    for k in range(p + 1):                           # old-value slices
        lo = p - k
        s[..., lo:p] = s[..., lo:p] - s[..., lo + 1:p + 1]
    s[..., 1:] /= pw[..., 1:]
    if np.all(ok):
        return s
    u = b.copy()
    for k in range(p + 1):
        lo = p - k
        u[..., lo:p] = u[..., lo:p] - r[..., None] * u[..., lo + 1:p + 1]
    return np.where(ok[..., None], s, u)


def op_m2l(a, rho):
    """Outgoing -> incoming, rho = source center - target center
    (operators.py:189-220); a[...,0] == 0 in the harmonic pipeline."""
    a = np.asarray(a, dtype=np.complex128)
    if np.any(rho == 0):
        raise ValueError("m2l shift must be nonzero (boxes are separated)")
    p = a.shape[-1] - 1
    pw = _pow_table(rho, p)
    c = np.empty_like(a)
    sgn = (-1.0) ** np.arange(1, p + 1)
    c[..., :p] = a[..., 1:] / pw[..., 1:] * sgn
    c[..., p] = 0.0
    for k in range(2, p + 1):                        # old-value slices
        lo = p - k
        c[..., lo:p] = c[..., lo:p] + c[..., lo + 1:p + 1]
    for k in range(p, 0, -1):                        # new-value cascade
        for j in range(k, p + 1):
            c[..., j] += c[..., j - 1]
    c[..., 1:] = (c[..., 1:] - a[..., :1] / np.arange(1, p + 1)) / pw[..., 1:]
    return c


def op_p2m(pos, g, center, p):
    """a0 = 0, a_j = -sum g (z - z0)^(j-1) (operators.py:63-75)."""
    w = np.asarray(g, dtype=np.complex128)
    d = np.asarray(pos) - center
    a = np.zeros(p + 1, dtype=np.complex128)
    for j in range(1, p + 1):
        a[j] = -w.sum()
        w = w * d
    return a


def op_p2l(pos, g, center, p):
    """b_k = sum g / (z - z0)^(k+1) (operators.py:78-93)."""
    d = np.asarray(pos) - center
    if np.any(d == 0):
        raise ValueError("p2l source coincides with the expansion center")
    inv = 1.0 / d
    w = np.asarray(g) * inv
    b = np.empty(p + 1, dtype=np.complex128)
    for k in range(p + 1):
        b[k] = w.sum()
        w = w * inv
    return b


def op_l2p(b, center, y):
    """Horner in (y - z0) (operators.py:227-234)."""
    w = np.asarray(y) - center
    acc = np.full(w.shape, b[-1], dtype=np.complex128)
    for j in range(len(b) - 2, -1, -1):
        acc = acc * w + b[j]
    return acc


def op_m2p(a, center, y):
    """Horner in 1/(y - z0) over a_p..a_1 (operators.py:237-255)."""
    u = np.asarray(y) - center
    if np.any(u == 0):
        raise ValueError("m2p target coincides with the expansion center")
    inv = 1.0 / u
    p = len(a) - 1
    acc = np.full(inv.shape, a[p], dtype=np.complex128)
    for j in range(p - 1, 0, -1):
        acc = acc * inv + a[j]
    return acc * inv


def op_p2p(src, g, tgt):
    """Near-field block with coincidence skipping (operators.py:258-292)."""
    dx = src.real[None, :] - tgt.real[:, None]
    dy = src.imag[None, :] - tgt.imag[:, None]
    r2 = dx * dx + dy * dy
    zero = r2 == 0.0
    with np.errstate(divide="ignore"):
        s = np.where(zero, 0.0, 1.0 / np.where(zero, 1.0, r2))
    return (dx * s).dot(g) - 1j * (dy * s).dot(g), int(zero.sum())


# ---------------------------------------------------------------------------
# engine  (engine.py:67-279)

@dataclass
class OResult:
    values: np.ndarray
    skips: int
    coincident_skips: int
    phase_seconds: dict = field(default_factory=dict)
    mult: list = field(default_factory=list)
    local: list = field(default_factory=list)
    phi_sorted: np.ndarray | None = None
    phi_far: np.ndarray | None = None     # tree order, L2P + M2P only (before P2P)


def p2m_leaves(T: OTree, p):
    """engine.py:67-82: segmented reduction over leaf ranges."""
    L = T.n_levels
    off = T.src_off[L]
    counts = np.diff(off)
    d = T.src_pos - np.repeat(T.center[L], counts)
    out = np.zeros((counts.size, p + 1), dtype=np.complex128)
    w = T.src_g.astype(np.complex128)
    for j in range(1, p + 1):
        out[:, j] = -np.add.reduceat(w, off[:-1])
        w = w * d
    return out


def evaluate(T: OTree, Ls: OLists, p: int, timings=True) -> OResult:
    """Phase order and accumulation order of engine.py:207-279."""
    t = {}
    L = T.n_levels
    mult = [None] * (L + 1)
    local = [np.zeros((4**l, p + 1), dtype=np.complex128) for l in range(L + 1)]
    soff = T.src_off[L]
    eoff = T.eval_off[L]

    t0 = time.perf_counter()
    if L > 0:
        mult[L] = p2m_leaves(T, p)
        for b in range(4**L):                      # engine.py:85-93
            for a in Ls.p2l_idx[Ls.p2l_off[b]:Ls.p2l_off[b + 1]]:
                local[L][b] += op_p2l(T.src_pos[soff[a]:soff[a + 1]],
                                      T.src_g[soff[a]:soff[a + 1]], T.center[L][b], p)
    t["p2m"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    for lev in range(L - 1, 0, -1):                # engine.py:96-100
        shifts = T.center[lev + 1] - np.repeat(T.center[lev], 4)
        mult[lev] = op_m2m(mult[lev + 1], shifts).reshape(-1, 4, p + 1).sum(axis=1)
    t["m2m"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    for lev in range(1, L + 1):                    # engine.py:103-123
        off, idx = Ls.weak_off[lev], Ls.weak_idx[lev]
        cnt = np.diff(off)
        tg = np.flatnonzero(cnt)
        if tg.size == 0:
            continue
        tgt = np.repeat(np.arange(cnt.size), cnt)
        c = T.center[lev]
        contrib = op_m2l(mult[lev][idx], c[idx] - c[tgt])
        local[lev][tg] += np.add.reduceat(contrib, off[:-1][tg], axis=0)
    t["m2l"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    for lev in range(1, L):                        # engine.py:126-129, 251-252
        shifts = np.repeat(T.center[lev], 4) - T.center[lev + 1]
        local[lev + 1] += op_l2l(np.repeat(local[lev], 4, axis=0), shifts)
    t["l2l"] = time.perf_counter() - t0

    phi = np.zeros(T.eval_pos.size, dtype=np.complex128)
    t0 = time.perf_counter()
    if L > 0:
        ecnt = np.diff(eoff)                         # engine.py:132-149
        w = T.eval_pos - np.repeat(T.center[L], ecnt)
        acc = np.repeat(local[L][:, p], ecnt)
        for j in range(p - 1, -1, -1):
            acc = acc * w + np.repeat(local[L][:, j], ecnt)
        phi += acc
        for b in range(4**L):                        # engine.py:152-160
            e0, e1 = eoff[b], eoff[b + 1]
            if e0 == e1:
                continue
            for a in Ls.m2p_idx[Ls.m2p_off[b]:Ls.m2p_off[b + 1]]:
                phi[e0:e1] += op_m2p(mult[L][a], T.center[L][a], T.eval_pos[e0:e1])
    t["l2p"] = time.perf_counter() - t0
    phi_far = phi.copy()

    t0 = time.perf_counter()
    skips = 0
    for b in range(4**L):                            # engine.py:163-182
        e0, e1 = eoff[b], eoff[b + 1]
        if e0 == e1:
            continue
        boxes = Ls.p2p_idx[Ls.p2p_off[b]:Ls.p2p_off[b + 1]]
        zs = np.concatenate([T.src_pos[soff[a]:soff[a + 1]] for a in boxes])
        gs = np.concatenate([T.src_g[soff[a]:soff[a + 1]] for a in boxes])
        contrib, ns = op_p2p(zs, gs, T.eval_pos[e0:e1])
        phi[e0:e1] += contrib
        skips += ns
    t["p2p"] = time.perf_counter() - t0

    values = np.empty_like(phi)
    values[T.eval_perm] = phi                        # engine.py:266-267
    expected_self = T.eval_pos.size if T.aliased else 0
    return OResult(values, skips, max(0, skips - expected_self), t, mult, local, phi, phi_far)


def fmm(positions, strengths, eval_positions=None, nd=35, theta=0.5, p=17):
    """Whole pipeline; returns (values, OResult, tree, lists)."""
    t0 = time.perf_counter()
    T = build_tree(positions, strengths, eval_positions, nd)
    t1 = time.perf_counter()
    Ls = build_connectivity(T, theta)
    t2 = time.perf_counter()
    R = evaluate(T, Ls, p)
    t3 = time.perf_counter()
    R.phase_seconds["sort"] = t1 - t0
    R.phase_seconds["connect"] = t2 - t1
    R.phase_seconds["total"] = t3 - t0
    return R.values, R, T, Ls


def direct(positions, strengths, eval_positions=None, chunk=1024):
    """All-pairs oracle, asymmetric mode (engine.py:282-300)."""
    zs = np.asarray(positions, dtype=np.complex128)
    g = np.asarray(strengths, dtype=np.float64)
    ze = zs if eval_positions is None else np.asarray(eval_positions, dtype=np.complex128)
    phi = np.zeros(ze.size, dtype=np.complex128)
    for t0 in range(0, ze.size, chunk):
        t1 = min(t0 + chunk, ze.size)
        for s0 in range(0, zs.size, 8192):
            s1 = min(s0 + 8192, zs.size)
            blk, _ = op_p2p(zs[s0:s1], g[s0:s1], ze[t0:t1])
            phi[t0:t1] += blk
    return phi


def max_rel(approx, exact):
    """engine.py:326-341."""
    approx, exact = np.asarray(approx), np.asarray(exact)
    if approx.shape != exact.shape:
        raise ValueError("field shapes differ")
    ok = exact != 0
    if not ok.any():
        raise ValueError("all reference values are zero; relative error undefined")
    return float(np.max(np.abs(approx[ok] - exact[ok]) / np.abs(exact[ok])))


# ---------------------------------------------------------------------------
# canonical forms used by the parity tests

def canonical_leaf_sets(src_off_finest, src_perm):
    """src_perm with every finest box's members sorted ascending: identical
    for the reference (any ISA), this oracle and the GPU engine."""
    out = np.array(src_perm, dtype=np.int64, copy=True)
    off = np.asarray(src_off_finest)
    for b in range(off.size - 1):
        out[off[b]:off[b + 1]].sort()
    return out
