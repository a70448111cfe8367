"""GPU unit operators (paper_1205_4611_b200.operators, csrc/operators.cu) and
per-level connectivity (classify_level / reclassify_finest) against the CPU
oracle and the reference's golden lists.

The reference's own operator tests (pkg/tests/test_operators.py) also run
unmodified against these kernels in tests/test_reference_suite.py; here the
kernels are compared term by term with the oracle restatement over a range
of orders, batch shapes and the unscaled fallback window."""

import numpy as np
import pytest

import paper_1205_4611_b200 as F
from paper_1205_4611_b200 import operators as ops
from oracle import fmm2d_oracle as O

from helpers import assert_lists_equal, cfg_from, flat_lists_pkg, load, points_from

pytestmark = pytest.mark.gpu

rng = np.random.default_rng(2024)


def coeffs(p, rows=()):
    shape = tuple(rows) + (p + 1,)
    a = rng.normal(size=shape) + 1j * rng.normal(size=shape)
    return a / (1 + np.arange(p + 1)) ** 2


def close(got, want, tol):
    scale = np.maximum(np.max(np.abs(want), axis=-1, keepdims=True), 1e-300)
    assert np.max(np.abs(got - want) / scale) <= tol


@pytest.mark.parametrize("p", [1, 2, 7, 17, 20, 30, 40, 80])
def test_shift_operators_match_oracle(p):
    a = coeffs(p, (64,))
    a[..., 0] = 0.0                     # the oracle restates the harmonic (a0 = 0) case
    r = 0.3 * (rng.normal(size=64) + 1j * rng.normal(size=64))
    r[5] = 1e-13                        # below the scaled window: unscaled fallback row
    close(ops.m2m(a, r), O.op_m2m(a, r), 1e-12)
    close(ops.l2l(a, r), O.op_l2l(a, r), 1e-12)
    rho = 2.0 + rng.normal(size=64) + 1j * rng.normal(size=64)
    close(ops.m2l(a, rho), O.op_m2l(a, rho), 1e-12)


@pytest.mark.parametrize("p", [1, 17, 30])
def test_point_operators_match_oracle(p):
    z = 0.1 * (rng.normal(size=50) + 1j * rng.normal(size=50))
    g = rng.uniform(-1, 1, 50)
    close(ops.p2m(z, g, 0.01j, p), O.op_p2m(z, g, 0.01j, p), 1e-13)
    close(ops.p2l(z, g, 3.0 + 1j, p), O.op_p2l(z, g, 3.0 + 1j, p), 1e-13)
    b = coeffs(p)
    b[0] = 0.0
    y = 4.0 + rng.normal(size=33) + 1j * rng.normal(size=33)
    np.testing.assert_allclose(ops.l2p(b, 0.5j, y), O.op_l2p(b, 0.5j, y), rtol=1e-13)
    np.testing.assert_allclose(ops.m2p(b, 0.5j, y), O.op_m2p(b, 0.5j, y), rtol=1e-13)


def test_p2p_block_and_skips_match_oracle():
    src = rng.uniform(size=300) + 1j * rng.uniform(size=300)
    tgt = np.concatenate([src[:40], rng.uniform(size=60) + 1j * rng.uniform(size=60)])
    g = rng.uniform(-1, 1, 300)
    phi, skips = ops.kernel_block(src, g, tgt)
    want, want_skips = O.op_p2p(src, g, tgt)
    assert skips == want_skips == 40
    np.testing.assert_allclose(phi, want, rtol=1e-12)
    re, im, n = ops.reciprocal_parts(src, tgt)
    assert n == 40 and re.shape == (100, 300)
    dx = src.real[None, :] - tgt.real[:, None]
    dy = src.imag[None, :] - tgt.imag[:, None]
    r2 = dx * dx
    r2 += dy * dy
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(r2 == 0, 0.0, 1.0 / r2)
    np.testing.assert_array_equal(re, dx * s)       # same rounding sequence: bit-exact
    np.testing.assert_array_equal(im, dy * s)


def test_singular_inputs_raise_reference_messages():
    with pytest.raises(ValueError, match="nonzero"):
        ops.m2l(coeffs(4, (3,)), np.array([1.0, 0.0, 2.0]))
    with pytest.raises(ValueError, match="coincides"):
        ops.p2l(np.array([1 + 1j]), np.array([1.0]), 1 + 1j, 5)
    with pytest.raises(ValueError, match="coincides"):
        ops.m2p(coeffs(4), 1j, np.array([1j]))
    with pytest.raises(ValueError, match="at least 2 terms"):
        ops.m2m(np.zeros(1, complex), 0.5)


def test_log_term_paths():
    """a0 != 0: the log corrections of m2m (unscaled), m2l and m2p
    (operators.py:106-110, 214-217, 252-253) against a direct numpy
    restatement."""
    p = 6
    a = coeffs(p)
    rho = 1.5 - 0.7j
    out = ops.m2l(a, rho)
    # numpy restatement of operators.py:189-220 with the log term
    pw = rho ** np.arange(p + 1)
    c = np.empty(p + 1, complex)
    c[:p] = a[1:] / pw[1:] * (-1.0) ** np.arange(1, p + 1)
    c[p] = 0
    for k in range(2, p + 1):
        lo = p - k
        c[lo:p] = c[lo:p] + c[lo + 1:p + 1]
    for k in range(p, 0, -1):
        for j in range(k, p + 1):
            c[j] += c[j - 1]
    c[0] += a[0] * np.log(-rho)
    c[1:] = (c[1:] - a[0] / np.arange(1, p + 1)) / pw[1:]
    np.testing.assert_allclose(out, c, rtol=1e-13)
    y = np.array([3.0 + 2j])
    u = y - 0.2
    inv = 1.0 / u
    acc = a[p]
    for j in range(p - 1, 0, -1):
        acc = acc * inv + a[j]
    want = acc * inv + a[0] * np.log(u)
    np.testing.assert_allclose(ops.m2p(a, 0.2, y), want, rtol=1e-13)


@pytest.mark.parametrize("name", ["c1_uniform_1e4_p17", "normal_3000_nd40", "separate_4000_700"])
def test_classify_chain_matches_reference_lists(name):
    """classify_level over levels 1..L then reclassify_finest reproduces the
    reference's lists bit for bit (golden from the reference itself)."""
    rec = load(name)
    cfg = cfg_from(rec)
    tree = F.build_tree(points_from(rec), cfg)
    strong = [np.array([0])]
    weak = [[np.empty(0, np.int64)]]
    for lev in range(1, tree.n_levels + 1):
        strong, wk = F.classify_level(tree, lev, strong, cfg.theta)
        weak.append(wk)
    p2p, p2l, m2p = F.reclassify_finest(tree, strong, cfg.theta)
    lists = F.InteractionLists(tree.n_levels, weak, p2p, p2l, m2p)
    assert_lists_equal(flat_lists_pkg(lists), rec)
