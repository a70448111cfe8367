"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import fmm2d_oracle as O
from paper_1205_4611_b200 import DistributionSpec, sample_points

from helpers import (GOLDEN, FULL_CASES, SAMPLED_CASES, TIE_CASES, assert_lists_equal, assert_tree_equal,
                     flat_lists_oracle, flat_tree_oracle, load, max_rel, sha, tree_sha)

SAMPLED_INPUTS = {
    "uniform_1e5_p20": DistributionSpec("uniform", 0.01, 0),
    "normal_1e5_p20": DistributionSpec("normal", 0.01, 0),
}


def _oracle_inputs(rec):
    ev = rec.get("eval_positions")
    return rec["positions"], rec["strengths"], ev


@pytest.mark.parametrize("name", FULL_CASES)
def test_oracle_tree_and_lists_match_reference(name):
    rec = load(name)
    pos, g, ev = _oracle_inputs(rec)
    nd, theta, p = rec["cfg"]
    T = O.build_tree(pos, g, ev, int(nd))
    assert_tree_equal(flat_tree_oracle(T), rec, ties=name in TIE_CASES)
    Ls = O.build_connectivity(T, float(theta))
    assert_lists_equal(flat_lists_oracle(Ls), rec)


@pytest.mark.parametrize("name", FULL_CASES)
def test_oracle_potentials_match_reference(name):
    rec = load(name)
    pos, g, ev = _oracle_inputs(rec)
    nd, theta, p = rec["cfg"]
    err = str(rec["error"])
    if err:
        with pytest.raises(ValueError, match="nonzero"):
            O.fmm(pos, g, ev, int(nd), float(theta), int(p))
        return
    vals, R, _, _ = O.fmm(pos, g, ev, int(nd), float(theta), int(p))
    # ties at cuts (coincident points) make in-box membership ISA dependent in
    # the reference; only the FMM tolerance is comparable there
    tol = 1e-7 if name in TIE_CASES else 5e-13
    assert max_rel(vals, rec["values"]) <= tol
    assert R.coincident_skips == int(rec["coincident_skips"])


@pytest.mark.parametrize("name", SAMPLED_CASES)
def test_oracle_matches_reference_1e5(name):
    rec = load(name)
    pts = sample_points(SAMPLED_INPUTS[name], 100_000)
    nd, theta, p = rec["cfg"]
    vals, R, T, Ls = O.fmm(pts.positions, pts.strengths, None, int(nd), float(theta), int(p))
    assert tree_sha(flat_tree_oracle(T)) == str(rec["tree_sha"])
    fl = flat_lists_oracle(Ls)
    assert sha(*[fl[k] for k in sorted(fl)]) == str(rec["lists_sha"])
    idx = rec["sample_idx"]
    assert max_rel(vals[idx], rec["sample_values"]) <= 5e-13


def test_dataset_generator_fingerprints():
    fp = dict(np.load(GOLDEN / "datasets.npz"))
    for key, want in fp.items():
        kind, seed = key.rsplit("_", 1)
        p = sample_points(DistributionSpec(kind, 0.01, int(seed)), 5000)
        assert sha(p.positions, p.strengths) == str(want), key


def test_oracle_direct_small_cases():
    # engine.py direct oracle semantics (test_engine.py:17-47 of the reference)
    phi = O.direct(np.array([0j, 1.0 + 0j]), np.ones(2))
    np.testing.assert_allclose(phi, [1.0, -1.0], rtol=1e-15)
    phi = O.direct(np.array([0j, 1.0 + 0j, 2.0 + 0j]), np.ones(3))
    assert phi[0] == pytest.approx(1.5)


def test_oracle_degenerate():
    with pytest.raises(O.OracleDegenerate, match="coincide"):
        O.build_tree(np.full(10, 0.5 + 0.5j), np.ones(10), None, 1)


@pytest.mark.parametrize("name", ["uniform_3000", "normal_dup_2701"])
def test_oracle_direct_matches_reference(name):
    """The oracle's direct sum against the reference's direct_evaluate in both
    modes (tests/golden/make_golden_direct.py); duplicates contribute nothing."""
    d = load("direct_sum")
    phi = O.direct(d[f"{name}_positions"], d[f"{name}_strengths"])
    assert O.max_rel(phi, d[f"{name}_asymmetric"]) <= 1e-13
    assert O.max_rel(phi, d[f"{name}_symmetric"]) <= 1e-12
