"""GPU parity: the CUDA engine against the reference's golden vectors and the
CPU oracle.  Trees and interaction lists bit-exact (canonical form),
potentials within 1e-12 relative (north_star tolerance)."""

import numpy as np
import pytest

import paper_1205_4611_b200 as F
from oracle import fmm2d_oracle as O

from helpers import (FULL_CASES, SAMPLED_CASES, TIE_CASES, assert_lists_equal, assert_tree_equal,
                     cfg_from, flat_lists_oracle, flat_lists_pkg, flat_tree_oracle, flat_tree_pkg,
                     load, max_rel, points_from, sha, tree_sha)

pytestmark = pytest.mark.gpu

PARITY = 1e-12      # potentials vs the reference at the same p/θ/N_d (north_star)

SAMPLED_INPUTS = {
    "uniform_1e5_p20": F.DistributionSpec("uniform", 0.01, 0),
    "normal_1e5_p20": F.DistributionSpec("normal", 0.01, 0),
}


# --- golden vectors produced by the reference ----------------------------------

@pytest.mark.parametrize("name", FULL_CASES)
def test_tree_matches_reference(name):
    rec = load(name)
    tree = F.build_tree(points_from(rec), cfg_from(rec))
    assert_tree_equal(flat_tree_pkg(tree), rec, ties=name in TIE_CASES)


@pytest.mark.parametrize("name", FULL_CASES)
def test_lists_match_reference(name):
    rec = load(name)
    cfg = cfg_from(rec)
    tree = F.build_tree(points_from(rec), cfg)
    lists = F.build_connectivity(tree, cfg.theta)
    assert_lists_equal(flat_lists_pkg(lists), rec)


@pytest.mark.parametrize("name", FULL_CASES)
def test_potentials_match_reference(name):
    rec = load(name)
    pts, cfg = points_from(rec), cfg_from(rec)
    if str(rec["error"]):
        with pytest.raises(ValueError, match="nonzero"):
            F.fmm_evaluate(pts, cfg)
        return
    values, report = F.fmm_evaluate(pts, cfg)
    tol = 1e-7 if name in TIE_CASES else PARITY
    assert max_rel(values, rec["values"]) <= tol
    assert report.coincident_skips == int(rec["coincident_skips"])
    assert report.n_boxes == int(rec["n_boxes"])
    for kind in ("weak", "p2p", "p2l", "m2p"):
        want = {int(a): int(b) for a, b in rec[f"hist_{kind}"]}
        assert report.list_histograms[kind] == want, kind


@pytest.mark.parametrize("name", SAMPLED_CASES)
def test_reference_1e5_cases(name):
    rec = load(name)
    pts = F.sample_points(SAMPLED_INPUTS[name], 100_000)
    cfg = cfg_from(rec)
    tree = F.build_tree(pts, cfg)
    assert tree_sha(flat_tree_pkg(tree)) == str(rec["tree_sha"])
    lists = F.build_connectivity(tree, cfg.theta)
    fl = flat_lists_pkg(lists)
    assert sha(*[fl[k] for k in sorted(fl)]) == str(rec["lists_sha"])
    values, _ = F.fmm_evaluate(pts, cfg)
    idx = rec["sample_idx"]
    assert max_rel(values[idx], rec["sample_values"]) <= PARITY


# --- fresh inputs against the oracle -------------------------------------------

def _rand_points(kind, n, seed, m=None, cluster=False):
    rng = np.random.default_rng(seed)
    pts = F.sample_points(F.DistributionSpec(kind, 0.001 if kind == "normal" else 0.01, seed), n)
    if m is None:
        return pts
    if cluster:   # evaluation points piled into one corner: very unbalanced leaves
        ev = 0.05 * (rng.uniform(size=m) + 1j * rng.uniform(size=m))
    else:
        ev = rng.uniform(size=m) + 1j * rng.uniform(size=m)
    return F.ParticleSet(pts.positions, pts.strengths, ev)


CASES = [
    ("uniform", 20_000, 1, None, False, F.TreeConfig(35, 0.5, 20)),
    ("normal", 20_000, 2, None, False, F.TreeConfig(35, 0.5, 20)),
    ("layer", 15_000, 3, None, False, F.TreeConfig(35, 0.5, 17)),
    ("uniform", 12_000, 4, 9_000, False, F.TreeConfig(35, 0.5, 30)),
    ("uniform", 8_000, 5, 5_000, True, F.TreeConfig(35, 0.5, 17)),
    ("normal", 30_000, 6, None, False, F.TreeConfig(20, 0.5, 12)),
    ("uniform", 5_000, 7, None, False, F.TreeConfig(100, 0.5, 8)),
    ("uniform", 3_000, 8, None, False, F.TreeConfig(1, 0.5, 4)),
    ("uniform", 6_000, 9, None, False, F.TreeConfig(35, 0.3, 24)),
    ("uniform", 6_000, 10, None, False, F.TreeConfig(35, 0.7, 40)),
    ("uniform", 2_000, 11, None, False, F.TreeConfig(35, 0.5, 1)),
    ("uniform", 45 * 2**8, 12, None, False, F.TreeConfig(45, 0.5, 17)),
    ("uniform", 700, 13, None, False, F.TreeConfig(1000, 0.5, 17)),   # zero levels
    # many separate evaluation points per leaf: the two-block P2P kernel
    # (> 32 points per leaf, several 64-point passes), uniform and clustered
    ("uniform", 4_000, 14, 30_000, False, F.TreeConfig(35, 0.5, 17)),
    ("uniform", 4_000, 15, 30_000, True, F.TreeConfig(35, 0.5, 17)),
    # exact-order M2L with the two-phase fold at the largest dense order
    ("normal", 8_000, 16, None, False, F.TreeConfig(35, 0.5, 32)),
]


@pytest.mark.parametrize("kind,n,seed,m,cluster,cfg", CASES)
def test_engine_matches_oracle(kind, n, seed, m, cluster, cfg):
    pts = _rand_points(kind, n, seed, m, cluster)
    ev = None if pts.evals_alias_sources else pts.eval_positions
    T = O.build_tree(pts.positions, pts.strengths, ev, cfg.n_desired_per_box)
    Ls = O.build_connectivity(T, cfg.theta)
    R = O.evaluate(T, Ls, cfg.p_terms)

    tree = F.build_tree(pts, cfg)
    assert_tree_equal(flat_tree_pkg(tree), flat_tree_oracle(T))
    lists = F.build_connectivity(tree, cfg.theta)
    assert_lists_equal(flat_lists_pkg(lists), flat_lists_oracle(Ls))
    values, report = F.fmm_evaluate(pts, cfg)
    assert max_rel(values, R.values) <= PARITY
    assert report.coincident_skips == R.coincident_skips
    assert report.n_levels == T.n_levels


def test_phase_seams_match_oracle():
    """Per-phase seams: multipole and local coefficients of every box
    (P2M+M2M and P2L+M2L+L2L) against the oracle, relative to each box's
    coefficient norm, and the far field at every evaluation point (L2P + M2P,
    before P2P; engine.py:132-160) against the oracle's."""
    pts = F.sample_points(F.DistributionSpec("uniform", seed=21), 20_000)
    cfg = F.TreeConfig(35, 0.5, 20)
    T = O.build_tree(pts.positions, pts.strengths, None, cfg.n_desired_per_box)
    Ls = O.build_connectivity(T, cfg.theta)
    R = O.evaluate(T, Ls, cfg.p_terms)
    F.fmm_evaluate(pts, cfg)
    mult, local = F.engine.export_expansions(cfg.p_terms, T.n_levels)
    for lev in range(1, T.n_levels + 1):
        for got, want in ((mult[lev], R.mult[lev]), (local[lev], R.local[lev])):
            scale = np.max(np.abs(want), axis=1, keepdims=True)
            scale[scale == 0] = 1.0
            assert np.max(np.abs(got - want) / scale) <= 1e-12, lev
    phi = F.engine.export_phi(pts.n_evals)
    want = R.phi_far
    assert phi.shape == want.shape
    assert np.max(np.abs(phi - want)) <= 1e-12 * np.max(np.abs(want))
    rel = np.abs(phi - want) / np.abs(want)
    assert np.median(rel) <= 1e-14, float(np.median(rel))


def test_tie_runs_of_rank_keys_fall_back_to_exact_keys():
    """300 points packed within 3e-11 in x (one run of equal 32-bit rank keys,
    longer than the in-kernel fix-up handles) plus spread points: the engine
    must rerun with exact 64-bit keys and still match the oracle."""
    rng = np.random.default_rng(77)
    x = np.concatenate([0.5 + 1e-13 * np.arange(300), rng.uniform(size=3000)])
    y = rng.uniform(size=x.size)
    pts = F.ParticleSet(x + 1j * y, rng.uniform(-1, 1, x.size))
    cfg = F.TreeConfig(20, 0.5, 17)
    T = O.build_tree(pts.positions, pts.strengths, None, 20)
    tree = F.build_tree(pts, cfg)
    assert_tree_equal(flat_tree_pkg(tree), flat_tree_oracle(T))
    values, _ = F.fmm_evaluate(pts, cfg)
    R = O.evaluate(T, O.build_connectivity(T, 0.5), 17)
    assert max_rel(values, R.values) <= PARITY
