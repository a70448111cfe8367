"""GPU engine behaviour: the reference's own engine/operator properties
(test_engine.py, test_tree.py, test_connectivity.py) on the CUDA path, plus
size-independent properties at BASELINE sizes."""

import numpy as np
import pytest

import paper_1205_4611_b200 as F

pytestmark = pytest.mark.gpu


def uniform(n, seed=0):
    return F.sample_points(F.DistributionSpec("uniform", seed=seed), n)


# --- direct evaluation (reference test_engine.py:17-47) -------------------------

def test_direct_two_particles():
    pts = F.ParticleSet(np.array([0j, 1.0 + 0j]), np.ones(2))
    np.testing.assert_allclose(F.direct_evaluate(pts), [1.0, -1.0], rtol=1e-15)


def test_direct_three_collinear():
    phi = F.direct_evaluate(F.ParticleSet(np.array([0j, 1.0 + 0j, 2.0 + 0j]), np.ones(3)))
    assert phi[0] == pytest.approx(1.5)


def test_direct_symmetric_requires_aliasing():
    pts = F.ParticleSet(np.array([0j, 1j]), np.ones(2), np.array([2.0 + 0j]))
    with pytest.raises(ValueError, match="alias"):
        F.direct_evaluate(pts, symmetric=True)


GOLD_DIRECT = ["uniform_3000", "normal_dup_2701"]


@pytest.mark.parametrize("name", GOLD_DIRECT)
@pytest.mark.parametrize("symmetric", [False, True])
def test_direct_matches_reference_goldens(name, symmetric):
    """Both modes against the reference's own direct_evaluate outputs
    (tests/golden/make_golden_direct.py); normal_dup has exact duplicates."""
    from helpers import load
    d = load("direct_sum")
    pts = F.ParticleSet(d[f"{name}_positions"], d[f"{name}_strengths"])
    want = d[f"{name}_symmetric" if symmetric else f"{name}_asymmetric"]
    got = F.direct_evaluate(pts, symmetric=symmetric)
    assert F.max_rel_error(got, want) <= 1e-12


@pytest.mark.parametrize("n", [1, 2, 255, 513, 70_001])
def test_direct_symmetric_equals_asymmetric(n):
    """Ragged super-tiles and chunks: the shared-reciprocal sum agrees with the
    asymmetric one to roundoff, and is deterministic run to run."""
    pts = uniform(n, seed=21)
    sym = F.direct_evaluate(pts, symmetric=True)
    asym = F.direct_evaluate(pts)
    if n == 1:
        assert sym[0] == 0 and asym[0] == 0
        return
    # two different summation orders over n terms: compare against the size of
    # the terms, |dphi_i| / sum_j |g_j / (z_j - z_i)| (a plain relative bound
    # grows with n where cancellation makes |phi_i| small)
    import torch
    dev = torch.device("cuda", 0)
    z = torch.from_numpy(pts.positions).to(dev)
    g = torch.from_numpy(np.abs(pts.strengths)).to(dev)
    scale = torch.empty(n, dtype=torch.float64, device=dev)
    for s0 in range(0, n, 256):
        d = torch.abs(z[None, :] - z[s0:s0 + 256, None])
        t = g[None, :] / d
        t[d == 0] = 0.0
        scale[s0:s0 + 256] = t.sum(dim=1)
    cond = np.abs(sym - asym) / scale.cpu().numpy()
    assert cond.max() <= 1e-15 * max(1.0, np.sqrt(n) / 16)
    assert F.max_rel_error(sym, asym) <= 1e-11
    assert np.array_equal(sym, F.direct_evaluate(pts, symmetric=True))


def test_direct_separate_eval_points():
    pts = F.ParticleSet(np.array([0j, 1.0 + 0j]), np.array([2.0, -1.0]),
                        np.array([0.5 + 0j, 3.0 + 0j]))
    expected = [2.0 / (0 - 0.5) - 1.0 / (1 - 0.5), 2.0 / (0 - 3.0) - 1.0 / (1 - 3.0)]
    np.testing.assert_allclose(F.direct_evaluate(pts), expected, rtol=1e-15)


# --- pipeline (reference test_engine.py:73-173) ----------------------------------

def test_zero_level_pipeline_equals_direct():
    pts = uniform(100, seed=8)
    values, report = F.fmm_evaluate(pts, F.TreeConfig(n_desired_per_box=100))
    assert report.n_levels == 0
    assert F.max_rel_error(values, F.direct_evaluate(pts)) <= 1e-14


def test_accuracy_small_uniform():
    pts = uniform(3000, seed=5)
    values, report = F.fmm_evaluate(pts)
    assert F.max_rel_error(values, F.direct_evaluate(pts, symmetric=True)) <= 1e-5
    assert report.n_levels >= 2


def test_accuracy_separate_eval_points():
    rng = np.random.default_rng(12)
    pts = F.ParticleSet(rng.uniform(size=4000) + 1j * rng.uniform(size=4000),
                        rng.uniform(-1, 1, 4000), rng.uniform(size=700) + 1j * rng.uniform(size=700))
    values, _ = F.fmm_evaluate(pts)
    assert F.max_rel_error(values, F.direct_evaluate(pts)) <= 1e-5


def test_strength_doubling_scales_exactly():
    pts = uniform(2000, seed=6)
    v1, _ = F.fmm_evaluate(pts)
    v2, _ = F.fmm_evaluate(F.ParticleSet(pts.positions, 2.0 * pts.strengths))
    np.testing.assert_array_equal(v2, 2.0 * v1)


def test_determinism_bitwise():
    pts = uniform(30_000, seed=7)
    v1, _ = F.fmm_evaluate(pts)
    v2, _ = F.fmm_evaluate(pts)
    np.testing.assert_array_equal(v1, v2)


def test_parallel_flag_is_accepted():
    pts = uniform(6000, seed=9)
    seq, _ = F.fmm_evaluate(pts, parallel=False)
    par, rep = F.fmm_evaluate(pts, parallel=True, n_workers=4)
    assert rep.parallel
    np.testing.assert_array_equal(par, seq)


def test_degenerate_input_propagates():
    pts = F.ParticleSet(np.full(64, 0.25 + 0.75j), np.ones(64))
    with pytest.raises(F.DegenerateInputError, match="coincide"):
        F.fmm_evaluate(pts, F.TreeConfig(n_desired_per_box=1))
    with pytest.raises(F.DegenerateInputError, match="at level 0"):
        F.build_tree(F.ParticleSet(np.full(10, 0.5 + 0.5j), np.ones(10)),
                     F.TreeConfig(n_desired_per_box=1))


def test_coincident_sources_are_skipped_consistently():
    rng = np.random.default_rng(10)
    base = rng.uniform(size=600) + 1j * rng.uniform(size=600)
    z = np.concatenate([base, base[:25]])
    pts = F.ParticleSet(z, rng.uniform(-1, 1, z.size))
    values, report = F.fmm_evaluate(pts, F.TreeConfig(n_desired_per_box=20))
    assert F.max_rel_error(values, F.direct_evaluate(pts)) <= 1e-5
    assert report.coincident_skips == 2 * 25


def test_report_contents():
    _, report = F.fmm_evaluate(uniform(2000, seed=13))
    assert set(report.phase_seconds) == set(F.PHASE_NAMES)
    assert all(t >= 0 for t in report.phase_seconds.values())
    assert report.total_seconds >= sum(report.phase_seconds.values()) - 1e-6
    assert report.n_boxes == sum(4**l for l in range(report.n_levels + 1))
    assert 1 <= report.finest_src_min <= report.finest_src_mean <= report.finest_src_max
    assert sum(report.list_histograms["p2p"].values()) == 4**report.n_levels


def test_four_corners_and_clamp():
    pts = F.ParticleSet(np.array([0, 1, 1j, 1 + 1j], dtype=complex), np.ones(4))
    tree = F.build_tree(pts, F.TreeConfig(n_desired_per_box=1))
    assert tree.n_levels == 1
    np.testing.assert_array_equal(tree.finest.src_counts(), [1, 1, 1, 1])
    tree = F.build_tree(F.ParticleSet(np.array([0j, 1 + 0j, 1j]), np.ones(3)),
                        F.TreeConfig(n_desired_per_box=1))
    assert tree.n_levels == 0


def test_root_box_is_tight_bounding_rectangle():
    pts = F.ParticleSet(np.array([0.25 + 0.5j, 0.75 + 0.25j]), np.ones(2), np.array([0.1 + 0.9j]))
    root = F.build_tree(pts, F.TreeConfig()).levels[0]
    assert root.center[0] == pytest.approx(complex(0.425, 0.575))
    assert root.half_width[0] == pytest.approx(0.325)
    assert root.half_height[0] == pytest.approx(0.325)


def test_p_out_of_range_is_a_value_error():
    with pytest.raises(ValueError, match="p_terms"):
        F.fmm_evaluate(uniform(500), F.TreeConfig(p_terms=65))


# --- size-independent properties at BASELINE sizes ------------------------------

def _check_tree_invariants(tree, pts):
    n = pts.n_sources
    for lev, lv in enumerate(tree.levels):
        assert lv.n_boxes == 4**lev
        assert lv.src_offsets[0] == 0 and lv.src_offsets[-1] == n
        assert np.all(np.diff(lv.src_offsets) >= 0) and np.all(np.diff(lv.eval_offsets) >= 0)
    for lev in range(tree.n_levels):
        np.testing.assert_array_equal(tree.levels[lev].src_offsets,
                                      tree.levels[lev + 1].src_offsets[::4])
        np.testing.assert_array_equal(tree.levels[lev].eval_offsets,
                                      tree.levels[lev + 1].eval_offsets[::4])
    assert np.array_equal(np.sort(tree.src_perm), np.arange(n))
    np.testing.assert_array_equal(tree.src_pos, pts.positions[tree.src_perm])
    np.testing.assert_array_equal(tree.src_strength, pts.strengths[tree.src_perm])
    assert np.array_equal(np.sort(tree.eval_perm), np.arange(pts.n_evals))
    lv = tree.finest
    for pos, offsets in ((tree.src_pos, lv.src_offsets), (tree.eval_pos, lv.eval_offsets)):
        cnt = np.diff(offsets)
        cx = np.repeat(lv.center.real, cnt)
        cy = np.repeat(lv.center.imag, cnt)
        assert np.all(np.abs(pos.real - cx) <= np.repeat(lv.half_width, cnt) * (1 + 1e-12) + 1e-15)
        assert np.all(np.abs(pos.imag - cy) <= np.repeat(lv.half_height, cnt) * (1 + 1e-12) + 1e-15)
    counts = lv.src_counts()
    assert counts.max() - counts.min() <= 1
    # canonical in-box order: ascending original index
    starts = lv.src_offsets[:-1]
    d = np.diff(tree.src_perm)
    boundary = np.zeros(n - 1, bool)
    boundary[starts[1:] - 1] = True
    assert np.all((d > 0) | boundary)


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["uniform", "normal"])
def test_c2_scale_tree_invariants_and_accuracy(kind):
    pts = F.sample_points(F.DistributionSpec(kind, 0.01, 0), 1_000_000)
    cfg = F.TreeConfig(35, 0.5, 20)
    tree = F.build_tree(pts, cfg)
    assert tree.n_levels == 8
    _check_tree_invariants(tree, pts)
    values, report = F.fmm_evaluate(pts, cfg)
    assert report.retries <= 1
    # accuracy against the GPU direct sum on a sample of targets
    idx = np.random.default_rng(1).choice(pts.n_sources, 512, replace=False)
    probe = F.ParticleSet(pts.positions, pts.strengths, pts.positions[idx].copy())
    exact = F.direct_evaluate(probe)
    # the probes coincide with sources: direct skips them exactly like the FMM
    # FMM truncation at p=20 (the reference states ~1e-6 at p=17)
    assert F.max_rel_error(values[idx], exact) <= (1e-8 if kind == "uniform" else 1e-6)


@pytest.mark.slow
def test_c4_separate_p30_accuracy():
    src = F.sample_points(F.DistributionSpec("uniform", seed=0), 1_000_000)
    ev = F.sample_points(F.DistributionSpec("uniform", seed=1), 1_000_000).positions
    pts = F.ParticleSet(src.positions, src.strengths, ev)
    values, report = F.fmm_evaluate(pts, F.TreeConfig(35, 0.5, 30))
    idx = np.random.default_rng(2).choice(pts.n_evals, 256, replace=False)
    exact = F.direct_evaluate(F.ParticleSet(src.positions, src.strengths, ev[idx].copy()))
    assert F.max_rel_error(values[idx], exact) <= 1e-10
