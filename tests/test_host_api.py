"""Host-side API surface of the drop-in (validation, level count, geometry
predicates, metric, CSV).  Mirrors the reference's own unit tests
(test_tree.py, test_geometry.py, test_engine.py).  CPU only."""

import csv

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1205_4611_b200 as F
from paper_1205_4611_b200 import (Box, InteractionLists, ParticleSet, TreeConfig, max_rel_error,
                                  num_levels, partition_median, split_direction, well_separated,
                                  well_separated_swapped, write_lists_csv)
from paper_1205_4611_b200.tree import clamped_levels


@pytest.mark.parametrize("n,nd,expected", [(2949120, 45, 8), (1179648, 45, 7), (45, 45, 0),
                                           (4, 1, 1)])
def test_num_levels(n, nd, expected):
    assert num_levels(n, nd) == expected
    lib = F._lib.load_library()
    assert lib.fmm2d_num_levels_raw(n, nd) == expected


def test_num_levels_rejects_bad_input():
    with pytest.raises(ValueError):
        num_levels(0, 45)


@pytest.mark.parametrize("n,nd", [(3, 1), (10, 1), (10_000, 35), (10**6, 35), (10**7, 35),
                                  (10**8, 35), (45 * 2**8, 45), (17, 100)])
def test_clamped_levels_agree_with_library(n, nd):
    assert clamped_levels(n, nd) == F._lib.load_library().fmm2d_num_levels(n, nd)


def test_partition_examples():
    coords = np.array([3.0, 1.0, 2.0])
    comp = np.arange(3)
    k = partition_median(coords, comp)
    assert k == 2 and sorted(coords[:2]) == [1.0, 2.0] and coords[2] == 3.0
    assert partition_median(np.array([5.0, 5.0, 5.0, 5.0]), np.arange(4)) == 2
    assert partition_median(np.array([1.0]), np.arange(1)) == 1


@given(st.lists(st.floats(min_value=-1e6, max_value=1e6, allow_nan=False), min_size=1,
                max_size=400))
@settings(max_examples=100, deadline=None)
def test_partition_matches_sort_oracle(values):
    coords = np.array(values)
    comp = np.arange(coords.size)
    original = coords.copy()
    k = partition_median(coords, comp)
    assert k == (coords.size + 1) // 2
    full = np.sort(values)
    np.testing.assert_array_equal(np.sort(coords[:k]), full[:k])
    np.testing.assert_array_equal(np.sort(coords[k:]), full[k:])
    np.testing.assert_array_equal(coords, original[comp])


def test_particle_set_validation():
    with pytest.raises(ValueError):
        ParticleSet(np.array([], dtype=complex), np.array([]))
    with pytest.raises(ValueError):
        ParticleSet(np.array([0j, 1j]), np.array([1.0]))
    with pytest.raises(ValueError):
        ParticleSet(np.array([0j]), np.array([np.nan]))
    with pytest.raises(ValueError, match="eval_positions"):
        ParticleSet(np.array([0j]), np.array([1.0]), np.array([np.inf + 0j]))
    p = ParticleSet(np.array([0j, 1j]), np.ones(2))
    assert p.evals_alias_sources and p.n_evals == 2


def test_tree_config_validation():
    for kw in (dict(theta=1.5), dict(n_desired_per_box=0), dict(p_terms=0), dict(theta=0.0)):
        with pytest.raises(ValueError):
            TreeConfig(**kw)
    assert TreeConfig() == TreeConfig(35, 0.5, 17)


def radius_box(center, r):
    return Box(center, 0.6 * r, 0.8 * r)


def test_geometry_substitution_cases():
    assert Box(0j, 3.0, 4.0).radius() == 5.0
    assert well_separated(radius_box(0j, 1.0), radius_box(3.0 + 0j, 1.0), 0.5)
    assert not well_separated(radius_box(0j, 1.0), radius_box(2.9 + 0j, 1.0), 0.5)
    assert well_separated(radius_box(0j, 2.0), radius_box(7.0 + 0j, 1.0), 0.5)
    a, b = radius_box(0j, 1.0), radius_box(2.0 + 0j, 0.2)
    assert not well_separated(a, b, 0.5) and well_separated_swapped(a, b, 0.5)
    assert well_separated_swapped(radius_box(0j, 1.0), Box(1.9 + 0j, 0.0, 0.0), 0.5)


@pytest.mark.parametrize("hw,hh,axis", [(2.0, 1.0, "x"), (1.0, 2.0, "y"), (1.5, 1.5, "x")])
def test_split_direction(hw, hh, axis):
    assert split_direction(Box(0j, hw, hh)) == axis


def test_max_rel_error_semantics():
    exact = np.array([1.0, 2.0, 4.0], dtype=complex)
    assert max_rel_error(exact, exact) == 0.0
    assert max_rel_error(1.01 * exact, exact) == pytest.approx(0.01, rel=1e-12)
    with pytest.raises(ValueError, match="zero"):
        max_rel_error(np.ones(2), np.zeros(2))
    with pytest.raises(ValueError, match="shapes"):
        max_rel_error(np.ones(2), np.ones(3))
    assert max_rel_error(np.array([123.0, 2.2]), np.array([0.0, 2.0])) == pytest.approx(0.1)


def test_write_lists_csv(tmp_path):
    lists = InteractionLists(1, [[np.empty(0, np.int64)], [np.array([2, 3]), np.empty(0, np.int64),
                                                           np.array([0]), np.array([0])]],
                             [np.array([0, 1])] * 4, [np.empty(0, np.int64)] * 4,
                             [np.empty(0, np.int64)] * 4)
    path = tmp_path / "l.csv"
    write_lists_csv(lists, path)
    rows = list(csv.DictReader(open(path)))
    assert len(rows) == 4 + 8
    assert {r["kind"] for r in rows} == {"weak", "p2p"}


def test_public_names_cover_reference_all():
    # the reference's complete __all__ (pkg/src/fmm2d/__init__.py:20-45)
    ref_all = {"Box", "BoxNode", "DegenerateInputError", "DistributionSpec", "EngineReport",
               "FmmTree", "InteractionLists", "ParticleSet", "TreeConfig", "build_connectivity",
               "build_tree", "classify_level", "direct_evaluate", "fmm_evaluate",
               "max_rel_error", "num_levels", "partition_median", "reclassify_finest",
               "sample_points", "split_direction", "well_separated", "well_separated_swapped",
               "write_lists_csv", "__version__"}
    assert ref_all <= set(F.__all__), ref_all - set(F.__all__)
    for name in ref_all:
        assert hasattr(F, name), name
    # submodules the reference's tests import (pkg/tests/*.py)
    from paper_1205_4611_b200 import connectivity, datasets, engine, geometry, operators, tree
    for fn in ("p2m", "p2l", "m2m", "l2l", "m2l", "l2p", "m2p", "reciprocal_parts",
               "kernel_block", "p2p_pair"):
        assert callable(getattr(operators, fn)), fn
    assert callable(engine._p2m_all)
    assert callable(connectivity.classify_level) and callable(connectivity.reclassify_finest)
    assert F.PHASE_NAMES == ("sort", "connect", "p2m", "m2m", "m2l", "l2l", "l2p", "p2p", "other")
