"""Parity at the headline configurations (C2-C5) against the REFERENCE.

Fixtures: tests/golden/make_golden_large.py ran the reference's own
``fmm_evaluate`` (sequential) on the bench's exact inputs and stored one
SHA-256 per canonical tree field and per CSR list field, the report's
histograms/skips, and sampled potentials (10k uniform + the 2k points of
smallest |phi|).  Here the GPU engine runs the same evaluation through the
public API; the tree and lists that evaluation actually used are exported
from the context (the C5 path: 32-bit rank keys, records from
``k_init_arrays``) and hashed with the same canonicalisation.

Bar (BASELINE.json north_star): tree and lists bit-exact; potentials
<= 1e-12 relative at C2-C4.  At C5 (1e7) the reference itself is only
self-consistent to 1.12e-12 (same input, default vs
SIMD-off numpy), so the bound there is that ISA floor and the test also
reports the condition-normalised error |dphi| / sum_j |g_j / (z_j - y)|.
"""

import numpy as np
import pytest

import paper_1205_4611_b200 as F
from paper_1205_4611_b200 import _lib
from paper_1205_4611_b200.connectivity import export_lists
from paper_1205_4611_b200.tree import export_tree

from helpers import flat_lists_pkg, flat_tree_pkg, load, sha

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HEADLINE = {
    # fixture: (kind, n, separate evals, p, potential bound)
    "c2_uniform_1e6_p20": ("uniform", 1_000_000, False, 20, 1e-12),
    "c3_normal_1e6_p20": ("normal", 1_000_000, False, 20, 1e-12),
    "c4_separate_1e6_p30": ("uniform", 1_000_000, True, 30, 1e-12),
    "c5_uniform_1e7_p20": ("uniform", 10_000_000, False, 20, None),   # see the ISA floor
}


def _inputs(kind, n, separate):
    pts = F.sample_points(F.DistributionSpec(kind, 0.01, 0), n)
    if separate:
        ev = F.sample_points(F.DistributionSpec("uniform", 0.01, 1), n).positions
        pts = F.ParticleSet(pts.positions, pts.strengths, ev)
    return pts


def _cond_norm_error(pts, idx, got, want):
    """max_i |got_i - want_i| / sum_j |g_j| / |z_j - y_i| (GPU, fp64 torch)."""
    import torch
    dev = torch.device("cuda", 0)
    z = torch.from_numpy(pts.positions).to(dev)
    g = torch.from_numpy(np.abs(pts.strengths)).to(dev)
    y = torch.from_numpy(pts.eval_positions[idx]).to(dev)
    denom = torch.empty(idx.size, dtype=torch.float64, device=dev)
    for s in range(0, idx.size, 16):
        d = torch.abs(z[None, :] - y[s:s + 16, None])
        t = g[None, :] / d
        t[d == 0] = 0.0
        denom[s:s + 16] = t.sum(dim=1)
    return float(np.max(np.abs(got - want) / denom.cpu().numpy()))


@pytest.mark.parametrize("name", list(HEADLINE))
def test_headline_config_matches_reference(name):
    rec = load(name)
    kind, n, separate, p, bound = HEADLINE[name]
    pts = _inputs(kind, n, separate)
    assert pts.n_sources == int(rec["n_sources"]) and pts.n_evals == int(rec["n_evals"])
    cfg = F.TreeConfig(35, 0.5, p)
    values, report = F.fmm_evaluate(pts, cfg)

    ctx = _lib.default_context(None)
    with ctx.lock:
        tree = export_tree(ctx, report.n_levels, pts.n_sources, pts.n_evals)
        lists = export_lists(ctx, report.n_levels)
    assert report.n_levels == int(rec["n_levels"])
    ft = flat_tree_pkg(tree)
    bad = [k for k in ft if sha(ft[k]) != str(rec["tree_sha_" + k])]
    assert not bad, f"tree fields differ from the reference: {bad}"
    fl = flat_lists_pkg(lists)
    bad = [k for k in fl if sha(fl[k]) != str(rec["lists_sha_" + k])]
    assert not bad, f"list fields differ from the reference: {bad}"

    assert report.n_boxes == int(rec["n_boxes"])
    assert report.coincident_skips == int(rec["coincident_skips"])
    assert report.finest_src_min == int(rec["finest_src_min"])
    assert report.finest_src_max == int(rec["finest_src_max"])
    for k in ("weak", "p2p", "p2l", "m2p"):
        want = {int(a): int(b) for a, b in rec[f"hist_{k}"]}
        assert report.list_histograms[k] == want, k

    idx = rec["sample_idx"]
    want = rec["sample_values"]
    got = values[idx]
    rel = np.abs(got - want) / np.abs(want)
    worst = float(rel.max())
    msg = f"{name}: max rel {worst:.3e} over {idx.size} sampled points"
    if bound is None:
        # 1e7: the reference is not reproducible to 1e-12 itself.  Its potentials
        # from numpy with SIMD dispatch disabled (same input, same code) differ
        # from the default build by up to floor = 1.12e-12 at these points
        # (tests/golden/*_isa.npz, make_golden_large.py --isa-variant).  Bar: the
        # GPU stays within 2x that floor everywhere, no more points above 1e-12
        # than twice the reference's own count, and a condition-normalised
        # error |dphi| / sum_j |g_j / (z_j - y)| far below double rounding.
        isa = load(name + "_isa")
        assert np.array_equal(isa["sample_idx"], idx)
        rel_isa = np.abs(isa["sample_values_isa"] - want) / np.abs(want)
        floor = float(rel_isa.max())
        cond = _cond_norm_error(pts, idx, got, want)
        msg += (f" | reference ISA floor {floor:.3e} ({int((rel_isa > 1e-12).sum())} points"
                f" > 1e-12; GPU {int((rel > 1e-12).sum())}) | condition-normalised {cond:.2e}")
        print(msg)
        assert worst <= 2 * floor, msg
        assert (rel > 1e-12).sum() <= 2 * max(1, (rel_isa > 1e-12).sum()), msg
        assert cond <= 1e-16, msg
    else:
        msg += f" (bound {bound:.2e})"
        print(msg)
        assert worst <= bound, msg
