"""bench.py host-side pieces (no GPU): the reference arm's JSON contract and
the per-phase roofline arithmetic."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_reference_arm_json():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--npoints", "3000", "--ref-cores", "2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "particles/s"
    assert line["value"] > 0 and line["cpu_baseline"]["cores"] == 2
    # the reference itself (oracle/_ref/site) on the bench's own config and N
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["cpu_baseline"]["same_config"] is True
    assert line["config"]["n_sources"] == 3000 and line["config"]["p"] == 20
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["metric"] == bench.METRIC


def test_phase_roofline_units():
    totals = {"weak": 3574218, "p2p": 887516, "p2l": 57286, "m2p": 57286}
    ms = {"sort": 0.5, "connect": 0.2, "p2m": 0.1, "m2m": 0.05, "m2l": 0.48, "l2l": 0.06,
          "l2p": 0.07, "p2p": 0.27}
    r = bench.phase_roofline(ms, totals, 10**6, 10**6, 8, 20, True, 36.5)
    # M2L: pairs x (2p(p+1) + 18p) flop / time
    expect = 3574218 * (2 * 20 * 21 + 18 * 20) / 0.48e-3 / 1e12
    assert abs(r["m2l"]["achieved"] - round(expect, 3)) < 1e-3
    assert r["sort"]["unit"] == "GB/s" and r["m2l"]["bound"] == "fp64"
    assert all(0 < v["frac"] < 1 for v in r.values())
