"""Bit-exactness of the θ-criterion magnitudes.  The device code
(csrc/common.cuh) and oracle/predicates.c hold the same formulas; here the C
restatement is pinned bitwise against numpy's np.hypot and np.abs(complex),
the two functions the reference calls (geometry.py:29, 40, 53).  CPU only."""

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "oracle" / "predicates.c"
LIB = ROOT / "oracle" / "_ref" / "libpredicates.so"


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        LIB.parent.mkdir(exist_ok=True)
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", str(LIB),
                        str(SRC), "-lm"], check=True)
    L = ctypes.CDLL(str(LIB))
    P = ctypes.POINTER(ctypes.c_double)
    for f in (L.orc_hypot_v, L.orc_cabs_v):
        f.argtypes = [P, P, P, ctypes.c_int64]
    return L


def _call(f, x, y):
    x = np.ascontiguousarray(x, float)
    y = np.ascontiguousarray(y, float)
    o = np.empty_like(x)
    P = ctypes.POINTER(ctypes.c_double)
    f(x.ctypes.data_as(P), y.ctypes.data_as(P), o.ctypes.data_as(P), x.size)
    return o


def _samples(n=400_000, seed=0):
    rng = np.random.default_rng(seed)
    mag = 2.0 ** rng.uniform(-40, 2, size=(2, n))
    x = mag[0] * rng.choice([-1, 1], n)
    y = mag[1] * rng.choice([-1, 1], n)
    x[:500] = 0.0
    y[500:1000] = 0.0
    x[1000:1500] = 2.0 ** rng.uniform(-1070, -1000, 500)
    x[1500:2000] = 2.0 ** rng.uniform(600, 1000, 500)
    # box-like half extents of a median-split unit square
    x[2000:4000] = rng.uniform(0, 0.5, 2000) / 2.0 ** rng.integers(0, 12, 2000)
    y[2000:4000] = rng.uniform(0, 0.5, 2000) / 2.0 ** rng.integers(0, 12, 2000)
    return x, y


def test_radius_is_bitwise_np_hypot(lib):
    x, y = _samples()
    assert np.array_equal(_call(lib.orc_hypot_v, x, y), np.hypot(x, y))


def test_distance_is_bitwise_np_abs_complex(lib):
    x, y = _samples(seed=1)
    assert np.array_equal(_call(lib.orc_cabs_v, x, y), np.abs(x + 1j * y))


def test_distance_short_arrays_and_tails(lib):
    x, y = _samples(seed=2)
    for m in range(1, 40):
        assert np.array_equal(_call(lib.orc_cabs_v, x[:m], y[:m]), np.abs(x[:m] + 1j * y[:m]))


def test_exact_boundary_3_4_5():
    # geometry tests pin 3-4-5 radii exactly (reference test_geometry.py:9-24)
    assert np.hypot(3.0, 4.0) == 5.0
