"""The C-ABI library loads and exports every symbol include/fmm2d.h declares.
No compute calls (CPU only)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1205_4611_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "fmm2d.h").read_text()
    return sorted(set(re.findall(r"\b(fmm2d_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_engine_entry_points():
    syms = declared_symbols()
    for must in ("fmm2d_create", "fmm2d_evaluate", "fmm2d_build_tree", "fmm2d_build_connectivity",
                 "fmm2d_direct", "fmm2d_export_tree", "fmm2d_export_lists"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    if not _lib.LIB_PATH.exists():
        pytest.fail(f"{_lib.LIB_PATH} not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_covers_the_header():
    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_binding_loads_and_host_only_calls_work():
    lib = _lib.load_library()
    # pure host entry points (no device needed)
    assert lib.fmm2d_num_levels(2949120, 45) == 8
    assert lib.fmm2d_num_levels(1179648, 45) == 7
    assert lib.fmm2d_num_levels(45, 45) == 0
    assert lib.fmm2d_num_levels(4, 1) == 1
    assert lib.fmm2d_num_levels(3, 1) == 0           # clamp: 4**L <= N
    assert lib.fmm2d_num_levels_raw(3, 1) == 1
    assert lib.fmm2d_num_levels(0, 45) == -1


def test_report_struct_layout():
    # phase_ms, device_ms, total_ms, n_levels+retries, n_boxes, min, max, mean,
    # skips, list_totals, max_len, h2d, d2h, kernel_launches
    assert ctypes.sizeof(_lib.Report) == 72 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 32 + 16 + 8 + 8 + 8
