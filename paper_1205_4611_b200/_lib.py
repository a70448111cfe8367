"""ctypes binding of libfmm2d.so (include/fmm2d.h) and a per-device context.

There is no CPU fallback: if the shared library or a CUDA device is missing,
every engine call raises.  The library is built in-tree by
``paper_1205_4611_b200._build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libfmm2d.so"

OK, EBADARG, EDEGENERATE, ESINGULAR, ECUDA, ENCCL, EOOM = 0, 2, 3, 5, 6, 7, 8
NPHASES = 9

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class Report(C.Structure):
    """fmm2d_report (include/fmm2d.h)."""

    _fields_ = [
        ("phase_ms", C.c_double * NPHASES),
        ("device_ms", C.c_double),
        ("total_ms", C.c_double),
        ("n_levels", C.c_int32),
        ("retries", C.c_int32),
        ("n_boxes", C.c_int64),
        ("finest_src_min", C.c_int64),
        ("finest_src_max", C.c_int64),
        ("finest_src_mean", C.c_double),
        ("p2p_skips", C.c_int64),
        ("list_totals", C.c_int64 * 4),
        ("max_len", C.c_int32 * 4),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("kernel_launches", C.c_int64),
    ]


_SIGS = {
    "fmm2d_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "fmm2d_destroy": (None, [C.c_void_p]),
    "fmm2d_last_error": (C.c_char_p, [C.c_void_p]),
    "fmm2d_num_levels": (C.c_int, [C.c_int64, C.c_int]),
    "fmm2d_num_levels_raw": (C.c_int, [C.c_int64, C.c_int]),
    "fmm2d_evaluate": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, C.c_int64, _dp, C.c_int,
                                 C.c_double, C.c_int, _dp, C.POINTER(Report)]),
    "fmm2d_evaluate_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_int64, C.c_void_p, C.c_int, C.c_double, C.c_int,
                                        C.c_void_p, C.POINTER(Report)]),
    "fmm2d_build_tree": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, C.c_int64, _dp, C.c_int,
                                   C.POINTER(C.c_int32)]),
    "fmm2d_degenerate_info": (C.c_int, [C.c_void_p, _i64p, _dp]),
    "fmm2d_export_tree": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _i64p, _i64p, _i64p, _i64p,
                                    _dp, _dp, _dp]),
    "fmm2d_build_connectivity": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_double]),
    "fmm2d_list_sizes": (C.c_int, [C.c_void_p, _i64p]),
    "fmm2d_export_lists": (C.c_int, [C.c_void_p] + [_i64p] * 8),
    "fmm2d_histogram": (C.c_int, [C.c_void_p, C.c_int, _i64p, C.c_int]),
    "fmm2d_export_expansions": (C.c_int, [C.c_void_p, _dp, _dp]),
    "fmm2d_export_phi": (C.c_int, [C.c_void_p, _dp]),
    "fmm2d_direct": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, C.c_int64, _dp, _dp]),
    "fmm2d_direct_symmetric": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, _dp]),
    # unit operators and per-level connectivity (operators.py, connectivity.py:47-96)
    "fmm2d_op_p2m": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _dp, _dp, _dp, C.c_int, _dp]),
    "fmm2d_op_p2l": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _dp, _dp, _dp, C.c_int, _dp]),
    "fmm2d_op_m2m": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, _dp, _dp, C.c_int]),
    "fmm2d_op_l2l": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, _dp, _dp]),
    "fmm2d_op_m2l": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, _dp, _dp, _dp]),
    "fmm2d_op_l2p": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp, C.c_int64, _dp, _dp]),
    "fmm2d_op_m2p": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp, C.c_int64, _dp, _dp]),
    "fmm2d_op_reciprocal_parts": (C.c_int, [C.c_void_p, C.c_int64, _dp, C.c_int64, _dp, _dp,
                                            _dp, _i64p]),
    "fmm2d_op_kernel_block": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, C.c_int64, _dp, _dp,
                                        _i64p]),
    "fmm2d_classify_level": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, _dp, _i64p, _i64p,
                                       C.c_double, _i64p, _i64p, _i64p, _i64p]),
    "fmm2d_reclassify_finest": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, _dp, _i64p, _i64p,
                                          C.c_double] + [_i64p] * 6),
    # distributed evaluation (one rank; collectives issued by the caller)
    "fmm2d_dist_setup": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_double,
                                   C.c_int, C.c_void_p, C.POINTER(C.c_int32)]),
    "fmm2d_dist_load": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                  C.c_void_p]),
    "fmm2d_dist_load_evals": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                        C.c_void_p]),
    "fmm2d_dist_eval_route": (C.c_int, [C.c_void_p, _i64p, C.POINTER(C.c_void_p)]),
    "fmm2d_dist_root": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fmm2d_dist_segbox": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "fmm2d_dist_check_segbox": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "fmm2d_dist_hist": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "fmm2d_dist_pick": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "fmm2d_dist_eqcount": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "fmm2d_dist_partition": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "fmm2d_dist_send_counts": (C.c_int, [C.c_void_p, _i64p, C.POINTER(C.c_void_p)]),
    "fmm2d_dist_build": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                   _i64p]),
    "fmm2d_dist_geom_pack": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fmm2d_dist_connect": (C.c_int, [C.c_void_p, C.c_void_p, _i64p]),
    "fmm2d_dist_requests": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "fmm2d_dist_item_doubles": (C.c_int, [C.c_void_p, C.c_int, _i64p]),
    "fmm2d_dist_pack": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]),
    "fmm2d_dist_unpack": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "fmm2d_dist_upward": (C.c_int, [C.c_void_p, C.c_void_p, _i64p]),
    "fmm2d_dist_upward_top": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fmm2d_dist_downward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Report)]),
    "fmm2d_scatter_values": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                       C.c_void_p]),
    "fmm2d_dist_end": (C.c_int, [C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load libfmm2d.so (raises if it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            # FMM2D_LIBRARY selects an alternative in-tree build (A/B measurements)
            path = Path(os.environ.get("FMM2D_LIBRARY", str(LIB_PATH)))
            if not path.exists():
                raise RuntimeError(
                    f"{path} is missing: build it with `python -m paper_1205_4611_b200._build` "
                    "(the engine has no CPU fallback)")
            lib = C.CDLL(str(path))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(_i64p)


class EngineError(RuntimeError):
    pass


class Context:
    """One libfmm2d context (device buffers, stream, events) on one GPU."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.fmm2d_create(C.byref(h), int(device))
        if rc != OK:
            raise EngineError(f"fmm2d_create failed on device {device} (code {rc}); "
                              "a CUDA device is required")
        self.h = h
        self.device = device
        self.lock = threading.RLock()

    def error(self) -> str:
        return self.lib.fmm2d_last_error(self.h).decode()

    def check(self, rc: int):
        if rc == OK:
            return
        msg = self.error()
        if rc == EDEGENERATE:
            from .tree import DegenerateInputError
            info = np.zeros(4, np.int64)
            xy = np.zeros(2)
            self.lib.fmm2d_degenerate_info(self.h, iptr(info), dptr(xy))
            raise DegenerateInputError(
                f"all {int(info[0])} source points in box {int(info[1])} at level "
                f"{int(info[2])} coincide at ({float(xy[0])}, {float(xy[1])}) but "
                f"{int(info[3])} more level(s) are required; reduce the level count or "
                "perturb the input")
        if rc in (EBADARG, ESINGULAR):
            raise ValueError(msg)
        if rc == EOOM:
            raise MemoryError(msg)
        raise EngineError(msg or f"libfmm2d error code {rc}")

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.fmm2d_destroy(self.h)
        except Exception:
            pass


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()


def default_context(device: int | None = None) -> Context:
    dev = 0 if device is None else int(device)
    with _ctx_lock:
        ctx = _contexts.get(dev)
        if ctx is None:
            ctx = Context(dev)
            _contexts[dev] = ctx
        return ctx
