"""ctypes binding of libmdsx.so (the C-ABI in include/mdsx.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises ``RuntimeError`` naming what is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import (DegenerateRankError, FormatError, InvalidInputError, MdsError,
                     NumericalError, ParamError, ShapeError)

LIB_PATH = Path(__file__).resolve().parent / "libmdsx.so"
# A/B measurements only (tools/): load another build of the library; entry
# points it lacks are left unbound
_LIB_OVERRIDE = os.environ.get("MDSX_LIB")
if _LIB_OVERRIDE:
    LIB_PATH = Path(_LIB_OVERRIDE).resolve()

OK, PARAM, SHAPE, INVALID, NUMERICAL, DEGENERATE, CUDA, UNSUPPORTED, FORMAT = range(9)
F64, F32 = 0, 1


class PieceStatus(C.Structure):
    _fields_ = [("code", C.c_int32), ("index", C.c_int32), ("value", C.c_double)]


class FastPlanC(C.Structure):
    """mdsx_fast_plan (include/mdsx.h)."""
    _fields_ = [("npieces", C.c_int32), ("n_leaves", C.c_int32), ("nlevels", C.c_int32),
                ("piece_off", C.c_void_p), ("row_idx", C.c_void_p), ("out_idx", C.c_void_p),
                ("ntracked", C.c_int64), ("trk_row", C.c_void_p), ("trk_leaf", C.c_void_p),
                ("level_njobs", C.c_void_p), ("job_off", C.c_void_p), ("job_src", C.c_void_p),
                ("job_tgt", C.c_void_p), ("trk_job", C.c_void_p), ("leaf_job", C.c_void_p)]


_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_int = C.c_int

# name -> (restype, argtypes)
SIGNATURES = {
    "mdsx_version": (_int, []),
    "mdsx_create": (_int, [_int, C.POINTER(_vp)]),
    "mdsx_destroy": (None, [_vp]),
    "mdsx_last_error": (C.c_char_p, [_vp]),
    "mdsx_launch_count": (_i64, [_vp]),
    "mdsx_timing_enable": (_int, [_vp, _int]),
    "mdsx_timing_report": (_i64, [_vp, C.c_char_p, _i64]),
    "mdsx_timing_trace": (_i64, [_vp, C.c_char_p, _i64]),
    "mdsx_sqdist_self": (_int, [_vp, _vp, _int, _i64, _i64, _i32, _vp, _i64, _vp]),
    "mdsx_sqdist_cross": (_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _int, _i32, _vp, _i64, _vp]),
    "mdsx_double_center": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "mdsx_sym_eigvals": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "mdsx_delta_check": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "mdsx_classical_pieces": (_int, [_vp, _vp, _int, _i64, _i32, _vp, _vp, _i32, _i32,
                                     _vp, _vp, _vp, _vp, _vp]),
    "mdsx_classical_delta": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "mdsx_gower_context_size": (_i64, [_i64, _i32, _i32]),
    "mdsx_gower_context": (_int, [_vp, _vp, _int, _i64, _i32, _vp, _i64, _vp, _i32, _vp, _vp,
                                  _vp, _vp]),
    "mdsx_gower_interpolate": (_int, [_vp, _vp, _i64, _i32, _i32, _vp, _int, _i64, _i64, _vp,
                                      _i64, _vp, _i32, _vp]),
    "mdsx_gower_tile_rows": (_i32, [_vp, _int, _i32, _i32]),
    "mdsx_gower_tiles": (_int, [_vp, _vp, _i64, _i32, _i32, _vp, _int, _i64, _vp, _vp, _vp, _i32,
                                _vp]),
    "mdsx_landmark_overwrite": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _vp]),
    "mdsx_interp_recenter": (_int, [_vp, _vp, _i64, _vp, _i64, _i32, _i64, _vp, _i64, _vp]),
    "mdsx_procrustes_fit": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp,
                                   _vp, _vp]),
    "mdsx_procrustes_apply": (_int, [_vp, _vp, _i32, _vp, _vp, _i32, _i64, _vp, _vp, _vp]),
    "mdsx_scatter_rows": (_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "mdsx_recenter": (_int, [_vp, _vp, _i64, _i32, _vp]),
    "mdsx_fast_mds": (_int, [_vp, _vp, _int, _i64, _i32, C.POINTER(FastPlanC), _i32, _i64, _i32,
                              _vp, _vp, _vp, _vp, _vp]),
    "mdsx_fast_finish": (_int, [_vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _i64, _vp, _vp]),
    "mdsx_divide_conquer": (_int, [_vp, _vp, _int, _i64, _i64, _i32, _vp, _vp, _i32, _i32, _i32,
                                   _vp, _vp, _vp, _vp, _vp]),
    "mdsx_divide_conquer_ex": (_int, [_vp, _vp, _int, _i64, _i64, _i32, _vp, _vp, _i32, _i32, _i32,
                                      _vp, _vp, _vp, _vp, _i32, _vp]),
    "mdsx_divide_conquer_sharded": (_int, [_vp, _vp, _int, _i64, _i64, _i32, _vp, _vp, _i32, _i32,
                                           _i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp,
                                           _vp]),
    "mdsx_fast_mds_sharded": (_int, [_vp, _vp, _int, _i64, _i32, C.POINTER(FastPlanC), _i32, _i64,
                                     _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "mdsx_segment_colsums": (_int, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "mdsx_shift_rows": (_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "mdsx_interpolation": (_int, [_vp, _vp, _int, _i64, _i64, _i32, _vp, _i64, _i32, _vp, _vp,
                                  _vp, _vp, _vp, _vp, _vp]),
    "mdsx_aligned_correlations": (_int, [_vp, _vp, _i64, _i32, _vp, _i32, _i64, _vp, _vp, _vp,
                                         _vp]),
    "mdsx_h2d": (_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "mdsx_active_columns": (_int, [_vp, _vp, _int, _i64, _i64, _i32, _vp, C.POINTER(_i32), _vp]),
    "mdsx_gather_columns": (_int, [_vp, _vp, _int, _i64, _i64, _vp, _i32, _i64, _vp, _vp]),
    "mdsx_plan_choices": (_int, [_vp, _i32, _i32, _vp, _vp, C.POINTER(_i32), C.POINTER(C.c_uint32)]),
    "mdsx_plan_permute": (_int, [_vp, _i64, _vp, C.POINTER(_i32), C.POINTER(C.c_uint32)]),
    "mdsx_idx_probe": (_int, [C.c_char_p, _i32, C.POINTER(_i64), C.POINTER(_i32),
                              C.POINTER(_i32), C.c_char_p, _i64]),
    "mdsx_idx_load_images": (_int, [_vp, C.c_char_p, _vp, _int, C.c_double, _vp]),
    "mdsx_csv_read": (_int, [C.c_char_p, _i32, _i32, _vp, C.POINTER(_i64), C.POINTER(_i64),
                             C.c_char_p, _i64]),
}

# host callback of mdsx_divide_conquer_sharded: int gather(void* ctx, void* stream)
GATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)

_lib = None
_lib_lock = threading.Lock()


def load() -> C.CDLL:
    """Load and type the shared library (no device work)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2007_11919_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                if _LIB_OVERRIDE and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class Handle:
    """One mdsx_handle per CUDA device (owns that device's workspace)."""

    _by_device: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int):
        lib = load()
        ptr = C.c_void_p()
        rc = lib.mdsx_create(device, C.byref(ptr))
        if rc != OK:
            raise RuntimeError(f"mdsx_create(device={device}) failed with status {rc}")
        self.ptr = ptr
        self.device = device
        self.lib = lib

    @classmethod
    def get(cls, device: int) -> "Handle":
        with cls._lock:
            h = cls._by_device.get(device)
            if h is None:
                h = cls._by_device[device] = Handle(device)
            return h

    def launches(self) -> int:
        return int(self.lib.mdsx_launch_count(self.ptr))

    def timing(self, on: bool) -> None:
        self.lib.mdsx_timing_enable(self.ptr, 1 if on else 0)

    def timing_report(self, with_work: bool = False) -> dict:
        """{kernel: (total_ms, launches)} since the last report; with_work:
        (total_ms, launches, executed flops credited by the launcher or 0)."""
        n = int(self.lib.mdsx_timing_report(self.ptr, None, 0))
        buf = C.create_string_buffer(n + 1)
        self.lib.mdsx_timing_report(self.ptr, buf, n + 1)
        out = {}
        for line in buf.value.decode().splitlines():
            name, ms, cnt, work = line.split()
            out[name] = (float(ms), int(cnt), float(work)) if with_work else (float(ms), int(cnt))
        return out

    def timing_trace(self) -> list:
        """[(kernel, start_ms, end_ms)] of the launches timed since the last
        report, relative to the first (mdsx_timing_trace)."""
        n = int(self.lib.mdsx_timing_trace(self.ptr, None, 0))
        buf = C.create_string_buffer(n + 1)
        self.lib.mdsx_timing_trace(self.ptr, buf, n + 1)
        out = []
        for line in buf.value.decode().splitlines():
            name, a, b = line.split()
            out.append((name, float(a), float(b)))
        return out

    def call(self, name: str, *args) -> None:
        rc = getattr(self.lib, name)(self.ptr, *args)
        if rc != OK:
            msg = self.lib.mdsx_last_error(self.ptr).decode(errors="replace")
            raise status_error(rc, msg or name)


def status_error(code: int, msg: str) -> Exception:
    return {
        PARAM: ParamError, SHAPE: ShapeError, INVALID: InvalidInputError,
        NUMERICAL: NumericalError, DEGENERATE: DegenerateRankError, FORMAT: FormatError,
    }.get(code, MdsError if code == UNSUPPORTED else RuntimeError)(msg)


def total_launches() -> int:
    return sum(h.launches() for h in Handle._by_device.values())
