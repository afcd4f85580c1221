"""ctypes binding of libmbgpu.so (C ABI declared in include/mbgpu.h).

There is no fallback: if the library is missing or no CUDA device is
present, :func:`load` raises :class:`NativeError` and the solver refuses to
run.  Build the library with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2005_05412_b200/csrc``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .reference import mblight


class NativeError(mblight.SolverError):
    """The CUDA library reported a failure (launch, allocation, argument), or
    it is missing: there is no CPU fallback."""


PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("MBGPU_LIB", PKG / "_build" / "libmbgpu.so"))
HEADER = PKG.parent / "include" / "mbgpu.h"

MBG_STEPPER = {"splitting": 0, "rk4": 1}
MBG_FLAG_PER_LAUNCH = 1
MBG_FLAG_PERSISTENT = 2
MBG_FLAG_DEFAULT_DEPTH = 4
MAX_REGIONS, MAX_QM, MAX_SOURCES, MAX_RECORDS, MAX_LEVELS, MAX_TILE_STEPS = 128, 4, 32, 64, 8, 128
MAX_BATCH_QM = 65536


class MbgGrid(C.Structure):
    _fields_ = [
        ("num_x", C.c_int64), ("num_t", C.c_int64), ("dt", C.c_double), ("dx", C.c_double),
        ("levels", C.c_int32), ("stepper", C.c_int32), ("tile_steps", C.c_int32),
        ("exact", C.c_int32), ("device", C.c_int32), ("flags", C.c_int32),
        ("win_lo", C.c_int64), ("win_hi", C.c_int64), ("own_lo", C.c_int64), ("own_hi", C.c_int64),
    ]


_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_h = C.c_void_p

# name -> (restype, argtypes); the exported surface of include/mbgpu.h
SIGNATURES = {
    "mbg_create": (C.c_int, [C.POINTER(MbgGrid), C.POINTER(_h)]),
    "mbg_destroy": (None, [_h]),
    "mbg_last_error": (C.c_char_p, [_h]),
    "mbg_version": (C.c_char_p, []),
    "mbg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "mbg_set_stream": (C.c_int, [_h, C.c_uint64]),
    "mbg_tile_steps": (C.c_int, [_h, _i32p]),
    "mbg_set_regions": (C.c_int, [_h, C.c_int32, _i64p, _i64p, _dp, _dp, _dp, _dp, _i32p]),
    "mbg_set_qm_bloch": (C.c_int, [_h, C.c_int32, _dp]),
    "mbg_set_qm_dense": (C.c_int, [_h, C.c_int32, _dp, _dp, _dp, _dp, C.c_int32, _i32p, _i32p, _dp,
                                   C.c_int32, _i32p, _dp, C.c_double]),
    "mbg_set_qm_rk4": (C.c_int, [_h, C.c_int32, _dp, _dp, _dp, _dp, C.c_int32, _i32p, _i32p, _dp,
                                 C.c_int32, _i32p, _dp, C.c_double]),
    "mbg_set_boundary": (C.c_int, [_h] + [C.c_double] * 6),
    "mbg_set_sources": (C.c_int, [_h, C.c_int32, _i64p, _i32p, _dp]),
    "mbg_set_source_rows": (C.c_int, [_h, C.c_int64, C.c_int64, _dp]),
    "mbg_stream_idle": (C.c_int, [_h, _i32p]),
    "mbg_set_records": (C.c_int, [_h, C.c_int32, _i32p, _i64p, _i32p, _i32p, _i64p]),
    "mbg_upload_fields": (C.c_int, [_h, _dp, _dp]),
    "mbg_upload_density": (C.c_int, [_h, _dp]),
    "mbg_upload_state": (C.c_int, [_h, _dp]),
    "mbg_download_fields": (C.c_int, [_h, _dp, _dp]),
    "mbg_download_state": (C.c_int, [_h, _dp]),
    "mbg_sample": (C.c_int, [_h, C.c_int64]),
    "mbg_advance": (C.c_int, [_h, C.c_int64, C.c_int64]),
    "mbg_synchronize": (C.c_int, [_h]),
    "mbg_poll_nonfinite": (C.c_int, [_h, _i64p]),
    "mbg_invariants": (C.c_int, [_h, _dp]),
    "mbg_invariants_accumulate": (C.c_int, [_h]),
    "mbg_invariants_read": (C.c_int, [_h, _dp]),
    "mbg_set_monitor": (C.c_int, [_h, C.c_int64]),
    "mbg_record_shape": (C.c_int, [_h, C.c_int32, _i64p, _i64p]),
    "mbg_download_record": (C.c_int, [_h, C.c_int32, _dp, _dp]),
    "mbg_set_record_rows": (C.c_int, [_h, C.c_int32, C.c_int64]),
    "mbg_download_record_rows": (C.c_int, [_h, C.c_int32, C.c_int64, C.c_int64, _dp, _dp]),
    "mbg_set_record_row0": (C.c_int, [_h, C.c_int32, C.c_int64]),
    "mbg_batch_points": (C.c_int, [_h, C.c_int32, _i32p, _dp, _dp, C.c_int32, _i32p, _i32p, _i32p, _i64p,
                                   C.POINTER(_dp), C.POINTER(_dp)]),
    "mbg_halo_words": (C.c_int, [_h, _i32p]),
    "mbg_pack_halo": (C.c_int, [_h, C.c_int64, C.c_int64, C.c_uint64]),
    "mbg_unpack_halo": (C.c_int, [_h, C.c_int64, C.c_int64, C.c_uint64]),
    "mbg_mailbox_alloc": (C.c_int, [C.c_int32, C.c_int64, C.POINTER(C.c_uint64), C.c_char_p]),
    "mbg_mailbox_free": (C.c_int, [C.c_int32, C.c_uint64]),
    "mbg_mailbox_map": (C.c_int, [C.c_int32, C.c_char_p, C.POINTER(C.c_uint64)]),
    "mbg_mailbox_unmap": (C.c_int, [C.c_int32, C.c_uint64]),
    "mbg_push_halo": (C.c_int, [_h, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "mbg_pull_halo": (C.c_int, [_h, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64]),
    "mbg_checkpoint_save": (C.c_int, [_h]),
    "mbg_checkpoint_restore": (C.c_int, [_h]),
    "mbg_fp64_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "mbg_fp64_peak_operands": (C.c_int, [C.c_int, C.c_int32, C.POINTER(C.c_double)]),
    "mbg_fp64_peak_sustained": (C.c_int, [C.c_int, C.c_double, C.POINTER(C.c_double)]),
    "mbg_event_begin": (C.c_int, [_h]),
    "mbg_event_end": (C.c_int, [_h, C.POINTER(C.c_float)]),
    "mbg_mark": (C.c_int, [_h, C.c_int32]),
    "mbg_mark_elapsed": (C.c_int, [_h, C.c_int32, C.c_int32, C.POINTER(C.c_float)]),
    "mbg_launch_count": (C.c_int, [_h, _i64p]),
}

MBG_IPC_HANDLE_BYTES = 64  # include/mbgpu.h

_LIB = None


def load(require_device: bool = True):
    """Load libmbgpu.so (once).  Raises NativeError when it is absent, or when
    ``require_device`` and no CUDA device is visible."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH} is missing: build it with `make -C {PKG / 'csrc'}` "
                "(the GPU solver has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    if require_device:
        n = C.c_int(0)
        if _LIB.mbg_device_count(C.byref(n)) != 0 or n.value < 1:
            raise NativeError("no CUDA device visible to libmbgpu.so (the GPU solver has no CPU fallback)")
    return _LIB


def ptr(a, kind=_dp):
    if a is None:
        return C.cast(None, kind)
    return a.ctypes.data_as(kind)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class Handle:
    """Owning wrapper of one ``mbg_solver``; every call is checked."""

    def __init__(self, grid: MbgGrid):
        self.lib = load()
        h = _h()
        rc = self.lib.mbg_create(C.byref(grid), C.byref(h))
        if rc != 0 or not h.value:
            raise NativeError(f"mbg_create failed ({rc}): invalid grid/window or CUDA error")
        self.h = h

    def call(self, name, *args):
        rc = getattr(self.lib, name)(self.h, *args)
        if rc != 0:
            msg = self.lib.mbg_last_error(self.h).decode(errors="replace")
            raise NativeError(f"{name} failed ({rc}): {msg}")

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.mbg_destroy(self.h)
            self.h = _h()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
