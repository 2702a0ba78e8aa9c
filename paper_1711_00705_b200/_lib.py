"""ctypes binding of libmdb200.so (the C ABI in include/mdb200.h).

There is deliberately no fallback: if the library is missing or cannot be
loaded, importing the package's device entry points fails loudly. ctypes
releases the GIL for every foreign call, like the reference's ``nogil``
kernels (/root/reference/pkg/src/minidist/_kernels/_accel.pyx:17,27).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from paper_1711_00705_b200 import errors

LIB_PATH = Path(__file__).resolve().parent / "libmdb200.so"

MD_MAX_RANKS = 16
MD_MAX_COLORS = 16
MD_MAX_WORKERS = 8
MD_SCHED_TREE = 0   # md_plan_set_schedule: per-color trees (the reference's schedule)
MD_SCHED_OWNER = 1  # owner-computes slices, same bits
MD_MAX_GROUP = 64
IPC_BYTES = 64
# md_plan_set_route / md_last_route (include/mdb200.h)
ROUTES = {"auto": 0, "tree": 1, "queue": 2, "ll": 3, "oneshot": 4, "stream": 5, "push": 6,
          "local": 7}
ROUTE_NAMES = {v: k for k, v in ROUTES.items()}
MD_UPDATE_REPLICATED = 0
MD_UPDATE_SHARDED = 1


class MdUpdate(C.Structure):
    """md_update_t (include/mdb200.h)."""

    _fields_ = [("w", C.POINTER(C.c_void_p)), ("mom", C.POINTER(C.c_void_p)),
                ("len", C.c_int64), ("c", C.c_float), ("mu", C.c_float), ("wd_b", C.c_float),
                ("mode", C.c_int32)]

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_f32 = C.c_float
_f64 = C.c_double
_pp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); every symbol include/mdb200.h declares
SIGNATURES = {
    "md_last_error": (C.c_char_p, []),
    "md_version": (C.c_int, []),
    "md_launch_count": (_u64, []),
    "md_add_f32": (C.c_int, [_vp, _i64, _vp, _i64, _vp]),
    "md_sub_scaled_f32": (C.c_int, [_vp, _i64, _vp, _i64, _f64, _vp]),
    "md_sgd_update": (C.c_int, [_vp, _vp, _vp, _i64, _f32, _f32, _f32, _vp]),
    "md_fill_rank_input": (C.c_int, [_vp, _i64, _i32, _i32, _vp]),
    "md_mem_export": (C.c_int, [_vp, C.c_char_p, C.POINTER(_u64)]),
    "md_mem_import": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "md_mem_close": (C.c_int, [_vp]),
    "md_enable_peer_access": (C.c_int, [C.c_int, C.c_int]),
    "md_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "md_comm_create": (C.c_int, [_i32, _i32, _i32, C.POINTER(_vp)]),
    "md_comm_destroy": (C.c_int, [_vp]),
    "md_comm_ctrl_ptr": (C.c_int, [_vp, C.POINTER(_vp)]),
    "md_comm_set_peer_ctrl": (C.c_int, [_vp, _pp, _i32]),
    "md_comm_take_error": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "md_comm_set_timeout": (C.c_int, [_vp, _f64]),
    "md_plan_create": (
        C.c_int,
        [_i32, _i32, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), _i32,
         C.POINTER(_vp)],
    ),
    "md_plan_destroy": (C.c_int, [_vp]),
    "md_plan_set_schedule": (C.c_int, [_vp, _i32]),
    "md_plan_set_route": (C.c_int, [_vp, _i32, _i64]),
    "md_last_route": (C.c_int, [_i32, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i32)]),
    "md_allreduce": (
        C.c_int,
        [_pp, _i32, _vp, _pp, _i64, _pp, _i32, _pp, _pp, _i64, _f32, _f32, _f32, _i64, _i32, _vp],
    ),
    "md_allreduce_ex": (
        C.c_int, [_pp, _i32, _vp, _pp, _i64, _pp, _i32, C.POINTER(MdUpdate), _i64, _i32, _vp]
    ),
    "md_trace_dump": (C.c_int, [_i32, C.c_char_p]),
    "md_mix64": (_u64, [C.POINTER(_u64), _i32]),
    "md_random_batch": (C.c_int, [_u64, _i64, _i64, _vp, _vp]),
    "md_stamp": (C.c_int, [_vp, _vp]),
    "md_random_batch_step": (C.c_int, [_u64, _u64, _u64, _vp, _i64, _i64, _vp, _vp]),
    "md_gather": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp]),
    "md_shuffle_plan": (
        C.c_int,
        [_u64, _u64, _i32, _i32, _u64, _i64, C.POINTER(_i64), _vp, _vp, _i64, C.POINTER(_i64),
         C.POINTER(_i64), _vp],
    ),
    "md_shuffle_index": (
        C.c_int, [_i32, _pp, _pp, _vp, _vp, _i64, _vp, _vp, _vp, C.POINTER(_u64), _vp]
    ),
    "md_shuffle_pull": (C.c_int, [_i32, _pp, _pp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "md_shuffle_sendlist": (C.c_int, [_i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "md_shuffle_push": (C.c_int, [_i32, _i32, _vp, _vp, _pp, _pp, _pp, _vp]),
    "md_copy_segments": (C.c_int, [_i32, _pp, _pp, C.POINTER(_u64), _vp]),
    "md_synth_records": (
        C.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _u64, C.c_uint32, _vp]
    ),
    "md_synth_verify": (
        C.c_int, [_vp, _vp, _vp, _vp, _i64, _u64, C.c_uint32, _vp, C.POINTER(_i64), _vp]
    ),
    "md_digest_f32": (C.c_int, [_vp, _i64, C.POINTER(_u64), _vp]),
    "md_toy_work_bytes": (_i64, [_i32, _i32, _i32, _i32]),
    "md_toy_grad": (C.c_int, [_vp, _i32, _i32, _i32, _pp, _i32, _pp, _i64, _i32, _pp, _i32, _vp,
                              _i64, _vp, _vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load (once) and return the library; raises ImportError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1711_00705_b200._build` "
            "(there is no CPU fallback for the device path)"
        )
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Raise the reference exception class mapped from an MD_ERR_* code."""
    if rc == 0:
        return
    msg = load().md_last_error().decode(errors="replace")
    cls = errors.FROM_CODE.get(rc, RuntimeError)
    raise cls(msg or f"libmdb200 error {rc}")


def _addr(p) -> int | None:
    if isinstance(p, C.c_void_p):
        return p.value
    return int(p) if p else None


def ptr_array(ptrs) -> C.Array:
    """Host array of device addresses (ints or opaque c_void_p handles)."""
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = _addr(p)
    return arr


def i32_array(vals) -> C.Array:
    arr = (C.c_int32 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr


def stream_ptr(stream) -> int | None:
    """cudaStream_t of a torch.cuda.Stream (None = legacy default stream)."""
    if stream is None:
        return None
    return int(stream.cuda_stream) or None


def last_route(device: int) -> tuple[str, int, bool]:
    """(route name, tile/segment elements, sharded) of the last md_allreduce
    this process launched on ``device``."""
    r, t, sh = C.c_int32(), C.c_int64(), C.c_int32()
    check(load().md_last_route(int(device), C.byref(r), C.byref(t), C.byref(sh)))
    return ROUTE_NAMES.get(r.value, str(r.value)), int(t.value), bool(sh.value)
