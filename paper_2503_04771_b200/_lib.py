"""ctypes binding of libbgx.so (C ABI declared in include/bgx.h).

The structs below mirror include/bgx.h field for field; tests/test_abi.py
checks their sizes/offsets against the header (compiled with gcc) and that
every symbol the header declares is exported.  There is no CPU fallback: if
the library cannot be loaded, every entry point raises ``BackendUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# BGX_LIB: an alternative build of the same library (A/B experiments with
# csrc/Makefile's `exp` target); the product default is the in-tree .so
LIB_PATH = os.environ.get("BGX_LIB") or os.path.join(_HERE, "libbgx.so")

MAX_RANK = 8
MAX_AXES = 12
MAX_OPERANDS = 6
MAX_RANKS = 8

# bgx_dtype
F32, F64, BF16, F16 = 0, 1, 2, 3
# bgx_mode
MODE_AUTO, MODE_EXACT, MODE_FFMA, MODE_TC, MODE_SIMT, MODE_TF32 = 0, 1, 2, 3, 4, 5
# bgx_contract_kernel results
KERNEL_TC, KERNEL_EXACT, KERNEL_FFMA, KERNEL_SIMT16 = 1, 2, 3, 4
KERNEL_NAMES = {KERNEL_TC: "tcgen05", KERNEL_EXACT: "simt-exact",
                KERNEL_FFMA: "simt-ffma", KERNEL_SIMT16: "simt-16bit"}
# bgx_status
OK, ERR_INVALID, ERR_UNSUPPORTED, ERR_CUDA, ERR_NO_DEVICE = 0, -1, -2, -3, -4

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_vp = ctypes.c_void_p


class BgxTensor(ctypes.Structure):
    _fields_ = [("data", _vp), ("dtype", _i32), ("rank", _i32),
                ("shape", _i64 * MAX_RANK), ("stride", _i64 * MAX_RANK)]


class BgxGenericDesc(ctypes.Structure):
    _fields_ = [("n_in", _i32), ("n_axes", _i32), ("n_par", _i32), ("dtype", _i32),
                ("extents", _i64 * MAX_AXES), ("ins", _vp * MAX_OPERANDS),
                ("strides", (_i64 * MAX_AXES) * MAX_OPERANDS),
                ("c0", _vp), ("out", _vp)]


class BgxSchedule(ctypes.Structure):
    _fields_ = [("tile_n", _i32), ("stages", _i32), ("cta_group", _i32),
                ("max_ctas", _i32), ("raster", _i32), ("reserved", _i32 * 3)]


class BgxContractDesc(ctypes.Structure):
    _fields_ = [("batch", _i64), ("M", _i64), ("N", _i64), ("K", _i64),
                ("a", _vp), ("a_stride", _i64 * 3),
                ("b", _vp), ("b_stride", _i64 * 3),
                ("c0", _vp), ("c_stride", _i64 * 3),
                ("out", _vp), ("o_stride", _i64 * 3),
                ("in_dtype", _i32), ("out_dtype", _i32), ("mode", _i32), ("flags", _i32),
                ("sched", BgxSchedule)]


RS_IN_KERNEL, RS_DEFERRED = 0, 1     # bgx_rs_plan.mode


class BgxRsPlan(ctypes.Structure):
    _fields_ = [("world", _i32), ("rank", _i32), ("cta_group", _i32), ("tile_n", _i32),
                ("local_splits", _i32), ("out_dtype", _i32), ("mode", _i32), ("reserved0", _i32),
                ("rows_per_owner", _i64),
                ("slot_bytes", _i64), ("counter_bytes", _i64), ("ws_bytes", _i64)]


class BgxReduceScatter(ctypes.Structure):
    _fields_ = [("plan", BgxRsPlan), ("slots", _vp * MAX_RANKS), ("counters", _vp * MAX_RANKS),
                ("out", _vp * MAX_RANKS), ("c0", _vp * MAX_RANKS), ("ws", _vp),
                ("ws_counters", _vp)]


# name -> (restype, argtypes): exactly the functions include/bgx.h declares
SIGNATURES = {
    "bgx_version": (ctypes.c_int, []),
    "bgx_last_error": (ctypes.c_char_p, []),
    "bgx_sm_count": (ctypes.c_int, []),
    "bgx_permute": (ctypes.c_int, [ctypes.POINTER(BgxTensor), ctypes.POINTER(BgxTensor),
                                   ctypes.POINTER(_i32), _vp]),
    "bgx_generic": (ctypes.c_int, [ctypes.POINTER(BgxGenericDesc), _vp]),
    "bgx_contract": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc), _vp]),
    "bgx_contract_kernel": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc)]),
    "bgx_contract_tile": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc),
                                         ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "bgx_contract_splitk_plan": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc),
                                                ctypes.POINTER(_i32), ctypes.POINTER(_i64)]),
    "bgx_contract_splitk": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc), _i32, _vp, _i64,
                                           _vp]),
    "bgx_contract_rs_plan": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc), _i32,
                                            ctypes.POINTER(BgxRsPlan)]),
    "bgx_contract_reduce_scatter": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc),
                                                   ctypes.POINTER(BgxReduceScatter), _vp]),
    "bgx_rs_reduce": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc),
                                     ctypes.POINTER(BgxReduceScatter), _vp]),
    "bgx_cast_f32": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i64, _vp]),
    "bgx_clock_sample": (ctypes.c_int, [_vp, _vp]),
    "bgx_rtc_compile": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p,
                                       ctypes.POINTER(_vp), ctypes.c_char_p, _i64]),
    "bgx_rtc_launch": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint32,
                                      ctypes.POINTER(_vp), _vp]),
    "bgx_rtc_free": (ctypes.c_int, [_vp]),
    "bgx_contract_sharded": (ctypes.c_int, [ctypes.POINTER(BgxContractDesc), ctypes.POINTER(_i32),
                                            ctypes.POINTER(_vp), _i32]),
    "bgx_nccl_unique_id": (ctypes.c_int, [_vp]),
    "bgx_nccl_comm_init": (ctypes.c_int, [ctypes.POINTER(_vp), _i32, _i32, _vp]),
    "bgx_nccl_comm_destroy": (ctypes.c_int, [_vp]),
    "bgx_ksplit_reduce": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp]),
    "bgx_shutdown": (ctypes.c_int, []),
    "bgx_generic_tree_plan": (ctypes.c_int, [ctypes.POINTER(BgxGenericDesc), ctypes.POINTER(_i64)]),
    "bgx_generic_tree": (ctypes.c_int, [ctypes.POINTER(BgxGenericDesc), _vp, _i64, _vp]),
}


class BackendUnavailable(RuntimeError):
    """libbgx.so is missing or failed to load (there is no CPU fallback)."""


class BackendError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[bgx status {status}] {message}")
        self.status = status


class Unsupported(BackendError):
    pass


_lock = threading.Lock()
_lib = None


def load():
    """Load libbgx.so once (raises BackendUnavailable if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendUnavailable(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    " or `make -C paper_2503_04771_b200/csrc`")
            try:
                lib = ctypes.CDLL(LIB_PATH)
            except OSError as e:  # pragma: no cover - environment specific
                raise BackendUnavailable(f"cannot load {LIB_PATH}: {e}") from e
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.bgx_version() != 1:
                raise BackendUnavailable("libbgx.so ABI version mismatch")
            _lib = lib
    return _lib


def check(status: int, what: str):
    if status == OK:
        return
    msg = load().bgx_last_error().decode(errors="replace")
    if status == ERR_UNSUPPORTED:
        raise Unsupported(status, f"{what}: {msg}")
    raise BackendError(status, f"{what}: {msg}")
