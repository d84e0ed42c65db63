"""ctypes binding of the CUDA library (include/ptap_b200.h).

The library is built in-tree (``_ptap_b200.so`` next to this file, see
``build.py``).  There is no CPU fallback: if the library is missing or no
CUDA device is present, every product entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError, OwnershipError, PartitionMismatchError, StructuralDriftError

_HERE = os.path.dirname(os.path.abspath(__file__))
# PTAP_LIB_PATH: an A/B build of the same library (csrc/Makefile VARIANT=...)
LIB_PATH = os.environ.get("PTAP_LIB_PATH") or os.path.join(_HERE, "_ptap_b200.so")

c_i64 = ctypes.c_int64
c_p = ctypes.c_void_p


class Csr(ctypes.Structure):
    _fields_ = [("nrows", c_i64), ("ncols", c_i64), ("nnz", c_i64),
                ("row_ptr", c_p), ("col", c_p), ("val", c_p)]


class Operands(ctypes.Structure):
    _fields_ = [("n_local", c_i64), ("m_global", c_i64), ("c_lo", c_i64), ("c_hi", c_i64),
                ("a_diag", Csr), ("a_off", Csr), ("p_diag", Csr), ("p_off", Csr),
                ("p_colmap", c_p), ("p_colmap_len", c_i64), ("p_remote", Csr)]


class Staging(ctypes.Structure):
    _fields_ = [("nrows", c_i64), ("nnz", c_i64), ("rows", c_p), ("row_ptr", c_p),
                ("col", c_p), ("val", c_p)]


class Received(ctypes.Structure):
    _fields_ = [("nsrc", ctypes.c_int32), ("src_rank", c_p), ("src_row_off", c_p), ("src_nnz_off", c_p),
                ("nrows", c_i64), ("nnz", c_i64), ("rows", c_p), ("row_ptr", c_p), ("col", c_p)]


class CView(ctypes.Structure):
    _fields_ = [("nrows", c_i64), ("ncols", c_i64), ("nnz", c_i64),
                ("row_ptr", c_p), ("col", c_p), ("val", c_p)]


class Memory(ctypes.Structure):
    _fields_ = [("current", c_i64 * 5), ("peak", c_i64 * 5), ("product_peak", c_i64),
                ("device_high_water", c_i64)]


class Counters(ctypes.Structure):
    _fields_ = [("symbolic_runs", c_i64), ("numeric_runs", c_i64),
                ("symbolic_row_kernel_calls", c_i64), ("numeric_row_kernel_calls", c_i64),
                ("kernel_launches", c_i64), ("nnz_c", c_i64), ("nnz_staging", c_i64),
                ("mac_ap", c_i64), ("mac_outer", c_i64), ("numeric_path", c_i64), ("map_bytes", c_i64),
                ("row_structures_ppm", c_i64)]


ALGORITHM_CODES = {"two-step": 0, "allatonce": 1, "merged": 2}

_EXPORTS = {
    "ptap_last_error": (ctypes.c_char_p, []),
    "ptap_version": (ctypes.c_char_p, []),
    "ptap_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(Operands), ctypes.POINTER(c_p)]),
    "ptap_plan_destroy": (ctypes.c_int, [c_p]),
    "ptap_plan_set_option": (ctypes.c_int, [c_p, ctypes.c_char_p, c_i64]),
    "ptap_plan_values_ready": (ctypes.c_int, [c_p, ctypes.POINTER(ctypes.c_int)]),
    "ptap_symbolic_send": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), c_p]),
    "ptap_plan_staging": (ctypes.c_int, [c_p, ctypes.POINTER(Staging)]),
    "ptap_symbolic_local": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), ctypes.POINTER(Received), c_p]),
    "ptap_numeric_send": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), c_p]),
    "ptap_numeric_local": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), c_p]),
    "ptap_numeric_merge": (ctypes.c_int, [c_p, c_p, c_p]),
    "ptap_numeric_local_rows": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), c_i64, c_i64, ctypes.c_int, c_p]),
    "ptap_plan_c_last_row": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), c_p, c_p]),
    "ptap_plan_check": (ctypes.c_int, [c_p, c_p]),
    "ptap_plan_status_async": (ctypes.c_int, [c_p, c_p]),
    "ptap_plan_status_poll": (ctypes.c_int, [c_p]),
    "ptap_pack_values": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), c_p, c_i64, c_p, c_p]),
    "ptap_plan_verify": (ctypes.c_int, [c_p, ctypes.POINTER(Operands), c_p]),
    "ptap_plan_get_ctilde": (ctypes.c_int, [c_p, ctypes.POINTER(CView)]),
    "ptap_plan_get_c": (ctypes.c_int, [c_p, ctypes.POINTER(CView)]),
    "ptap_plan_release_cache": (ctypes.c_int, [c_p]),
    "ptap_plan_memory": (ctypes.c_int, [c_p, ctypes.POINTER(Memory)]),
    "ptap_plan_counters": (ctypes.c_int, [c_p, ctypes.POINTER(Counters)]),
    "ptap_spgemm_ap_symbolic": (ctypes.c_int, [ctypes.POINTER(Operands), ctypes.POINTER(c_i64),
                                               ctypes.POINTER(c_p), ctypes.POINTER(c_p), c_p]),
    "ptap_spgemm_ap_numeric": (ctypes.c_int, [ctypes.POINTER(Operands), c_p, c_p, c_p, c_p]),
    "ptap_device_free": (ctypes.c_int, [c_p, c_p]),
    "ptap_transpose": (ctypes.c_int, [c_i64, c_i64, c_p, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p]),
    "ptap_gen_stencil_rowptr": (ctypes.c_int, [ctypes.c_int, c_i64, c_i64, c_i64, c_p,
                                               ctypes.POINTER(c_i64), c_p]),
    "ptap_gen_stencil_fill": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, c_i64, c_i64,
                                             c_i64, c_p, c_p, c_p, c_p]),
    "ptap_gen_trilinear_rowptr": (ctypes.c_int, [c_i64, c_i64, c_i64, c_p, ctypes.POINTER(c_i64), c_p]),
    "ptap_gen_trilinear_fill": (ctypes.c_int, [c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "ptap_gen_block_transport_rowptr": (ctypes.c_int, [c_i64, ctypes.c_int, c_i64, c_i64, c_i64, c_p,
                                                       ctypes.POINTER(c_i64), c_p, ctypes.POINTER(c_i64), c_p]),
    "ptap_gen_block_transport_a": (ctypes.c_int, [c_i64, ctypes.c_int, ctypes.c_uint64, c_i64, c_i64, c_p, c_p,
                                                  c_p, c_p]),
    "ptap_gen_spmv_dinv": (ctypes.c_int, [c_i64, c_p, c_p, c_p, c_p, c_p, c_p]),
    "ptap_gen_block_transport_p": (ctypes.c_int, [c_i64, ctypes.c_int, c_i64, ctypes.c_double, c_i64, c_i64, c_p,
                                                  c_p, c_p, c_p, c_p, c_p]),
    "ptap_gen_knn": (ctypes.c_int, [c_i64, c_p, c_p, ctypes.c_int, ctypes.c_int, c_p, c_p, c_p]),
    "ptap_l2_flush": (ctypes.c_int, [c_p]),
}

_lib = None


def exported_symbols() -> list:
    return sorted(_EXPORTS)


def load(require_device: bool = True):
    """Load the library; raise DeviceError (never fall back) when it is
    missing, or when ``require_device`` and no CUDA device is visible."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 triple product has no CPU path")
    return _lib


_STATUS_EXC = {1: ValueError, 2: PartitionMismatchError, 3: StructuralDriftError, 4: OwnershipError,
               5: DeviceError, 6: DeviceError}


def check(status: int, what: str = ""):
    if status != 0:
        msg = load(require_device=False).ptap_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(status, DeviceError)(f"{what}: {msg}" if what else msg)
