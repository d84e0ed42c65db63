"""ctypes front end of the CPU oracle (oracle/ptap_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs import this module,
and only as the checker or the timed CPU baseline -- never as the product.

The C file restates the reference algorithms (``/root/reference/pkg/src/ptap``,
see the file:line map in its header) with the reference's exact per-entry
summation order, so its output is bit-identical to the reference at the same
rank count; ``tests/test_oracle_golden.py`` pins that against fixtures
generated from the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libptap_oracle.so")

ALGORITHM_CODES = {"two-step": 0, "allatonce": 1, "merged": 2}


class OracleStats(ctypes.Structure):
    _fields_ = [
        ("rows_sym", ctypes.c_int64),
        ("rows_num", ctypes.c_int64),
        ("nnz_c", ctypes.c_int64),
        ("mac_ap", ctypes.c_int64),
        ("mac_outer", ctypes.c_int64),
        ("staged_entries", ctypes.c_int64),
    ]


_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (make in oracle/); returns the .so path."""
    src = os.path.join(_HERE, "ptap_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        p64 = ctypes.POINTER(ctypes.c_int64)
        pd = ctypes.POINTER(ctypes.c_double)
        L.ptap_oracle_symbolic.restype = ctypes.c_void_p
        L.ptap_oracle_symbolic.argtypes = [ctypes.c_int64, ctypes.c_int64, p64, p64, p64, p64,
                                           ctypes.c_int, ctypes.c_int, ctypes.POINTER(OracleStats)]
        L.ptap_oracle_nnz.restype = ctypes.c_int64
        L.ptap_oracle_nnz.argtypes = [ctypes.c_void_p]
        L.ptap_oracle_pattern.restype = None
        L.ptap_oracle_pattern.argtypes = [ctypes.c_void_p, p64, p64]
        L.ptap_oracle_numeric.restype = ctypes.c_int
        L.ptap_oracle_numeric.argtypes = [ctypes.c_void_p, p64, p64, pd, p64, p64, pd, pd,
                                          ctypes.POINTER(OracleStats)]
        L.ptap_oracle_free.restype = None
        L.ptap_oracle_free.argtypes = [ctypes.c_void_p]
        L.ptap_oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


@dataclass
class OracleResult:
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    stats: dict


class OraclePlan:
    """Symbolic once, numeric many times -- the reference's plan protocol."""

    def __init__(self, n, m, a_ip, a_j, p_ip, p_j, nranks=1, algorithm="allatonce"):
        self.n, self.m = int(n), int(m)
        self._a_ip, self._a_j = _i64(a_ip), _i64(a_j)
        self._p_ip, self._p_j = _i64(p_ip), _i64(p_j)
        self.sym_stats = OracleStats()
        L = lib()
        self._h = L.ptap_oracle_symbolic(
            self.n, self.m, _p(self._a_ip, ctypes.c_int64), _p(self._a_j, ctypes.c_int64),
            _p(self._p_ip, ctypes.c_int64), _p(self._p_j, ctypes.c_int64),
            int(nranks), ALGORITHM_CODES[algorithm], ctypes.byref(self.sym_stats))
        self.nnz = int(L.ptap_oracle_nnz(self._h))
        self.row_ptr = np.empty(self.m + 1, np.int64)
        self.col = np.empty(self.nnz, np.int64)
        L.ptap_oracle_pattern(self._h, _p(self.row_ptr, ctypes.c_int64), _p(self.col, ctypes.c_int64))

    def numeric(self, a_v, p_v, out=None):
        a_v, p_v = _f64(a_v), _f64(p_v)
        if out is None:
            out = np.empty(self.nnz, np.float64)
        st = OracleStats()
        lib().ptap_oracle_numeric(
            self._h, _p(self._a_ip, ctypes.c_int64), _p(self._a_j, ctypes.c_int64), _p(a_v, ctypes.c_double),
            _p(self._p_ip, ctypes.c_int64), _p(self._p_j, ctypes.c_int64), _p(p_v, ctypes.c_double),
            _p(out, ctypes.c_double), ctypes.byref(st))
        self.num_stats = st
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().ptap_oracle_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stats_dict(s: OracleStats) -> dict:
    return {name: int(getattr(s, name)) for name, _ in OracleStats._fields_}


def oracle_ptap(n, m, a_ip, a_j, a_v, p_ip, p_j, p_v, nranks=1, algorithm="allatonce") -> OracleResult:
    """C = P^T A P assembled globally, exactly as the reference computes it."""
    plan = OraclePlan(n, m, a_ip, a_j, p_ip, p_j, nranks, algorithm)
    vals = plan.numeric(a_v, p_v)
    st = _stats_dict(plan.sym_stats)
    st.update({k: v for k, v in _stats_dict(plan.num_stats).items() if k in ("rows_num", "mac_ap", "mac_outer")})
    res = OracleResult(plan.row_ptr, plan.col, vals, st)
    plan.close()
    return res


def max_threads() -> int:
    return int(lib().ptap_oracle_max_threads())
