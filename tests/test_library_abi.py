"""The C-ABI library loads and exports every entry point include/ptap_b200.h
declares (no compute: this runs without a GPU)."""

import os
import re

import pytest

from paper_1905_08423_b200 import _lib
from paper_1905_08423_b200.errors import DeviceError

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ptap_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ptap_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_bound_symbols():
    assert declared_symbols() == _lib.exported_symbols()


def test_library_exports_every_declared_symbol():
    L = _lib.load(require_device=False)
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.ptap_version().startswith(b"ptap_b200")


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(DeviceError):
        _lib.load()


def test_status_codes_map_to_reference_exceptions():
    from paper_1905_08423_b200.errors import OwnershipError, PartitionMismatchError, StructuralDriftError
    assert _lib._STATUS_EXC[2] is PartitionMismatchError
    assert _lib._STATUS_EXC[3] is StructuralDriftError
    assert _lib._STATUS_EXC[4] is OwnershipError
    assert _lib._STATUS_EXC[5] is DeviceError


def test_null_and_bad_arguments_are_status_codes():
    """Host-side validation of every phase entry point: null plan/operands or
    an unknown algorithm come back as PTAP_ERR_VALUE (1) with a message, never
    as a crash (no device needed: nothing reaches a kernel)."""
    import ctypes
    L = _lib.load(require_device=False)
    null = ctypes.c_void_p(0)
    out = ctypes.c_void_p()
    assert L.ptap_plan_create(7, None, ctypes.byref(out)) == 1
    assert b"algorithm" in L.ptap_last_error()
    assert L.ptap_plan_create(1, None, ctypes.byref(out)) == 1
    for fn in ("ptap_symbolic_send", "ptap_numeric_send", "ptap_numeric_local"):
        assert getattr(L, fn)(null, None, null) == 1, fn
    assert L.ptap_symbolic_local(null, None, None, null) == 1
    assert L.ptap_numeric_local_rows(null, None, 0, 0, 0, null) == 1
    assert L.ptap_plan_c_last_row(null, None, null, null) == 1
    assert L.ptap_plan_check(null, null) == 1
    assert b"null plan" in L.ptap_last_error()
