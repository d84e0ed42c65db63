import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_cases():
    return sorted(f[:-4] for f in os.listdir(GOLDEN_DIR) if f.endswith(".npz"))


def load_golden(name):
    """(meta, A arrays, P arrays, results) for one fixture; inputs built by
    this repo's generators are rebuilt and checked against the stored digest."""
    import hashlib

    from paper_1905_08423_b200 import problems as gen

    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    n, m = int(z["n"]), int(z["m"])
    if "a_ip" in z.files:
        a = (z["a_ip"], z["a_j"], z["a_v"])
        p = (z["p_ip"], z["p_j"], z["p_v"])
    else:
        A, P = gen.config_operands(gen.CONFIGS[str(z["gen"])], n_fine=int(z["n_fine"]))
        h = hashlib.sha256()
        for arr in (A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices, P.values):
            h.update(np.ascontiguousarray(arr).tobytes())
        assert h.hexdigest() == str(z["input_digest"]), f"generator drifted for {name}"
        a = (A.row_offsets, A.col_indices, A.values)
        p = (P.row_offsets, P.col_indices, P.values)
    results = {}
    for nr in z["ranks"]:
        for alg in ("two-step", "allatonce", "merged"):
            tag = f"np{int(nr)}_{alg}"
            results[(int(nr), alg)] = (z[tag + "_ip"], z[tag + "_j"], z[tag + "_v"])
    return n, m, a, p, results


def rel_err(got, want):
    scale = max(np.abs(want).max(initial=0.0), 1e-300)
    return float(np.abs(got - want).max(initial=0.0) / scale)


def row_scaled_err(ip, got, want):
    """max_ij |got-want| / max_k |want_ik| (SURVEY.md §8(c) gate)."""
    if want.size == 0:
        return 0.0
    rows = np.repeat(np.arange(ip.size - 1), np.diff(ip))
    rmax = np.zeros(ip.size - 1)
    np.maximum.at(rmax, rows, np.abs(want))
    den = np.maximum(rmax[rows], 1e-300)
    return float((np.abs(got - want) / den).max(initial=0.0))


def csr_from_arrays(nrows, ncols, ip, j, v):
    from paper_1905_08423_b200 import CsrMatrix
    return CsrMatrix(nrows, ncols, ip, j, v, check=False)


def run_ptap(a_glob, p_glob, nranks, algorithm, cache="keep"):
    """Distribute, one symbolic + one numeric pass on the CUDA path, assemble C
    (the reference's tests/conftest.py:48-58 helper, on this package)."""
    import paper_1905_08423_b200 as pk

    def prog(ctx):
        a, p = pk.distribute(a_glob, p_glob, ctx.nranks, ctx.rank)
        c, plan = pk.ptap(a, p, algorithm, ctx, cache=cache)
        return c.local, plan.counters, ctx.ledger.snapshot()

    results = pk.spawn_ranks(nranks, prog)
    c = pk.assemble_global([r[0] for r in results], ncols=p_glob.ncols)
    return c, results


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
