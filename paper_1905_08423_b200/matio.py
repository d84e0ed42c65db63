"""Matrix interchange: Matrix Market text (the reference's src/mmio.py:18-73
contract) and a binary .npz layout for inputs too large for text.

Matrix Market: ``%%MatrixMarket matrix coordinate real general``, 1-based
indices on disk, values printed with 17 significant digits so a round trip
reproduces every float64 bit; duplicates are summed on read (``from_triplets``
semantics); malformed files raise ``MatrixMarketError`` with the 1-based line
of the problem.  The parser is vectorised (one numpy pass over the entry
lines) so the config-sized inputs load in seconds, not minutes.

``.npz``: arrays ``shape`` (nrows, ncols), ``row_offsets`` (int64),
``col_indices`` (int64) and, when present, ``values`` (float64) -- the
CsrMatrix layout, read back without any re-sorting.
"""

from __future__ import annotations

import numpy as np

from .errors import MatrixMarketError
from .sparse import CsrMatrix

_HEADER = "%%MatrixMarket matrix coordinate real general"


def write_matrix_market(path, m: CsrMatrix) -> None:
    rows, cols, vals = m.to_triplets()
    if vals is None:
        vals = np.ones(rows.shape[0])
    with open(path, "w") as f:
        f.write(_HEADER + "\n")
        f.write(f"{m.nrows} {m.ncols} {m.nnz}\n")
        if rows.size:
            lines = [f"{r + 1} {c + 1} {v:.17g}" for r, c, v in zip(rows.tolist(), cols.tolist(), vals.tolist())]
            f.write("\n".join(lines))
            f.write("\n")


def read_matrix_market(path) -> CsrMatrix:
    with open(path) as f:
        text = f.read()
    lines = text.splitlines()
    if not lines or not lines[0].startswith("%%MatrixMarket"):
        raise MatrixMarketError("missing MatrixMarket banner", line=1)
    fields = [s.lower() for s in lines[0].split()[1:5]]
    if fields != ["matrix", "coordinate", "real", "general"]:
        raise MatrixMarketError(f"unsupported header {lines[0].strip()!r}", line=1)
    # size line: first non-comment, non-blank line after the banner
    k = 1
    while k < len(lines) and (not lines[k].strip() or lines[k].lstrip().startswith("%")):
        k += 1
    if k >= len(lines):
        raise MatrixMarketError("missing size line", line=len(lines))
    parts = lines[k].split()
    if len(parts) != 3:
        raise MatrixMarketError("size line must be 'nrows ncols nnz'", line=k + 1)
    try:
        nrows, ncols, nnz = (int(x) for x in parts)
    except ValueError:
        raise MatrixMarketError(f"bad size line {lines[k].strip()!r}", line=k + 1) from None
    entry_lines = [(i + 1, s) for i, s in enumerate(lines[k + 1:], start=k + 1)
                   if s.strip() and not s.lstrip().startswith("%")]
    if len(entry_lines) != nnz:
        raise MatrixMarketError(f"header promises {nnz} entries but file has {len(entry_lines)}",
                                line=len(lines))
    if nnz == 0:
        return CsrMatrix(nrows, ncols, np.zeros(nrows + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    toks = [s.split() for _, s in entry_lines]
    bad = next((ln for (ln, _), t in zip(entry_lines, toks) if len(t) != 3), None)
    if bad is not None:
        raise MatrixMarketError("entry must be 'row col value'", line=bad)
    arr = np.array(toks)
    try:
        r = arr[:, 0].astype(np.int64) - 1
        c = arr[:, 1].astype(np.int64) - 1
        v = arr[:, 2].astype(np.float64)
    except ValueError:
        # find the first offending line for the message
        for (ln, s), t in zip(entry_lines, toks):
            try:
                int(t[0]), int(t[1]), float(t[2])
            except ValueError:
                raise MatrixMarketError(f"bad entry {s.strip()!r}", line=ln) from None
        raise
    if r.min() < 0 or c.min() < 0 or r.max() >= nrows or c.max() >= ncols:
        i = int(np.nonzero((r < 0) | (c < 0) | (r >= nrows) | (c >= ncols))[0][0])
        raise MatrixMarketError("entry index out of range", line=entry_lines[i][0])
    try:
        return CsrMatrix.from_triplets(nrows, ncols, r, c, v)
    except Exception as exc:
        raise MatrixMarketError(str(exc)) from exc


def save_npz(path, m: CsrMatrix) -> None:
    arrays = {"shape": np.array([m.nrows, m.ncols], np.int64), "row_offsets": m.row_offsets,
              "col_indices": m.col_indices}
    if m.values is not None:
        arrays["values"] = m.values
    np.savez(path, **arrays)


def load_npz(path) -> CsrMatrix:
    with np.load(path) as d:
        nrows, ncols = (int(x) for x in d["shape"])
        vals = d["values"] if "values" in d.files else None
        return CsrMatrix(nrows, ncols, d["row_offsets"].astype(np.int64), d["col_indices"].astype(np.int64),
                         None if vals is None else vals.astype(np.float64))
