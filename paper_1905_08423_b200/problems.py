"""Seeded synthetic inputs for the BASELINE.json configurations.

None of the five BASELINE generators exist in the reference (SURVEY.md
§8(d)); the reference only ships a 27-point graph Laplacian on a (2n-1)^3
grid (src/problems.py:56-116), which is mirrored here as
``model_problem_global`` for its own tests.  Every generator is a pure
function of global indices (and a seed), so any row block is identical no
matter how the rows are split across ranks, and the host (numpy) and device
(CUDA, csrc/ptap_gen.cu) versions produce bit-identical CSR.

Choices the configs leave open (documented in DESIGN.md):
  * grids are ordered lexicographically, x fastest; contiguous row blocks are
    z-slabs;
  * trilinear P maps coarse point c to fine point 2c; odd fine points
    interpolate c and c+1 with weight 1/2 per dimension, and the out-of-range
    c+1 at the last odd fine point is dropped;
  * config 3's off-diagonal weights are -(0.5 + u) with u in [0, 1) drawn by
    a counter-based hash of the undirected edge {i, j} (symmetric by
    construction), and the diagonal is the left-to-right sum of |offdiag| in
    ascending column order, plus 1e-2.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse import CsrMatrix

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def edge_uniform(i: np.ndarray, j: np.ndarray, nglobal: int, seed: int) -> np.ndarray:
    """u in [0,1) for the undirected edge {i,j}: 53 random bits * 2^-53."""
    lo = np.minimum(i, j).astype(np.uint64)
    hi = np.maximum(i, j).astype(np.uint64)
    with np.errstate(over="ignore"):
        key = lo * np.uint64(nglobal) + hi + np.uint64(seed) * _M2
    bits = splitmix64(key) >> np.uint64(11)
    return bits.astype(np.float64) * (2.0 ** -53)


def _stencil_offsets(points: int):
    if points == 7:
        # (dx, dy, dz) in ascending column order: -n^2, -n, -1, 0, +1, +n, +n^2
        return [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    if points == 27:
        return [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    raise ValueError("points must be 7 or 27")


def stencil_pattern(n: int, points: int, row_lo: int = 0, row_hi: int | None = None):
    """(row_ptr, col, offset_id) of a 7/27-point stencil on an n^3 grid for
    rows [row_lo, row_hi); columns ascending within each row."""
    N = n ** 3
    row_hi = N if row_hi is None else row_hi
    rows = np.arange(row_lo, row_hi, dtype=np.int64)
    x = rows % n
    y = (rows // n) % n
    z = rows // (n * n)
    offs = _stencil_offsets(points)
    masks = []
    for dx, dy, dz in offs:
        ok = (x + dx >= 0) & (x + dx < n) & (y + dy >= 0) & (y + dy < n) & (z + dz >= 0) & (z + dz < n)
        masks.append(ok)
    M = np.stack(masks, axis=1)  # rows x offsets, offsets in ascending column order
    counts = M.sum(axis=1)
    ip = np.zeros(rows.size + 1, np.int64)
    np.cumsum(counts, out=ip[1:])
    r_idx, o_idx = np.nonzero(M)  # row-major, so per row in ascending offset = ascending column
    delta = np.array([dx + n * dy + n * n * dz for dx, dy, dz in offs], np.int64)
    col = rows[r_idx] + delta[o_idx]
    return ip, col, o_idx, rows[r_idx]


def poisson7(n: int, row_lo: int = 0, row_hi: int | None = None) -> CsrMatrix:
    """7-point Poisson on n^3 interior unknowns: 6 on the diagonal, -1 off."""
    ip, col, oid, _ = stencil_pattern(n, 7, row_lo, row_hi)
    vals = np.where(oid == 3, 6.0, -1.0)
    nr = ip.size - 1
    return CsrMatrix(nr, n ** 3, ip, col, vals, check=False)


def random27(n: int, seed: int, row_lo: int = 0, row_hi: int | None = None) -> CsrMatrix:
    """Config 3's operator: 27-point on n^3, offdiag -(0.5+u) symmetric,
    diag = sum|offdiag| (ascending column order) + 1e-2."""
    N = n ** 3
    ip, col, oid, rowid = stencil_pattern(n, 27, row_lo, row_hi)
    off = -(0.5 + edge_uniform(rowid, col, N, seed))
    is_diag = oid == 13
    vals = np.where(is_diag, 0.0, off)
    nr = ip.size - 1
    # left fold of |offdiag| in ascending column order, one row at a time in lockstep
    acc = np.zeros(nr, np.float64)
    counts = np.diff(ip)
    maxc = int(counts.max(initial=0))
    for t in range(maxc):
        live = counts > t
        pos = ip[:-1][live] + t
        v = vals[pos]
        acc[live] = acc[live] + np.abs(v)  # diagonal slot contributes |0.0| = 0, a no-op add
    acc = acc + 1e-2
    diag_pos = np.nonzero(is_diag)[0]
    vals[diag_pos] = acc
    return CsrMatrix(nr, N, ip, col, vals, check=False)


def trilinear_1d(nc: int):
    """1D interpolation from nc coarse to 2*nc fine points: list of
    (fine, coarse, weight) with weights 1 and 1/2."""
    f, c, w = [], [], []
    for fi in range(2 * nc):
        b = fi // 2
        if fi % 2 == 0:
            f.append(fi); c.append(b); w.append(1.0)
        else:
            f.append(fi); c.append(b); w.append(0.5)
            if b + 1 < nc:
                f.append(fi); c.append(b + 1); w.append(0.5)
    return np.array(f, np.int64), np.array(c, np.int64), np.array(w)


def trilinear(nc: int, row_lo: int = 0, row_hi: int | None = None) -> CsrMatrix:
    """Trilinear P from nc^3 coarse to (2nc)^3 fine points (weights 1, 1/2,
    1/4, 1/8); columns ascending within each row."""
    nf = 2 * nc
    f1, c1, w1 = trilinear_1d(nc)
    ip1 = np.zeros(nf + 1, np.int64)
    np.add.at(ip1, f1 + 1, 1)
    np.cumsum(ip1, out=ip1)
    N = nf ** 3
    row_hi = N if row_hi is None else row_hi
    rows = np.arange(row_lo, row_hi, dtype=np.int64)
    x = rows % nf
    y = (rows // nf) % nf
    z = rows // (nf * nf)
    cx = ip1[x + 1] - ip1[x]
    cy = ip1[y + 1] - ip1[y]
    cz = ip1[z + 1] - ip1[z]
    counts = cx * cy * cz
    ip = np.zeros(rows.size + 1, np.int64)
    np.cumsum(counts, out=ip[1:])
    nnz = int(ip[-1])
    col = np.empty(nnz, np.int64)
    val = np.empty(nnz, np.float64)
    # ascending coarse column = (cz, cy, cx) lexicographic with cz major
    r = np.repeat(np.arange(rows.size), counts)
    k = np.arange(nnz) - ip[:-1][r]
    kx = k % cx[r]
    ky = (k // cx[r]) % cy[r]
    kz = k // (cx[r] * cy[r])
    ex = ip1[x[r]] + kx
    ey = ip1[y[r]] + ky
    ez = ip1[z[r]] + kz
    col[:] = c1[ex] + nc * (c1[ey] + nc * c1[ez])
    val[:] = w1[ex] * w1[ey] * w1[ez]
    return CsrMatrix(rows.size, nc ** 3, ip, col, val, check=False)


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n_fine: int      # fine points per dimension
    points: int      # 7 or 27
    seed: int = 0
    levels: int = 1


CONFIGS = {
    "cfg1": ConfigSpec("cfg1: 7-pt Poisson 32^3 -> 16^3", 32, 7),
    "cfg2": ConfigSpec("cfg2: 7-pt Poisson 128^3 -> 64^3", 128, 7),
    "cfg3": ConfigSpec("cfg3: 27-pt random 256^3 -> 128^3 -> 64^3", 256, 27, seed=20190520, levels=2),
}


def config_operands(spec: ConfigSpec, n_fine: int | None = None, row_lo=0, row_hi=None):
    """(A, P) for level 1 of a configuration, optionally at a reduced grid."""
    n = spec.n_fine if n_fine is None else n_fine
    if spec.points == 7:
        a = poisson7(n, row_lo, row_hi)
    else:
        a = random27(n, spec.seed, row_lo, row_hi)
    p = trilinear(n // 2, row_lo, row_hi)
    return a, p


# -- the reference's own model problem (src/problems.py:56-116) ------------


def model_problem_global(cx: int, cy: int, cz: int):
    """27-point graph Laplacian on the (2c-1)^3 fine grid with trilinear P to
    the c^3 coarse grid, as the reference's ``model_problem`` builds it."""
    fx, fy, fz = 2 * cx - 1, 2 * cy - 1, 2 * cz - 1
    N = fx * fy * fz
    ids = np.arange(N, dtype=np.int64)
    ix, iy, iz = ids % fx, (ids // fx) % fy, ids // (fx * fy)
    rows, cols, vals = [], [], []
    deg = np.zeros(N)
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                jx, jy, jz = ix + dx, iy + dy, iz + dz
                ok = (jx >= 0) & (jx < fx) & (jy >= 0) & (jy < fy) & (jz >= 0) & (jz < fz)
                if dx == dy == dz == 0:
                    continue
                deg += ok
                rows.append(ids[ok]); cols.append(jx[ok] + fx * (jy[ok] + fy * jz[ok]))
                vals.append(np.full(int(ok.sum()), -1.0))
    rows.append(ids); cols.append(ids); vals.append(deg)
    a = CsrMatrix.from_triplets(N, N, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    bx, by, bz = ix // 2, iy // 2, iz // 2
    rx, ry, rz = ix % 2, iy % 2, iz % 2
    w = np.ldexp(1.0, -(rx + ry + rz))
    pr, pc, pv = [], [], []
    for ox in (0, 1):
        for oy in (0, 1):
            for oz in (0, 1):
                ok = (rx >= ox) & (ry >= oy) & (rz >= oz)
                pr.append(ids[ok]); pc.append(bx[ok] + ox + cx * (by[ok] + oy + cy * (bz[ok] + oz)))
                pv.append(w[ok])
    p = CsrMatrix.from_triplets(N, cx * cy * cz, np.concatenate(pr), np.concatenate(pc), np.concatenate(pv))
    return a, p


def random_instance(n: int, m: int, density: float, seed: int):
    """Bernoulli-structured random (A, P) with a forced nonzero diagonal on A
    (same recipe as the reference's src/problems.py:129-144)."""
    rng = np.random.default_rng(seed)
    mask_a = rng.random((n, n)) < density
    np.fill_diagonal(mask_a, True)
    vals_a = rng.uniform(-1.0, 1.0, (n, n))
    mask_p = rng.random((n, m)) < density
    vals_p = rng.uniform(-1.0, 1.0, (n, m))
    ar, ac = np.nonzero(mask_a)
    pr, pc = np.nonzero(mask_p)
    return (CsrMatrix.from_triplets(n, n, ar, ac, vals_a[ar, ac]),
            CsrMatrix.from_triplets(n, m, pr, pc, vals_p[pr, pc]))
