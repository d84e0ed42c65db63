"""Seeded generators for BASELINE.json configs 4 and 5 (host, numpy/scipy).

These are algebraic-multigrid style inputs whose P is *smoothed
aggregation*, so unlike configs 1-3 their P rows are wide (config 4: ~12
entries) or irregular (config 5: unstructured, natural point order).  They
are input generators, not part of the product path: scipy builds them the
way an AMG setup phase would, and the triple product is then run through the
package's CUDA path like any other CSR input.  None of them exists in the
reference; the open choices are listed here and in
DESIGN.md §2:

config 4 (``block_transport``), multi-group transport mimic
  * nodes on an nn^3 grid, x fastest; row = node * ncomp + component
    (component fastest);
  * inside a node: a symmetric dense ncomp x ncomp coupling, off-diagonal
    values U(-0.1, 0.1) drawn by a counter-based hash of the unordered
    (row, col) pair;
  * across nodes: 7-point coupling per component, -U(0.5, 1.5), symmetric by
    the same edge hash;
  * diagonal = sum |offdiag| (folded left to right in ascending column order)
    + 1e-2 (strict diagonal dominance);
  * P: 3x3x3 node aggregates (the last aggregate per dimension is short when
    3 does not divide nn), piecewise-constant tentative P per component, one
    damped-Jacobi step P = (I - w D^-1 A) P_tent with
    w = (4/3) / lambda_max(D^-1 A), lambda_max from 10 power iterations on a
    vector drawn from numpy's default_rng(seed).

config 5 (``knn_laplacian``), unstructured graph Laplacian
  * npts points uniform in the unit cube from default_rng(seed);
  * symmetric 26-nearest-neighbour graph (union of the directed kNN edges,
    scipy cKDTree), weights 1/distance;
  * A = weighted-degree diagonal + 1e-3, off-diagonals -w (int64 row_ptr);
  * P: greedy distance-2 aggregation in natural point order (a point whose
    neighbours are all unaggregated roots an aggregate of itself and those
    neighbours; every leftover point joins the aggregate of its first
    aggregated neighbour in ascending index order), piecewise-constant
    tentative P, then P = (I - w D^-1 A) P_tent with
    w = (2/3) / max_i sum_j |A_ij| / A_ii.

P's stored pattern is the structural pattern of P_tent + D^-1 A P_tent (no
entry is dropped when it happens to cancel).
"""

from __future__ import annotations

import numpy as np

from .problems import edge_uniform
from .sparse import CsrMatrix


def _to_csr(m) -> CsrMatrix:
    m = m.tocsr()
    m.sort_indices()
    return CsrMatrix(m.shape[0], m.shape[1], m.indptr.astype(np.int64), m.indices.astype(np.int64),
                     m.data.astype(np.float64), check=False)


def _structural_smooth(A, P_tent, omega: float):
    """P = P_tent - omega D^-1 A P_tent keeping the structural pattern."""
    import scipy.sparse as sp

    dinv = 1.0 / A.diagonal()
    DA = sp.diags(dinv) @ A
    AP = (DA @ P_tent).tocsr()
    # structural pattern of AP: product of the 0/1 patterns (nothing cancels)
    pat = (abs(DA).sign() @ P_tent.sign()).tocsr()
    pat.data[:] = 0.0
    AP = (AP + pat).tocsr()
    AP.sort_indices()
    P = (P_tent.tocsr() - omega * AP).tocsr()
    # re-add the union pattern (subtraction may drop exact zeros)
    union = (P_tent.sign() + pat).tocsr()
    union.data[:] = 0.0
    P = (P + union).tocsr()
    P.sort_indices()
    return P


def _row_abs_fold(m) -> np.ndarray:
    """sum_j |m_ij| folded left to right in ascending column order (the order
    the device generator uses; scipy's own row sum is pairwise on long rows)."""
    ip, v = m.indptr, np.abs(m.data)
    ln = np.diff(ip)
    acc = np.zeros(m.shape[0])
    for k in range(int(ln.max(initial=0))):
        rows = np.nonzero(ln > k)[0]
        acc[rows] = acc[rows] + v[ip[rows] + k]
    return acc


def _power_lambda_max(DA, seed: int, iters: int = 10) -> float:
    rng = np.random.default_rng(seed)
    v = rng.random(DA.shape[0])
    lam = 0.0
    for _ in range(iters):
        w = DA @ v
        lam = float(np.linalg.norm(w) / np.linalg.norm(v))
        v = w / np.linalg.norm(w)
    return lam


def block_transport(nn: int, ncomp: int = 10, seed: int = 20190520, agg: int = 3):
    """Config 4 at an nn^3 node grid: returns (A, P) as CsrMatrix."""
    import scipy.sparse as sp

    nnode = nn ** 3
    n = nnode * ncomp
    node = np.arange(nnode, dtype=np.int64)
    x, y, z = node % nn, (node // nn) % nn, node // (nn * nn)
    rows, cols = [], []
    # in-node dense coupling (off-diagonal)
    ci, cj = np.meshgrid(np.arange(ncomp), np.arange(ncomp), indexing="ij")
    off = ci != cj
    ci, cj = ci[off], cj[off]
    rows.append((node[:, None] * ncomp + ci[None, :]).ravel())
    cols.append((node[:, None] * ncomp + cj[None, :]).ravel())
    inblock = [np.ones(rows[-1].size, bool)]
    # 7-point coupling per component
    comp = np.arange(ncomp, dtype=np.int64)
    for dx, dy, dz in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        ok = (x + dx >= 0) & (x + dx < nn) & (y + dy >= 0) & (y + dy < nn) & (z + dz >= 0) & (z + dz < nn)
        src = node[ok]
        dst = (x[ok] + dx) + nn * ((y[ok] + dy) + nn * (z[ok] + dz))
        rows.append((src[:, None] * ncomp + comp[None, :]).ravel())
        cols.append((dst[:, None] * ncomp + comp[None, :]).ravel())
        inblock.append(np.zeros(rows[-1].size, bool))
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    ib = np.concatenate(inblock)
    u = edge_uniform(r, c, n, seed)
    v = np.where(ib, -0.1 + 0.2 * u, -(0.5 + u))
    off_m = sp.csr_matrix((v, (r, c)), shape=(n, n))
    off_m.sort_indices()
    diag = _row_abs_fold(off_m) + 1e-2
    A = (off_m + sp.diags(diag)).tocsr()
    A.sort_indices()
    # tentative P: 3x3x3 node aggregates, one column per (aggregate, component)
    na = -(-nn // agg)
    aggid = (x // agg) + na * ((y // agg) + na * (z // agg))
    pr = np.arange(n, dtype=np.int64)
    pc = aggid[pr // ncomp] * ncomp + pr % ncomp
    P_tent = sp.csr_matrix((np.ones(n), (pr, pc)), shape=(n, na ** 3 * ncomp))
    DA = sp.diags(1.0 / A.diagonal()) @ A
    omega = (4.0 / 3.0) / _power_lambda_max(DA, seed)
    P = _structural_smooth(A, P_tent, omega)
    return _to_csr(A), _to_csr(P)


def _greedy_aggregate_py(indptr: np.ndarray, indices: np.ndarray, n: int) -> np.ndarray:
    """Greedy distance-2 aggregation in natural order (see module docstring)."""
    agg = np.full(n, -1, np.int64)
    nagg = 0
    for i in range(n):
        if agg[i] >= 0:
            continue
        nb = indices[indptr[i]:indptr[i + 1]]
        nb = nb[nb != i]
        if np.all(agg[nb] < 0):
            agg[i] = nagg
            agg[nb] = nagg
            nagg += 1
    for i in range(n):
        if agg[i] >= 0:
            continue
        nb = indices[indptr[i]:indptr[i + 1]]
        nb = nb[(nb != i) & (agg[nb] >= 0)]
        agg[i] = agg[nb.min()] if nb.size else nagg
        if not nb.size:
            nagg += 1
    return agg


def _greedy_aggregate_loops(indptr, indices, n):
    """The same two passes as _greedy_aggregate_py, as scalar loops (numba)."""
    agg = np.full(n, -1, np.int64)
    nagg = 0
    for i in range(n):
        if agg[i] >= 0:
            continue
        free = True
        for q in range(indptr[i], indptr[i + 1]):
            j = indices[q]
            if j != i and agg[j] >= 0:
                free = False
                break
        if free:
            agg[i] = nagg
            for q in range(indptr[i], indptr[i + 1]):
                agg[indices[q]] = nagg
            nagg += 1
    # second pass: a leftover joins the aggregate of its smallest-index
    # aggregated neighbour (leftovers assigned earlier in this pass count)
    for i in range(n):
        if agg[i] >= 0:
            continue
        best = -1
        for q in range(indptr[i], indptr[i + 1]):
            j = indices[q]
            if j != i and agg[j] >= 0 and (best < 0 or j < best):
                best = j
        if best >= 0:
            agg[i] = agg[best]
        else:
            agg[i] = nagg
            nagg += 1
    return agg


def _greedy_aggregate(indptr: np.ndarray, indices: np.ndarray, n: int) -> np.ndarray:
    """Greedy distance-2 aggregation (numba-compiled loops when numba is
    importable, else the numpy version; both give the same aggregates)."""
    try:
        import numba
    except ImportError:
        return _greedy_aggregate_py(indptr, indices, n)
    global _greedy_jit
    if _greedy_jit is None:
        _greedy_jit = numba.njit(cache=False)(_greedy_aggregate_loops)
    return _greedy_jit(indptr.astype(np.int64), indices.astype(np.int64), n)


_greedy_jit = None


def knn_laplacian(npts: int, k: int = 26, seed: int = 20190520):
    """Config 5 at npts points: returns (A, P) as CsrMatrix."""
    import scipy.sparse as sp
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.random((npts, 3))
    dist, nbr = cKDTree(pts).query(pts, k=k + 1, workers=-1)
    # symmetric union of the directed edges, weight 1/distance (both
    # directions carry the same rounded distance, so max() is the union)
    indptr = np.arange(0, npts * k + 1, k, dtype=np.int64)
    Wd = sp.csr_matrix((1.0 / dist[:, 1:].ravel(), nbr[:, 1:].ravel().astype(np.int64), indptr),
                       shape=(npts, npts))
    del dist, nbr
    Wd.sort_indices()
    W = Wd.maximum(Wd.T.tocsr()).tocsr()
    del Wd
    W.sort_indices()
    deg = np.asarray(W.sum(axis=1)).ravel()
    A = (sp.diags(deg + 1e-3) - W).tocsr()
    A.sort_indices()
    agg = _greedy_aggregate(W.indptr, W.indices, npts)
    nagg = int(agg.max()) + 1
    P_tent = sp.csr_matrix((np.ones(npts), (np.arange(npts), agg)), shape=(npts, nagg))
    dinv = 1.0 / A.diagonal()
    rowsum = np.asarray(abs(A).sum(axis=1)).ravel() * dinv
    omega = (2.0 / 3.0) / float(rowsum.max())
    P = _structural_smooth(A, P_tent, omega)
    return _to_csr(A), _to_csr(P)
