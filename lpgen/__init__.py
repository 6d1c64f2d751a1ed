"""Seeded synthetic LP instance generators.

Shared by the oracle tests, the GPU parity tests and bench.py.  This module
holds only instance construction (random draws, stacking K = [G; A], and the
closed-form optimum of instances that are optimal by construction); it holds
none of the PDHG method's arithmetic and imports neither ``oracle`` nor the
product package.

The LP container follows PAPER.md Eq. (1)/(2): K = [G; A] with the
m1 ">=" rows first, q = (h; b), box bounds l <= x <= u with +-inf allowed.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

INF = np.inf


@dataclass
class LP:
    n: int
    m1: int
    m2: int
    row_ptr: np.ndarray      # int64, m+1
    col_idx: np.ndarray      # int32, nnz (sorted within each row)
    val: np.ndarray          # float64, nnz
    c: np.ndarray
    q: np.ndarray
    l: np.ndarray
    u: np.ndarray
    dense: bool = False      # True when K is stored with every entry (row-major pattern)
    obj_star: Optional[float] = None
    x_star: Optional[np.ndarray] = None
    y_star: Optional[np.ndarray] = None
    lam_star: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return self.m1 + self.m2

    @property
    def nnz(self) -> int:
        return int(self.val.size)

    def dense_K(self) -> np.ndarray:
        K = np.zeros((self.m, self.n))
        rows = np.repeat(np.arange(self.m), np.diff(self.row_ptr))
        K[rows, self.col_idx] = self.val
        return K

    def with_costs(self, c=None, q=None) -> "LP":
        return LP(self.n, self.m1, self.m2, self.row_ptr, self.col_idx, self.val,
                  self.c if c is None else np.asarray(c, np.float64),
                  self.q if q is None else np.asarray(q, np.float64),
                  self.l, self.u, self.dense)


def csr_from_dense(K: np.ndarray, keep_zeros: bool = False):
    K = np.asarray(K, dtype=np.float64)
    m, n = K.shape
    mask = np.ones_like(K, dtype=bool) if keep_zeros else (K != 0)
    row_ptr = np.zeros(m + 1, np.int64)
    row_ptr[1:] = np.cumsum(mask.sum(axis=1))
    rows, cols = np.nonzero(mask)
    return row_ptr, cols.astype(np.int32), K[rows, cols].astype(np.float64)


def stack(c, G=None, h=None, A=None, b=None, l=None, u=None, dense=False) -> LP:
    """K = [G; A], q = (h; b).  G, A dense arrays (or None)."""
    c = np.asarray(c, np.float64)
    n = c.size
    G = np.zeros((0, n)) if G is None else np.atleast_2d(np.asarray(G, np.float64))
    A = np.zeros((0, n)) if A is None else np.atleast_2d(np.asarray(A, np.float64))
    h = np.zeros(0) if h is None else np.atleast_1d(np.asarray(h, np.float64))
    b = np.zeros(0) if b is None else np.atleast_1d(np.asarray(b, np.float64))
    if G.shape[1] != n or A.shape[1] != n or h.size != G.shape[0] or b.size != A.shape[0]:
        raise ValueError("dimension mismatch")
    K = np.vstack([G, A])
    rp, ci, v = csr_from_dense(K, keep_zeros=dense)
    l = np.full(n, -INF) if l is None else np.asarray(l, np.float64)
    u = np.full(n, INF) if u is None else np.asarray(u, np.float64)
    return LP(n, G.shape[0], A.shape[0], rp, ci, v, c, np.concatenate([h, b]), l, u, dense)


def tiny_spec() -> LP:
    """min 2x1 + x2 s.t. x1 + x2 >= 1, 0 <= x <= 1 (optimum 1 at (0, 1))."""
    lp = stack([2.0, 1.0], G=[[1.0, 1.0]], h=[1.0], l=[0.0, 0.0], u=[1.0, 1.0])
    lp.obj_star = 1.0
    return lp


# ----------------------------------------------------------------- G-RAND --

def _row_pattern(rng, m, n, r):
    """m rows with r distinct, sorted, uniformly drawn columns each."""
    if r > n:
        raise ValueError("r > n")
    cols = rng.integers(0, n, size=(m, r), dtype=np.int64 if n >= 2**31 else np.int32)
    cols.sort(axis=1)
    while True:
        dup = np.nonzero((cols[:, 1:] == cols[:, :-1]).any(axis=1))[0] if r > 1 else np.zeros(0, int)
        if dup.size == 0:
            return cols
        new = rng.integers(0, n, size=(dup.size, r), dtype=cols.dtype)
        new.sort(axis=1)
        cols[dup] = new


def _csr_with_cover(rng, m, n, r):
    """Pattern step 1 of G-RAND: r distinct columns per row; any empty column
    receives one entry in a uniformly random row."""
    cols = _row_pattern(rng, m, n, r)
    counts = np.bincount(cols.ravel(), minlength=n)
    empty = np.nonzero(counts == 0)[0]
    extra_rows = rng.integers(0, m, size=empty.size)
    lens = np.full(m, r, np.int64)
    np.add.at(lens, extra_rows, 1)
    row_ptr = np.zeros(m + 1, np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    col_idx = np.empty(int(row_ptr[-1]), np.int32)
    plain = lens == r
    starts = row_ptr[:-1][plain]
    col_idx[(starts[:, None] + np.arange(r)[None, :]).ravel()] = cols[plain].ravel()
    for i in np.unique(extra_rows):
        merged = np.sort(np.concatenate([cols[i], empty[extra_rows == i]]))
        col_idx[row_ptr[i]:row_ptr[i + 1]] = merged
    return row_ptr, col_idx


def _csr_matvec(row_ptr, col_idx, val, x):
    prod = val * x[col_idx]
    out = np.zeros(row_ptr.size - 1)
    nonempty = np.diff(row_ptr) > 0
    out[nonempty] = np.add.reduceat(prod, row_ptr[:-1][nonempty])
    return out


def _csr_rmatvec(row_ptr, col_idx, val, y, n):
    rows = np.repeat(np.arange(row_ptr.size - 1), np.diff(row_ptr))
    return np.bincount(col_idx, weights=val * y[rows], minlength=n)


def _bounds_and_primal(rng, n):
    """Bounds (70% [0,inf), 20% [0,10], 10% free) and x*, lambda* (G-RAND steps 3-4)."""
    t = rng.uniform(size=n)
    l = np.where(t < 0.9, 0.0, -INF)
    u = np.where(t < 0.7, INF, np.where(t < 0.9, 10.0, INF))
    rj = rng.uniform(size=n)
    lam_mag = rng.uniform(0.1, 1.0, size=n)
    in_box = rng.uniform(0.1, 9.9, size=n)
    in_half = 0.1 + rng.exponential(1.0, size=n)
    in_free = rng.normal(size=n)
    at_l = (rj < 0.3) & np.isfinite(l)
    at_u = (~at_l) & (rj < 0.5) & np.isfinite(u)
    boxed = np.isfinite(l) & np.isfinite(u)
    half = np.isfinite(l) & ~np.isfinite(u)
    interior = np.where(boxed, in_box, np.where(half, in_half, in_free))
    x = np.where(at_l, l, np.where(at_u, u, interior))
    lam = np.where(at_l, lam_mag, np.where(at_u, -lam_mag, 0.0))
    return l, u, x, lam


def _duals_and_rhs(rng, Kx, m1, m2):
    """G-RAND step 5: >= rows active w.p. 1/2 (y* ~ U(0.1,1), h = Kx*), else
    y* = 0 and h = Kx* - U(0.1,1); = rows y* ~ N(0,1), b = Kx*."""
    active = rng.uniform(size=m1) < 0.5
    yact = rng.uniform(0.1, 1.0, size=m1)
    slack = rng.uniform(0.1, 1.0, size=m1)
    yeq = rng.normal(size=m2)
    y = np.concatenate([np.where(active, yact, 0.0), yeq])
    q = Kx.copy()
    q[:m1] = Kx[:m1] - np.where(active, 0.0, slack)
    return y, q


def _dual_value(q, y, l, u, lam):
    lp, lm = np.maximum(lam, 0.0), np.maximum(-lam, 0.0)
    fl, fu = np.isfinite(l), np.isfinite(u)
    return float(q @ y + np.sum(l[fl] * lp[fl]) - np.sum(u[fu] * lm[fu]))


def g_rand(m: int, n: int, r: int, seed: int, m1: Optional[int] = None) -> LP:
    """G-RAND(m, n, r, seed): random sparse LP, feasible by construction with a
    known optimum.  C1 = (50, 100, 10, 1), C4 = (1e5, 2e5, 20, 4),
    C5 = (5e6, 1e7, 20, 5)."""
    rng = np.random.default_rng(seed)
    m1 = m // 2 if m1 is None else m1
    m2 = m - m1
    row_ptr, col_idx = _csr_with_cover(rng, m, n, r)
    val = rng.normal(size=col_idx.size)
    l, u, xs, lam = _bounds_and_primal(rng, n)
    Kx = _csr_matvec(row_ptr, col_idx, val, xs)
    ys, q = _duals_and_rhs(rng, Kx, m1, m2)
    c = _csr_rmatvec(row_ptr, col_idx, val, ys, n) + lam
    lp = LP(n, m1, m2, row_ptr, col_idx, val, c, q, l, u)
    lp.obj_star = float(c @ xs)
    lp.x_star, lp.y_star, lp.lam_star = xs, ys, lam
    dv = _dual_value(q, ys, l, u, lam)
    assert abs(dv - lp.obj_star) <= 1e-9 * (1 + abs(lp.obj_star)), (dv, lp.obj_star)
    lp.meta = dict(generator="G-RAND", m=m, n=n, r=r, seed=seed)
    return lp


def g_powerlaw(m: int, n: int, r_mean: float, seed: int, alpha: float = 1.6, r_max: Optional[int] = None,
               m1: Optional[int] = None) -> LP:
    """G-POWERLAW: G-RAND's construction (known optimum) with skewed row lengths -- lengths drawn
    from a Pareto tail with exponent `alpha`, scaled to mean ~r_mean and clipped at r_max (default
    n // 2): a few rows hold thousands of entries, most a handful (SURVEY north star (1):
    "warp-per-row / merge-path" load balancing; the scale-free degree mixes of real LPs).
    Columns per row are distinct and uniform; every column gets at least one entry."""
    rng = np.random.default_rng(seed)
    m1 = m // 2 if m1 is None else m1
    m2 = m - m1
    r_max = n // 2 if r_max is None else r_max
    raw = rng.pareto(alpha, size=m) + 1.0
    lens = np.clip(np.round(raw * (r_mean / raw.mean())), 1, r_max).astype(np.int64)
    rows = []
    for i in range(m):
        rows.append(np.sort(rng.choice(n, size=int(lens[i]), replace=False)))
    cover = np.zeros(n, bool)
    for c in rows:
        cover[c] = True
    for j in np.nonzero(~cover)[0]:
        i = int(rng.integers(0, m))
        rows[i] = np.sort(np.append(rows[i], j))
    lens = np.array([c.size for c in rows], np.int64)
    row_ptr = np.zeros(m + 1, np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    col_idx = np.concatenate(rows).astype(np.int32)
    val = rng.normal(size=col_idx.size)
    l, u, xs, lam = _bounds_and_primal(rng, n)
    Kx = _csr_matvec(row_ptr, col_idx, val, xs)
    ys, q = _duals_and_rhs(rng, Kx, m1, m2)
    c = _csr_rmatvec(row_ptr, col_idx, val, ys, n) + lam
    lp = LP(n, m1, m2, row_ptr, col_idx, val, c, q, l, u)
    lp.obj_star = float(c @ xs)
    lp.x_star, lp.y_star, lp.lam_star = xs, ys, lam
    lp.meta = dict(generator="G-POWERLAW", m=m, n=n, r_mean=r_mean, alpha=alpha, seed=seed,
                   max_row=int(lens.max()))
    return lp


# ----------------------------------------------------------------- G-GRID --

def grid_arcs(k: int = 5):
    """Arcs of a k x k grid DAG with moves right and down, in the order: for
    each node row i, its horizontal arcs, then (i < k-1) its vertical arcs."""
    arcs = []
    for i in range(k):
        for j in range(k - 1):
            arcs.append((i * k + j, i * k + j + 1))
        if i < k - 1:
            for j in range(k):
                arcs.append((i * k + j, (i + 1) * k + j))
    return arcs


def grid_lp(k: int = 5) -> LP:
    """Flow LP of PAPER.md Eq. (warcraft shortest path LP) on the
    right/down grid: K_v = +1 on arcs leaving v, -1 on arcs entering v,
    q = e_source - e_sink, 0 <= x <= 1, all rows equalities (m1 = 0)."""
    arcs = grid_arcs(k)
    V, E = k * k, len(arcs)
    K = np.zeros((V, E))
    for e, (s, t) in enumerate(arcs):
        K[s, e] += 1.0
        K[t, e] -= 1.0
    q = np.zeros(V)
    q[0], q[V - 1] = 1.0, -1.0
    rp, ci, v = csr_from_dense(K)
    return LP(E, 0, V, rp, ci, v, np.ones(E), q, np.zeros(E), np.ones(E))


def pyepo_costs(n_arcs: int, batch: int, seed: int, deg: int = 4, noise: float = 0.5,
                p: int = 5, seed_B: int = 135):
    """PyEPO-style shortest-path costs: B ~ Bern(1/2)^{E x p} (seed_B),
    c_b = [((B f_b)/sqrt(p) + 3)^deg + 1] / 3.5^deg * U(1-noise, 1+noise)^E."""
    B = (np.random.default_rng(seed_B).uniform(size=(n_arcs, p)) < 0.5).astype(np.float64)
    rng = np.random.default_rng(seed)
    F = rng.normal(size=(batch, p))
    eps = rng.uniform(1.0 - noise, 1.0 + noise, size=(batch, n_arcs))
    return (((F @ B.T) / np.sqrt(p) + 3.0) ** deg + 1.0) / 3.5 ** deg * eps


def grid_dp_optimum(k: int, c: np.ndarray) -> float:
    """Shortest source->sink path cost on the right/down grid DAG by dynamic
    programming (ground truth: the flow LP is totally unimodular)."""
    arcs = grid_arcs(k)
    dist = np.full(k * k, INF)
    dist[0] = 0.0
    incoming = [[] for _ in range(k * k)]
    for e, (s, t) in enumerate(arcs):
        incoming[t].append((s, e))
    for v in range(1, k * k):
        dist[v] = min(dist[s] + c[e] for s, e in incoming[v])
    return float(dist[-1])


def g_grid(batch: int = 1024, k: int = 5, seed: int = 2):
    """G-GRID (C2): one shared flow LP and a batch x E cost matrix."""
    lp = grid_lp(k)
    C = pyepo_costs(lp.n, batch, seed)
    lp = lp.with_costs(c=C[0])
    lp.meta = dict(generator="G-GRID", k=k, batch=batch, seed=seed)
    return lp, C


# ---------------------------------------------------------------- G-DENSE --

def g_dense(m: int = 200, n: int = 400, batch: int = 256, seed: int = 3, m1: Optional[int] = None):
    """G-DENSE (C3): shared dense N(0,1) K (stored with every entry) and shared
    bounds; per instance its own x*, lambda*, y* and active set give q_b, c_b and
    obj*_b in closed form.  Returns (lp, C, Q, obj_star)."""
    rng = np.random.default_rng(seed)
    m1 = m // 2 if m1 is None else m1
    m2 = m - m1
    K = rng.normal(size=(m, n))
    rp, ci, v = csr_from_dense(K, keep_zeros=True)
    t = rng.uniform(size=n)
    l = np.where(t < 0.9, 0.0, -INF)
    u = np.where(t < 0.7, INF, np.where(t < 0.9, 10.0, INF))
    C = np.empty((batch, n))
    Q = np.empty((batch, m))
    obj = np.empty(batch)
    for b in range(batch):
        rj = rng.uniform(size=n)
        lam_mag = rng.uniform(0.1, 1.0, size=n)
        in_box = rng.uniform(0.1, 9.9, size=n)
        in_half = 0.1 + rng.exponential(1.0, size=n)
        in_free = rng.normal(size=n)
        at_l = (rj < 0.3) & np.isfinite(l)
        at_u = (~at_l) & (rj < 0.5) & np.isfinite(u)
        boxed = np.isfinite(l) & np.isfinite(u)
        half = np.isfinite(l) & ~np.isfinite(u)
        x = np.where(at_l, l, np.where(at_u, u, np.where(boxed, in_box, np.where(half, in_half, in_free))))
        lam = np.where(at_l, lam_mag, np.where(at_u, -lam_mag, 0.0))
        y, q = _duals_and_rhs(rng, K @ x, m1, m2)
        C[b] = K.T @ y + lam
        Q[b] = q
        obj[b] = C[b] @ x
    lp = LP(n, m1, m2, rp, ci, v, C[0].copy(), Q[0].copy(), l, u, dense=True)
    lp.meta = dict(generator="G-DENSE", m=m, n=n, batch=batch, seed=seed)
    return lp, C, Q, obj


# -------------------------------------------------------- small test LPs --

def random_small_lp(seed: int, n: int = 4, m1: int = 2, m2: int = 1, box: float = 3.0) -> LP:
    """A small dense LP with finite boxes (always bounded), feasible through a
    random interior point; for brute-force vertex enumeration tests."""
    rng = np.random.default_rng(seed)
    G = rng.normal(size=(m1, n))
    A = rng.normal(size=(m2, n))
    l = -rng.uniform(0.0, box, size=n)
    u = rng.uniform(0.5, box, size=n)
    x0 = rng.uniform(l, u)
    h = G @ x0 - rng.uniform(0.0, 1.0, size=m1)
    b = A @ x0
    c = rng.normal(size=n)
    return stack(c, G=G, h=h, A=A, b=b, l=l, u=u)


# ----------------------------------------------------------- G-INFEAS --

def g_infeasible(kind: str, seed: int, m1: int = 12, m2: int = 4, n: int = 24, box: float = 5.0,
                 density: float = 0.4, dense: bool = False) -> LP:
    """Small dense LPs infeasible by construction (SURVEY §8(f) row 1 test inputs).

    kind="primal": a feasible random LP (random interior point x0) plus one more
    ">=" row -sum_i y_i G_i x >= -sum_i y_i h_i + delta with y >= 0 on 3 rows and
    delta > 0: adding it to sum_i y_i (G_i x >= h_i) gives 0 >= delta, so the
    rows have no solution at all (Farkas; the box plays no part).
    kind="dual": a feasible random LP where column j has G[:, j] >= 0, A[:, j] = 0,
    u_j = +inf and c_j < 0, so x0 + t e_j stays feasible for every t >= 0 while
    c'x decreases without bound (the LP is unbounded, its dual infeasible)."""
    rng = np.random.default_rng(seed)
    G = rng.normal(size=(m1, n)) * (rng.random((m1, n)) < density)
    A = rng.normal(size=(m2, n)) * (rng.random((m2, n)) < density)
    l = -rng.uniform(0.5, box, size=n)
    u = rng.uniform(0.5, box, size=n)
    x0 = rng.uniform(l, u)
    c = rng.normal(size=n)
    if kind == "dual":
        j = int(rng.integers(n))
        G[:, j] = np.abs(G[:, j])
        A[:, j] = 0.0
        u[j] = INF
        c[j] = -abs(c[j]) - 0.5
        x0[j] = l[j] + 1.0
    h = G @ x0 - rng.uniform(0.0, 1.0, size=m1)
    b = A @ x0
    if kind == "primal":
        rows = rng.choice(m1, size=3, replace=False)
        y = np.zeros(m1)
        y[rows] = rng.uniform(0.5, 2.0, size=3)
        G = np.vstack([G, -(y @ G)])
        h = np.append(h, -(y @ h) + rng.uniform(0.5, 2.0))
    elif kind != "dual":
        raise ValueError(kind)
    lp = stack(c, G=G, h=h, A=A, b=b, l=l, u=u, dense=dense)
    lp.meta = dict(generator="G-INFEAS", kind=kind, seed=seed)
    return lp


# ------------------------------------------------------ G-WARCRAFT / G-KNAP --
# Paper-shaped SPO+ workloads.

WARCRAFT_TERRAIN = np.array([0.8, 1.2, 5.3, 7.7, 9.2])   # Warcraft-map vertex costs (synthetic stand-in)


def warcraft_arcs(k: int):
    """Directed arcs of the 8-connected k x k grid (both directions): for each node in
    row-major order, its out-arcs to neighbours in (di, dj) order.  k = 12 gives 1012
    arcs, k = 30 gives 6844."""
    arcs = []
    for i in range(k):
        for j in range(k):
            for di in (-1, 0, 1):
                for dj in (-1, 0, 1):
                    if (di or dj) and 0 <= i + di < k and 0 <= j + dj < k:
                        arcs.append((i * k + j, (i + di) * k + j + dj))
    return arcs


def warcraft_lp(k: int) -> LP:
    """PAPER.md Eq. (warcraft shortest path LP) on the 8-connected grid:
    one equality row per node (+1 on arcs leaving it, -1 on arcs entering it),
    q = e_s - e_t with s the top-left and t the bottom-right node, 0 <= x <= 1."""
    arcs = warcraft_arcs(k)
    V, E = k * k, len(arcs)
    rows = [[] for _ in range(V)]
    for e, (s, t) in enumerate(arcs):
        rows[s].append((e, 1.0))
        rows[t].append((e, -1.0))
    row_ptr = np.zeros(V + 1, np.int64)
    col_idx, val = [], []
    for v in range(V):
        ent = sorted(rows[v])
        col_idx += [e for e, _ in ent]
        val += [w for _, w in ent]
        row_ptr[v + 1] = len(col_idx)
    q = np.zeros(V)
    q[0], q[V - 1] = 1.0, -1.0
    lp = LP(E, 0, V, row_ptr, np.asarray(col_idx, np.int32), np.asarray(val), np.ones(E), q,
            np.zeros(E), np.ones(E))
    lp.meta = dict(generator="G-WARCRAFT", k=k)
    return lp


def warcraft_costs(k: int, batch: int, seed: int, noise: float = 0.0):
    """Arc costs of `batch` synthetic maps: each vertex draws a terrain cost, an arc
    costs its head vertex's terrain (entering cost); optional multiplicative noise
    U(1 - noise, 1 + noise) stands in for a predictor's error."""
    rng = np.random.default_rng(seed)
    heads = np.array([t for _, t in warcraft_arcs(k)])
    node = WARCRAFT_TERRAIN[rng.integers(0, WARCRAFT_TERRAIN.size, size=(batch, k * k))]
    C = node[:, heads]
    if noise:
        C = C * rng.uniform(1.0 - noise, 1.0 + noise, size=C.shape)
    return C


def warcraft_optimum(k: int, c: np.ndarray) -> float:
    """Shortest s -> t path cost by Dijkstra (costs > 0; the flow LP is totally unimodular)."""
    import heapq
    adj = [[] for _ in range(k * k)]
    for e, (s, t) in enumerate(warcraft_arcs(k)):
        adj[s].append((t, float(c[e])))
    dist = np.full(k * k, INF)
    dist[0] = 0.0
    pq = [(0.0, 0)]
    while pq:
        d, v = heapq.heappop(pq)
        if d > dist[v]:
            continue
        for t, w in adj[v]:
            if d + w < dist[t]:
                dist[t] = d + w
                heapq.heappush(pq, (d + w, t))
    return float(dist[-1])


def knapsack_lp(N: int, d: int, seed: int, capacity: float = 500.0, dense: bool = True) -> LP:
    """LP relaxation of the multi-dimensional knapsack of PAPER.md Eq. (knapsack)
    as a minimisation: min -c'x s.t. -W x >= -h (d rows), 0 <= x <= 1, W_ij ~ U{3..8},
    h_j = 500; c set per instance by knapsack_values."""
    rng = np.random.default_rng(seed)
    W = rng.integers(3, 9, size=(d, N)).astype(np.float64)
    lp = stack(-np.ones(N), G=-W, h=np.full(d, -capacity), l=np.zeros(N), u=np.ones(N), dense=dense)
    lp.meta = dict(generator="G-KNAP", N=N, d=d, seed=seed)
    return lp


def knapsack_values(N: int, batch: int, seed: int, deg: int = 4, noise: float = 0.0, p: int = 5):
    """Item values by the PyEPO polynomial: c = [((B f)/sqrt(p) + 3)^deg + 1] / 3.5^deg
    times U(1 - noise, 1 + noise); returned as the minimisation costs -c (batch x N)."""
    return -pyepo_costs(N, batch, seed, deg=deg, noise=noise, p=p, seed_B=seed + 1)
