"""Oracle of the aggregation-multigrid inner solve for S_D.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper applies B_2^-1 with an exact MUMPS solve of the approximate Schur
complement S = -B diag(A)^-1 B^T.  Precond kind 3
(Block-Schur-AMG) replaces that exact solve by one symmetric aggregation V-cycle
on S_D (reading R22), a fixed linear operator, so plain GMRES applies.

Definition (the GPU follows it step by step):
  * strength: off-diagonal (i, j) is strong iff |A_ij| >= theta sqrt(A_ii A_jj), theta = 0.08
    on the finest level, THETA_COARSE = 0.04 below it (the smoothed-aggregation
    operator of level 1 has many weak entries; 0.08 stalls its coarsening)
  * keys: key(i) = ((splitmix64(i) >> 33) << 30) | i  (distinct, index recoverable)
  * MIS-2 (Luby, deterministic): repeat { k1 = max key over N[i], k2 = max k1 over
    N[i] (N = strong neighbours incl. i; roots count as +inf, excluded as -1);
    an undecided i with k2 == key(i) becomes a root, one with k2 == +inf is
    excluded } until no node is undecided
  * aggregates: roots numbered in index order; pass 1: a non-root joins the
    root of largest key among its strong neighbours; pass 2: a still free node
    joins the aggregate of its largest-key assigned strong neighbour; pass 3:
    the rest become singletons in index order
  * prolongator: on the first SA_LEVELS = 1 level(s) the smoothed aggregation
    prolongator P = (I - omega D^-1 A) T with T piecewise constant on the
    aggregates and omega = 4 / (3 lmax) (Vanek, Mandel & Brezina 1996: one damped
    Jacobi step on the tentative prolongator); below, P = T.  A_c = P^T A P; stop
    when n <= COARSE_SIZE, at MAX_LEVELS, or when a level coarsens by less than 1/0.75;
    exact-zero rule: an entry of P or A_c exists iff some term of its sum exists, whatever
    the sum's value (with_structure), so the level sizes are integers both sides agree on
  * coarsest level (COARSE_SIZE = 2048): dense inverse applied as a matvec, else
    (stagnated coarsening) a degree-COARSE_DEGREE = 32 Chebyshev smoother (C3: the
    11,794-row coarsest; degree 8 / 16 / 32 / exact inverse give 118 / 101 / 95 / 95
    GMRES iterations, R22)
  * smoother C_l(b): degree-DEGREE (3; degree 2 was measured on the GPU and rejected: full C3
    111 iterations / 151.0 ms instead of 95 / 143.5 ms, full C5 91.0 s instead of 88.7 s)
    point-Jacobi Chebyshev from x0 = 0 (Saad
    Alg. 12.1, exactly oracle.solver.chebyshev) on [lmax/RATIO, lmax] with the
    Gershgorin bound lmax = max_i sum_j |A_ij| / A_ii
  * V(b) at level l: x = C(b); r = b - A x; x += P V(P^T r); x += C(b - A x)
    (restriction P^T r is the aggregate sum of r when P = T)
Parity unpinned by the paper (iteration counts).  Pinned in
tests/test_oracle_pins.py: MIS-2 property, aggregate validity, Galerkin identity,
a one-level hierarchy is an exact solve, symmetry of the V-cycle operator.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .solver import chebyshev

THETA = 0.08
THETA_COARSE = 0.04
SA_LEVELS = 1
COARSE_SIZE = 2048
MAX_LEVELS = 12
DEGREE = 3
RATIO = 30.0
COARSE_DEGREE = 32
STAGNATION = 0.75
P_DEGREE = 2       # smoother of the p-multigrid (SchurMG, n_p > 1): Chebyshev(P_DEGREE) on [2/P_RATIO, 2]
P_RATIO = 6.0
P_COARSE_DEGREE = 8   # Chebyshev degree of a non-dense coarsest level of the SchurMG hierarchy
KEY_INDEX_BITS = 30
ROOT_KEY = np.int64(np.iinfo(np.int64).max)


def keys(n: int) -> np.ndarray:
    """key(i) = ((splitmix64(i) >> 33) << 30) | i, i < 2^30."""
    assert n < (1 << KEY_INDEX_BITS)
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = i + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (((z >> np.uint64(33)) << np.uint64(KEY_INDEX_BITS)) | i).astype(np.int64)


def strong_graph(A, theta=THETA):
    """CSR pattern of the strong connections plus the diagonal."""
    C = A.tocoo()
    d = A.diagonal()
    keep = (C.row == C.col) | (np.abs(C.data) >= theta * np.sqrt(np.abs(d[C.row] * d[C.col])))
    G = sp.csr_matrix((np.ones(int(keep.sum()), dtype=np.int8), (C.row[keep], C.col[keep])), shape=A.shape)
    G.sort_indices()
    return G


def nbr_max(G, val):
    """out[i] = max_{j in N[i]} val[j]."""
    out = np.full(G.shape[0], np.iinfo(np.int64).min, dtype=np.int64)
    rows = np.repeat(np.arange(G.shape[0]), np.diff(G.indptr))
    np.maximum.at(out, rows, val[G.indices])
    return out


def aggregate(A, theta=THETA):
    """Returns (agg (n,), nc, roots mask)."""
    n = A.shape[0]
    G = strong_graph(A, theta)
    key = keys(n)
    U, R, X = 0, 1, 2
    state = np.zeros(n, dtype=np.int8)
    while np.any(state == U):
        k = np.where(state == U, key, np.where(state == R, ROOT_KEY, np.int64(-1)))
        k2 = nbr_max(G, nbr_max(G, k))
        und = state == U
        new_root = und & (k2 == key)
        excl = und & ~new_root & (k2 == ROOT_KEY)
        state[new_root] = R
        state[excl] = X
    mask = (1 << KEY_INDEX_BITS) - 1
    is_root = state == R
    agg = np.full(n, -1, dtype=np.int64)
    agg[is_root] = np.arange(int(is_root.sum()))
    # pass 1
    best = nbr_max(G, np.where(is_root, key, np.int64(-1)))
    m1 = (agg < 0) & (best >= 0)
    agg1 = agg.copy()
    agg1[m1] = agg[best[m1] & mask]
    # pass 2
    best2 = nbr_max(G, np.where(agg1 >= 0, key, np.int64(-1)))
    m2 = (agg1 < 0) & (best2 >= 0)
    agg2 = agg1.copy()
    agg2[m2] = agg1[best2[m2] & mask]
    # pass 3
    left = np.nonzero(agg2 < 0)[0]
    nroot = int(is_root.sum())
    agg2[left] = nroot + np.arange(left.size)
    return agg2, nroot + left.size, is_root


def with_structure(C, pattern):
    """C with an explicit entry (possibly 0.0) wherever `pattern` has one.  The exact-zero
    rule of the hierarchy (one rule on both sides, R22): an entry of a product
    exists iff some term contributes to it, whatever the terms sum to.  scipy's sparse
    product drops a sum that cancels to exactly 0.0, so the structural pattern is taken from
    the same product of the absolute values (no cancellation) and merged back in."""
    a, b = C.tocoo(), pattern.tocoo()
    M = sp.csr_matrix((np.concatenate([a.data, np.zeros(b.nnz)]),
                       (np.concatenate([a.row, b.row]), np.concatenate([a.col, b.col]))), shape=C.shape)
    M.sum_duplicates()
    M.sort_indices()
    return M


def triple_product(P, A):
    """A_c = P^T A P with the structural pattern of the product (with_structure)."""
    A = A.tocsr()
    return with_structure((P.T @ A @ P).tocsr(), (abs(P).T @ abs(A) @ abs(P)).tocsr())


def galerkin(A, agg, nc):
    n = A.shape[0]
    P = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nc))
    return triple_product(P, A)


def smoothed_prolongator(A, agg, nc, lmax):
    """P = (I - omega D^-1 A) T, omega = 4 / (3 lmax), T_{i, agg_i} = 1."""
    n = A.shape[0]
    T = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nc))
    omega = 4.0 / (3.0 * lmax)
    P = (T - omega * (sp.diags(1.0 / A.diagonal()) @ (A.tocsr() @ T))).tocsr()
    return with_structure(P, (T + abs(A.tocsr()) @ T).tocsr())


def gershgorin(A):
    a = abs(A).sum(axis=1).A1
    return float(np.max(a / A.diagonal()))


@dataclass
class Level:
    A: sp.csr_matrix
    Dinv: sp.dia_matrix
    lmax: float
    agg: np.ndarray | None = None
    nc: int = 0
    P: sp.csr_matrix | None = None     # smoothed prolongator (None: piecewise constant on agg)


class AMG:
    """Aggregation V-cycle hierarchy for an SPD matrix (point Jacobi smoothing)."""

    def __init__(self, A, theta=THETA, coarse_size=COARSE_SIZE, max_levels=MAX_LEVELS, coarse_degree=None):
        self.coarse_degree = coarse_degree   # None: the module's COARSE_DEGREE (kinds 3, 4)
        self.levels = []
        A = A.tocsr()
        while True:
            lev = Level(A, sp.diags(1.0 / A.diagonal()), gershgorin(A))
            self.levels.append(lev)
            if A.shape[0] <= coarse_size or len(self.levels) >= max_levels:
                break
            agg, nc, _ = aggregate(A, theta if len(self.levels) == 1 else THETA_COARSE)
            if nc > STAGNATION * A.shape[0]:
                break
            lev.agg, lev.nc = agg, nc
            if len(self.levels) <= SA_LEVELS:
                lev.P = smoothed_prolongator(A, agg, nc, lev.lmax)
                A = triple_product(lev.P, A)
            else:
                A = galerkin(A, agg, nc)
        last = self.levels[-1]
        self.coarse_inv = np.linalg.inv(last.A.toarray()) if last.A.shape[0] <= coarse_size else None

    def to_float32(self):
        """The same hierarchy with every matrix, inverse and prolongator rounded to FP32
        (precond kind 4: the V-cycle runs in FP32; the Chebyshev intervals keep the
        FP64 Gershgorin bounds).  vcycle() then takes and returns float32 vectors."""
        import copy
        h = copy.copy(self)
        h.levels = []
        for lev in self.levels:
            h.levels.append(Level(lev.A.astype(np.float32), lev.Dinv.astype(np.float32), lev.lmax, lev.agg, lev.nc,
                                  None if lev.P is None else lev.P.astype(np.float32)))
        h.coarse_inv = None if self.coarse_inv is None else self.coarse_inv.astype(np.float32)
        return h

    def smooth(self, lev, b, degree=DEGREE):
        return chebyshev(lev.A, lev.Dinv, b, degree, lev.lmax, RATIO)

    def vcycle(self, b, level=0):
        lev = self.levels[level]
        if level == len(self.levels) - 1:
            if self.coarse_inv is not None:
                return self.coarse_inv @ b
            return self.smooth(lev, b, COARSE_DEGREE if self.coarse_degree is None else self.coarse_degree)
        x = self.smooth(lev, b)
        r = b - lev.A @ x
        if lev.P is not None:
            x = x + lev.P @ self.vcycle(lev.P.T @ r, level + 1)
        else:
            bc = np.bincount(lev.agg, weights=r, minlength=lev.nc).astype(r.dtype)
            xc = self.vcycle(bc, level + 1)
            x = x + xc[lev.agg]
        x = x + self.smooth(lev, b - lev.A @ x)
        return x


class SchurMG:
    """V-cycle used as the preconditioner of Block-Reg's inner PCG on
    S_eps = S_D + eps W ("use it ... as the PCG preconditioner
    inside Block-Reg"; reading R23).  It is built on the matrix S handed
    in, and oracle.solver hands in S_eps itself, not S_D: where K is small, eps W
    exceeds the local spectrum of S_D, and a V-cycle of S_D alone leaves
    cond(V S_eps) ~ 1 + eps / lambda_min (C5-type 12^3: 38 PCG steps to 1e-6 with
    the V-cycle of S_D, 8 with the V-cycle of S_eps, 58 with block Jacobi).
    A fixed symmetric positive definite operator, so plain PCG applies.

      * n_p = 1 (k = 0): one V-cycle of AMG(S), the kind-3 construction above.
      * n_p > 1 (k >= 1), two-grid p-multigrid onto the element-mean moment:
          C(b)  = degree-P_DEGREE (2) Chebyshev with the element-block Jacobi D_B of S
                  on [2/P_RATIO, 2] = [1/3, 2] (oracle.solver.chebyshev; lambda_max(D_B^-1 S) <= 2,
                  reading R15: x'S_eps x <= 2 x'D_B x + eps x'W x; the bound is tight, 1.91 on
                  a 48^3 C5-type mesh), x0 = 0.  Degree 2 on the upper 5/6 of the spectrum
                  instead of degree 3 on [2/30, 2]: the same PCG step count on the C5 family
                  (96^3: 22 vs 23 steps to 1e-8) for two S products per V-cycle fewer
          R r   = r[0::n_p]   (pressure moments are element-major with the mean
                  moment (1/|P|) int q first: a constant pressure has zero
                  higher moments, so injection of the mean is the P_0 coarse space)
          S_c   = R S R^T = S[0::n_p, 0::n_p], solved by one V-cycle of AMG(S_c)
          V(b)  : x = C(b); r = b - S x; x[0::n_p] += AMG(S_c).vcycle(r[0::n_p]);
                  x += C(b - S x)
      * a non-dense coarsest level of either hierarchy (stagnated coarsening: the 18,380-row
        coarsest of C5's mean-moment block) is smoothed by Chebyshev(P_COARSE_DEGREE = 8), not
        the 32 of kind 3: inside a PCG that runs to a tolerance the coarsest solve hardly
        matters (C5-type 96^3, steps to 1e-8: degree 32 / 16 / 8 / 4 -> 22 / 22 / 23 / 28)
    """

    def __init__(self, S, nb, DBinv=None, max_levels=MAX_LEVELS):
        self.S = S.tocsr()
        self.nb = nb
        if nb == 1:
            self.amg = AMG(self.S, coarse_degree=P_COARSE_DEGREE, max_levels=max_levels)
        else:
            from .solver import block_jacobi_inv
            self.DBinv = block_jacobi_inv(self.S, nb) if DBinv is None else DBinv
            self.Sc = self.S[0::nb, 0::nb].tocsr()
            self.Sc.sort_indices()
            self.amg = AMG(self.Sc, coarse_degree=P_COARSE_DEGREE, max_levels=max_levels)

    def smooth(self, b):
        return chebyshev(self.S, self.DBinv, b, P_DEGREE, 2.0, P_RATIO)

    def __call__(self, b):
        if self.nb == 1:
            return self.amg.vcycle(b)
        nb = self.nb
        x = self.smooth(b)
        r = b - self.S @ x
        x = x.copy()
        x[0::nb] += self.amg.vcycle(r[0::nb])
        x = x + self.smooth(b - self.S @ x)
        return x
