"""CPU oracle for the hot path: block-preconditioned (F)GMRES on the mixed-VEM
saddle-point system.  TEST INFRASTRUCTURE ONLY: may be imported by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs;
never by the product package.  Shares no code with the CUDA path.

Plain fp64 numpy/scipy, written in the order of the paper / SURVEY.md §8(c):
  * spmv_saddle      y = [M x_u + B^T x_p ; B x_u]
  * schur_diag       S_D = B diag(M)^-1 B^T
  * block_jacobi_inv element-block Jacobi D_B^-1 of S_D (n_p x n_p blocks)  (reading R15)
  * chebyshev        degree-d block-Jacobi Chebyshev on [2/ratio, 2]       (O6; Saad Alg. 12.1)
  * block_schur      B_1 = diag(M), B_2^-1 ~ -C_d(S_D)           (reading R15)
  * pcg              block-Jacobi PCG from x0 = 0                (reading R16)
  * block_reg        B_2^-1 = (eps W)^-1, B_1^-1 by Woodbury with diag(M)
                     and an inner PCG on S_D + eps W             (reading R16)
                     whose preconditioner is the element-block Jacobi of
                     S_D + eps W (inner_precond = 0) or one V-cycle of S_D + eps W
                     (inner_precond = 1, oracle/amg.py SchurMG; N1, reading R23)
  * block_reg_m      kind 5: B_2^-1 = (eps W)^-1, B_1^-1 y = PCG on
                     K = M + B^T (eps W)^-1 B (the paper's regularised velocity
                     block itself) preconditioned by the kind-2 B_1,
                     to a relative tolerance k_rtol (reading R24)
  * gmres            right-preconditioned GMRES(m) / FGMRES(m), CGS2 Arnoldi,
                     Givens rotations                            (O8)
  * dense_solve      LAPACK LU of the assembled saddle matrix    (O9)

Pins (tests/test_oracle_pins.py): Chebyshev against the closed-form scaled
Chebyshev residual polynomial; GMRES against brute-force minimal-residual
least squares and against LU; PCG/Woodbury against dense inverses; S_D at k=0
against the two-point-flux closed form.  The iteration counts of the
Chebyshev/PCG stand-ins are *parity unpinned* by the paper (only GPU-vs-oracle
applies), see DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

PRECOND_NONE = 0
PRECOND_BLOCK_SCHUR = 1
PRECOND_BLOCK_REG = 2
PRECOND_BLOCK_SCHUR_AMG = 3     # Block-Schur with one aggregation V-cycle on S_D (oracle/amg.py, R22)
PRECOND_BLOCK_SCHUR_AMG_F32 = 4  # the same V-cycle in FP32 inside the FP64 GMRES
PRECOND_BLOCK_REG_M = 5          # Block-Reg with an M-aware velocity block: PCG on M + B^T (eps W)^-1 B (R24)
INNER_JACOBI = 0                 # Block-Reg inner PCG preconditioner: element-block Jacobi of S_D + eps W
INNER_MG = 1                     # ... one V-cycle of S_D + eps W (oracle/amg.py SchurMG)


def spmv_saddle(M, B, x):
    """y = A x with A = [M B^T; B 0] (C = 0)."""
    nu = M.shape[0]
    xu, xp = x[:nu], x[nu:]
    return np.concatenate([M @ xu + B.T @ xp, B @ xu])


def schur_diag(M, B):
    """S_D = B diag(M)^-1 B^T; the paper's approximate Schur complement is
    S = -C - S_D with C = 0."""
    d = M.diagonal()
    if np.any(d <= 0):
        raise ValueError("non-positive diag(M)")
    return (B @ sp.diags(1.0 / d) @ B.T).tocsr()


def gershgorin_lmax(S):
    """Gershgorin bound of diag(S)^-1 S: max_i sum_j |S_ij| / S_ii (reported only)."""
    a = abs(S).sum(axis=1).A1
    return float(np.max(a / S.diagonal()))


# lambda_max(D_B^-1 S_D) <= 2 for the element-block Jacobi D_B of S_D = B D^-1 B^T
# whenever every velocity DOF touches at most two elements (reading R15):
# S_D = sum_j b_j b_j^T / d_j, each term a PSD matrix on <= 2 element blocks, and a
# PSD 2x2-block matrix is bounded by twice its block diagonal.
LAMBDA_MAX_BLOCK_JACOBI = 2.0


def block_jacobi_inv(S, nb):
    """D_B^-1: inverses of the nb x nb diagonal blocks of S (pressure DOFs are
    numbered element-major, so block e = rows/cols [e nb, (e+1) nb)).  nb = 1 is
    point Jacobi."""
    n = S.shape[0]
    if nb == 1:
        return sp.diags(1.0 / S.diagonal()).tocsr()
    ne = n // nb
    S = S.tocsr()
    blocks = np.zeros((ne, nb, nb))
    for a in range(nb):
        for b in range(nb):
            blocks[:, a, b] = np.asarray(S[np.arange(ne) * nb + a, np.arange(ne) * nb + b]).ravel()
    inv = np.linalg.inv(blocks)
    r = (np.arange(ne)[:, None, None] * nb + np.arange(nb)[None, :, None]).repeat(nb, axis=2)
    c = (np.arange(ne)[:, None, None] * nb + np.arange(nb)[None, None, :]).repeat(nb, axis=1)
    return sp.csr_matrix((inv.ravel(), (r.ravel(), c.ravel())), shape=S.shape)


def chebyshev(S, Dinv, v, degree, lmax, ratio):
    """Degree-`degree` Chebyshev iteration for S x = v, preconditioner D^-1
    (a matrix: element-block Jacobi), interval [lmax/ratio, lmax], x0 = 0.  Saad, Iterative
    Methods, Alg. 12.1, exactly as SURVEY.md §8(c) O6 writes it:
        theta = (b+a)/2, delta = (b-a)/2, sigma = theta/delta, rho_0 = 1/sigma
        r_0 = v, d_0 = D^-1 r_0 / theta, x = d_0
        for i = 1 .. degree-1:
            r_i = r_{i-1} - S d_{i-1}
            rho_i = 1/(2 sigma - rho_{i-1})
            d_i = rho_i rho_{i-1} d_{i-1} + (2 rho_i / delta) D^-1 r_i
            x += d_i
    """
    b = lmax
    a = lmax / ratio
    theta = 0.5 * (b + a)
    delta = 0.5 * (b - a)
    sigma = theta / delta
    rho = 1.0 / sigma
    r = v.copy()
    d = (Dinv @ r) / theta
    x = d.copy()
    for _ in range(1, degree):
        r = r - S @ d
        rho_new = 1.0 / (2.0 * sigma - rho)
        d = rho_new * rho * d + (2.0 * rho_new / delta) * (Dinv @ r)
        rho = rho_new
        x = x + d
    return x


def pcg(A, Dinv, b, rtol, maxit):
    """Preconditioned CG (preconditioner Dinv: a matrix, or a callable z = Dinv(r))
    from x0 = 0; stops when ||r||_2 <= rtol ||b||_2 (Hestenes-Stiefel recurrences).
    Returns (x, iterations, converged)."""
    if callable(Dinv):
        prec = Dinv
    else:
        def prec(r):
            return Dinv @ r
    x = np.zeros_like(b)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return x, 0, True
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        q = A @ p
        alpha = rz / (p @ q)
        x = x + alpha * p
        r = r - alpha * q
        if np.linalg.norm(r) <= rtol * bn:
            return x, it, True
        z = prec(r)
        rz_new = r @ z
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    return x, maxit, False


def pcg_k(Kmul, prec, b, rtol, maxit):
    """PCG for the regularised velocity block K y = b (kind 5, reading R24) from
    y0 = 0 with the SPD preconditioner `prec`; stops when the preconditioned
    residual norm sqrt(r.z) <= rtol sqrt(r_0.z_0) (K = M + B^T (eps W)^-1 B has
    eigenvalues of order 1/eps on range(B^T), so the 2-norm of r would only
    measure that part).  Returns (y, iterations, converged)."""
    y = np.zeros_like(b)
    if not np.any(b):
        return y, 0, True
    r = b.copy()
    z = prec(r)
    rz = r @ z
    rz0 = rz
    p = z.copy()
    for it in range(1, maxit + 1):
        q = Kmul(p)
        alpha = rz / (p @ q)
        y = y + alpha * p
        r = r - alpha * q
        z = prec(r)
        rz_new = r @ z
        if np.sqrt(abs(rz_new)) <= rtol * np.sqrt(rz0):
            return y, it, True
        p = z + (rz_new / rz) * p
        rz = rz_new
    return y, maxit, False


@dataclass
class Preconditioner:
    kind: int
    M: object
    B: object
    cheb_degree: int = 16
    cheb_ratio: float = 30.0
    eps: float = 0.0
    inner_rtol: float = 1e-14
    inner_maxit: int = 10000
    exact_schur: bool = False          # pins only: B_2^-1 = -S_D^-1 exactly
    block: int = 1                     # n_p: pressure DOFs per element (element-block Jacobi)
    inner_precond: int = INNER_MG      # Block-Reg inner PCG preconditioner (R23)
    k_rtol: float = 0.1                # kind 5: relative tolerance of the PCG on K (R24)
    k_maxit: int = 500
    k_inner_rtol: float = 1e-8         # kind 5: inner PCG tolerance of the Woodbury preconditioner (R24)
    inner_iterations: int = 0
    k_iterations: int = 0
    inner_failed: bool = False
    _cache: dict = field(default_factory=dict)

    def __post_init__(self):
        self.nu = self.M.shape[0]
        self.dM = self.M.diagonal().copy()
        if self.kind in (PRECOND_BLOCK_SCHUR, PRECOND_BLOCK_REG, PRECOND_BLOCK_SCHUR_AMG, PRECOND_BLOCK_SCHUR_AMG_F32,
                         PRECOND_BLOCK_REG_M):
            self.SD = schur_diag(self.M, self.B)
            self.dS = self.SD.diagonal().copy()
            if np.any(self.dS <= 0):
                raise ValueError("non-positive diag(S_D)")
            self.DBinv = block_jacobi_inv(self.SD, self.block)
            self.lmax = LAMBDA_MAX_BLOCK_JACOBI
        if self.kind in (PRECOND_BLOCK_SCHUR_AMG, PRECOND_BLOCK_SCHUR_AMG_F32):
            if self.block != 1:
                raise NotImplementedError("Block-Schur-AMG is defined for n_p = 1 (k = 0) in this round")
            from .amg import AMG
            self.amg = AMG(self.SD)
            if self.kind == PRECOND_BLOCK_SCHUR_AMG_F32:
                self.amg = self.amg.to_float32()
        if self.kind in (PRECOND_BLOCK_REG, PRECOND_BLOCK_REG_M):
            if self.eps <= 0:
                raise ValueError("eps must be > 0")
            self.Seps = (self.SD + self.eps * sp.identity(self.SD.shape[0], format="csr")).tocsr()
            if self.inner_precond == INNER_MG:
                from .amg import SchurMG
                self.inner_prec = SchurMG(self.Seps, self.block)
            else:
                self.inner_prec = block_jacobi_inv(self.Seps, self.block)

    @property
    def flexible(self) -> bool:
        # FGMRES for the variable preconditioners: Block-Reg (inner PCG) and the FP32
        # V-cycle (its rounding makes P^-1 (V y) differ from sum_j y_j P^-1 v_j)
        return self.kind in (PRECOND_BLOCK_REG, PRECOND_BLOCK_SCHUR_AMG_F32, PRECOND_BLOCK_REG_M)

    def woodbury_d(self, vu, rtol=None):
        """(diag(M) + B^T (eps W)^-1 B)^-1 vu = D^-1 vu - D^-1 B^T (eps W + S_D)^-1 B D^-1 vu
        (Woodbury; the inner solve is the PCG of reading R16/R23 to rtol, default inner_rtol)."""
        t0 = vu / self.dM
        s = self.B @ t0
        t, its, ok = pcg(self.Seps, self.inner_prec, s, self.inner_rtol if rtol is None else rtol, self.inner_maxit)
        self.inner_iterations += its
        self.inner_failed |= not ok
        return t0 - (self.B.T @ t) / self.dM

    def kmul(self, y):
        """K y = M y + B^T (eps W)^-1 B y, W = I."""
        return self.M @ y + (self.B.T @ (self.B @ y)) / self.eps

    def apply(self, v):
        nu = self.nu
        if self.kind == PRECOND_NONE:
            return v.copy()
        vu, vp = v[:nu], v[nu:]
        if self.kind == PRECOND_BLOCK_SCHUR:
            zu = vu / self.dM
            if self.exact_schur:
                import scipy.sparse.linalg as spl
                if "lu" not in self._cache:
                    self._cache["lu"] = spl.splu(self.SD.tocsc())
                zp = -self._cache["lu"].solve(vp)
            else:
                zp = -chebyshev(self.SD, self.DBinv, vp, self.cheb_degree, self.lmax, self.cheb_ratio)
            return np.concatenate([zu, zp])
        if self.kind == PRECOND_BLOCK_SCHUR_AMG:
            return np.concatenate([vu / self.dM, -self.amg.vcycle(vp)])
        if self.kind == PRECOND_BLOCK_SCHUR_AMG_F32:
            return np.concatenate([vu / self.dM, -self.amg.vcycle(vp.astype(np.float32)).astype(np.float64)])
        if self.kind == PRECOND_BLOCK_REG:
            # B_2^-1 = (eps W)^-1 with W = I
            zp = vp / self.eps
            # B_1^-1 = (D + B^T (eps W)^-1 B)^-1 = D^-1 - D^-1 B^T (eps W + B D^-1 B^T)^-1 B D^-1
            zu = self.woodbury_d(vu)
            return np.concatenate([zu, zp])
        if self.kind == PRECOND_BLOCK_REG_M:
            zp = vp / self.eps
            # B_1^-1 ~ K^-1 = (M + B^T (eps W)^-1 B)^-1 by PCG, preconditioned by the kind-2 B_1
            zu, its, ok = pcg_k(self.kmul, lambda r: self.woodbury_d(r, self.k_inner_rtol), vu, self.k_rtol,
                                self.k_maxit)
            self.k_iterations += its
            self.inner_failed |= not ok
            return np.concatenate([zu, zp])
        raise ValueError(f"unsupported precond kind {self.kind}")


@dataclass
class GmresResult:
    x: np.ndarray
    iterations: int
    restarts: int
    converged: bool
    breakdown: bool
    rel_residual_true: float
    rel_residual_est: float
    history: list


def gmres(matvec, precond, b, rtol=1e-10, restart=30, maxit=10000, flexible=False, reorth=1, basis32=False):
    """Right-preconditioned restarted GMRES(m) (flexible=True: FGMRES(m), which
    stores Z_j = P^-1 v_j), x0 = 0, classical Gram-Schmidt applied twice
    (CGS2; reorth=0: once, CGS1), Givens rotations.  Follows SURVEY.md §8(c) O8:
      beta = ||b||; converged when |g_{j+1}| <= rtol * beta; happy breakdown when
      h_{j+1,j} <= 1e-14 ||A z_j||; at cycle end x += P^-1 (V y) (or Z y), the
      true residual r = b - A x is recomputed and the solve stops only if
      ||r|| <= rtol * beta.  `iterations` counts Arnoldi steps.

    basis32 (traffic-reduced Krylov: a compressed basis): every basis
    vector is the float32 rounding of the vector Arnoldi produced, fl32(r) / beta and
    fl32(w) / ||fl32(w)||, used as such everywhere (preconditioner input, dot products,
    updates, the combination at the cycle end), all arithmetic staying in float64; the
    Arnoldi relation then holds up to 6e-8 per step and the true-residual restart
    (iterative refinement) recovers the full accuracy.
    """
    n = b.shape[0]
    x = np.zeros(n)
    bnorm = np.linalg.norm(b)
    hist = []
    if bnorm == 0.0:
        return GmresResult(x, 0, 0, True, False, 0.0, 0.0, hist)
    r = b.copy()
    beta = bnorm
    its = 0
    restarts = 0
    breakdown = False
    est = 1.0
    while True:
        m = restart
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n)) if flexible else None
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = (r.astype(np.float32).astype(np.float64) if basis32 else r) / beta
        j_done = 0
        conv = False
        for j in range(m):
            z = precond(V[j])
            if flexible:
                Z[j] = z
            w = matvec(z)
            its += 1
            wnorm0 = np.linalg.norm(w)
            h1 = V[:j + 1] @ w
            w = w - V[:j + 1].T @ h1
            if reorth:
                h2 = V[:j + 1] @ w
                w = w - V[:j + 1].T @ h2
                H[:j + 1, j] = h1 + h2
            else:
                H[:j + 1, j] = h1
            if basis32:
                w = w.astype(np.float32).astype(np.float64)
            hn = np.linalg.norm(w)
            H[j + 1, j] = hn
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            rr = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / rr
            sn[j] = H[j + 1, j] / rr
            H[j, j] = rr
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / bnorm
            hist.append(est)
            j_done = j + 1
            if abs(g[j + 1]) <= rtol * bnorm:
                conv = True
                break
            if hn <= 1e-14 * wnorm0:
                breakdown = True
                break
            if its >= maxit:
                break
            V[j + 1] = w / hn
        # y = R^-1 g (back substitution)
        k = j_done
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        if flexible:
            x = x + Z[:k].T @ y
        else:
            x = x + precond(V[:k].T @ y)
        r = b - matvec(x)
        beta = np.linalg.norm(r)
        true_rel = beta / bnorm
        if true_rel <= rtol:
            return GmresResult(x, its, restarts, True, breakdown, true_rel, est, hist)
        # a (numerically) invariant Krylov space ends the cycle; the solve only
        # fails on a breakdown at the first step of a cycle (no progress possible)
        if its >= maxit or (breakdown and j_done == 1):
            return GmresResult(x, its, restarts, False, breakdown, true_rel, est, hist)
        breakdown = False
        restarts += 1


def solve(M, B, rhs, precond_kind=PRECOND_BLOCK_SCHUR, rtol=1e-10, restart=30, maxit=10000,
          eps=0.0, cheb_degree=16, cheb_ratio=30.0, inner_rtol=1e-14, inner_maxit=10000,
          exact_schur=False, block=1, reorth=-1, inner_precond=INNER_MG, k_rtol=0.1, k_maxit=500,
          k_inner_rtol=1e-8, basis32=False):
    """Oracle counterpart of vem_mixed_upload + vem_mixed_solve; `block` is
    the number of pressure DOFs per element (layout.n_p_dof).  reorth = -1
    (auto, reading R17): CGS1 for GMRES, CGS2 for the Block-Reg
    FGMRES (kinds 2 and 5), CGS1 for the FP32-V-cycle FGMRES (kind 4)."""
    if reorth < 0:
        reorth = 1 if precond_kind in (PRECOND_BLOCK_REG, PRECOND_BLOCK_REG_M) else 0
    P = Preconditioner(precond_kind, M, B, cheb_degree, cheb_ratio, eps, inner_rtol, inner_maxit,
                       exact_schur, block=block, inner_precond=inner_precond, k_rtol=k_rtol, k_maxit=k_maxit,
                       k_inner_rtol=k_inner_rtol)
    res = gmres(lambda x: spmv_saddle(M, B, x), P.apply, rhs, rtol, restart, maxit, P.flexible, reorth, basis32)
    res.inner_iterations = P.inner_iterations
    res.k_iterations = P.k_iterations
    res.inner_failed = P.inner_failed
    return res


def dense_solve(M, B, rhs):
    """x = A^-1 rhs by LAPACK LU of the dense saddle matrix (O9; small cases)."""
    A = sp.bmat([[M, B.T], [B, None]]).toarray()
    return np.linalg.solve(A, rhs)
