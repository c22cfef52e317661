"""Pins for the CPU oracle (oracle/solver.py) against what mathematics fixes.

* Chebyshev: the residual after a degree-d Jacobi-preconditioned Chebyshev
  iteration equals the closed-form scaled Chebyshev polynomial
  T_d((theta - lambda)/delta) / T_d(theta/delta) applied in the eigenbasis of
  D^-1/2 S D^-1/2 (numpy.polynomial.chebyshev, not the recurrence).
* GMRES: after j steps (no restart) the residual is the brute-force minimum
  over the explicit Krylov space (least squares); restarted GMRES / FGMRES
  agree with LAPACK LU to 1e-8 (O9); identity -> 1 iteration; exact diagonal
  preconditioner on a diagonal system -> 1 iteration.
* PCG: agrees with a dense solve; Jacobi on a diagonal matrix -> 1 iteration.
* Block-Reg velocity block: the Woodbury form equals the dense inverse of
  diag(M) + B^T (eps W)^-1 B.
* Exact Block-Schur on the K = I cube with the sin source converges in 2
  iterations (the right-hand side is an eigenvector).
"""
import numpy as np
import pytest
import scipy.sparse as sp
from numpy.polynomial import chebyshev as npcheb

from oracle import solver as O
from vemgen import configs

RNG = np.random.default_rng(77)


def _spd(n, cond=50.0):
    Q, _ = np.linalg.qr(RNG.normal(size=(n, n)))
    lam = np.geomspace(1.0, cond, n)
    return (Q * lam) @ Q.T


@pytest.mark.parametrize("degree", [1, 2, 5, 16])
def test_chebyshev_closed_form(degree):
    n = 40
    S = _spd(n) + np.diag(RNG.uniform(1, 5, n))
    d = np.diag(S).copy()
    Dh = np.diag(1 / np.sqrt(d))
    lam, U = np.linalg.eigh(Dh @ S @ Dh)
    lmax, ratio = 1.05 * lam.max(), 30.0
    v = RNG.normal(size=n)
    x = O.chebyshev(sp.csr_matrix(S), sp.diags(1 / d), v, degree, lmax, ratio)
    a, b = lmax / ratio, lmax
    theta, delta = (a + b) / 2, (b - a) / 2
    cd = np.zeros(degree + 1)
    cd[-1] = 1.0
    rho = npcheb.chebval((theta - lam) / delta, cd) / npcheb.chebval(theta / delta, cd)
    # r = D^1/2 U rho(L) U^T D^-1/2 v
    r_ref = np.sqrt(d) * (U @ (rho * (U.T @ (v / np.sqrt(d)))))
    r = v - S @ x
    assert np.abs(r - r_ref).max() < 1e-12 * np.abs(v).max()


def test_chebyshev_linear():
    S = sp.csr_matrix(_spd(30) + 3 * np.eye(30))
    d = S.diagonal()
    a, b = RNG.normal(size=30), RNG.normal(size=30)
    f = lambda v: O.chebyshev(S, sp.diags(1 / d), v, 16, 2.0, 30.0)  # noqa: E731
    assert np.abs(f(2 * a - 3 * b) - (2 * f(a) - 3 * f(b))).max() < 1e-13 * np.abs(f(a)).max() * 10


@pytest.mark.parametrize("j", [1, 3, 7])
@pytest.mark.parametrize("flexible", [False, True])
def test_gmres_minimal_residual_bruteforce(j, flexible):
    n = 25
    A = RNG.normal(size=(n, n)) + 6 * np.eye(n)
    Pm = np.diag(RNG.uniform(0.5, 2.0, n))
    b = RNG.normal(size=n)
    res = O.gmres(lambda x: A @ x, lambda v: Pm @ v, b, rtol=1e-30, restart=50, maxit=j,
                  flexible=flexible)
    assert res.iterations == j
    AP = A @ Pm
    Kr = [b]
    for _ in range(j - 1):
        Kr.append(AP @ Kr[-1])
    Kr = np.stack(Kr, 1)
    Qk, _ = np.linalg.qr(Kr)
    y, *_ = np.linalg.lstsq(AP @ Qk, b, rcond=None)
    r_ref = np.linalg.norm(b - AP @ Qk @ y)
    r = np.linalg.norm(b - A @ res.x)
    assert abs(r - r_ref) <= 1e-10 * np.linalg.norm(b)


def test_gmres_identity_and_diagonal_one_iteration():
    b = RNG.normal(size=50)
    r = O.gmres(lambda x: x, lambda v: v, b, 1e-12, 30)
    assert r.iterations == 1 and r.converged
    dg = RNG.uniform(1, 10, 50)
    r = O.gmres(lambda x: dg * x, lambda v: v / dg, b, 1e-12, 30)
    assert r.iterations == 1 and r.converged and np.abs(r.x - b / dg).max() < 1e-12


@pytest.mark.parametrize("kind", [O.PRECOND_BLOCK_SCHUR, O.PRECOND_BLOCK_REG])
def test_gmres_vs_lu_c1(kind):
    s = configs.CONFIGS["C1"].build()
    xd = O.dense_solve(s.M, s.B, s.rhs)
    r = O.solve(s.M, s.B, s.rhs, kind, 1e-10, 30, eps=configs.eps_for(s), block=s.layout.n_p_dof)
    assert r.converged and r.rel_residual_true <= 1e-10
    assert np.abs(r.x - xd).max() <= 1e-8 * np.abs(xd).max()


def test_gmres_vs_lu_k1_tets_and_k2_cubes():
    s = configs.CONFIGS["C2s"].build()
    xd = O.dense_solve(s.M, s.B, s.rhs)
    for kind in (O.PRECOND_BLOCK_SCHUR, O.PRECOND_BLOCK_REG):
        r = O.solve(s.M, s.B, s.rhs, kind, 1e-10, 30, eps=configs.eps_for(s), block=s.layout.n_p_dof)
        assert r.converged
        nu = s.layout.n_u
        for sl in (slice(0, nu), slice(nu, None)):
            assert np.abs(r.x[sl] - xd[sl]).max() <= 1e-8 * np.abs(xd[sl]).max()
    s = configs.CONFIGS["C4s"].build()
    xd = O.dense_solve(s.M, s.B, s.rhs)
    r = O.solve(s.M, s.B, s.rhs, O.PRECOND_BLOCK_REG, 1e-10, 50, eps=configs.eps_for(s), block=s.layout.n_p_dof)
    assert r.converged
    nu = s.layout.n_u
    for sl in (slice(0, nu), slice(nu, None)):
        assert np.abs(r.x[sl] - xd[sl]).max() <= 1e-8 * np.abs(xd[sl]).max()


def test_exact_schur_eigenvector_case():
    s = configs.CONFIGS["C1"].build()
    r = O.solve(s.M, s.B, s.rhs, O.PRECOND_BLOCK_SCHUR, 1e-10, 30, exact_schur=True)
    assert r.converged and r.iterations == 2


def test_pcg_dense_and_diagonal():
    A = _spd(60, 1e3)
    b = RNG.normal(size=60)
    x, its, ok = O.pcg(sp.csr_matrix(A), sp.diags(1 / np.diag(A)), b, 1e-12, 1000)
    assert ok and np.abs(x - np.linalg.solve(A, b)).max() < 1e-9 * np.abs(x).max()
    dg = RNG.uniform(1, 100, 60)
    x, its, ok = O.pcg(sp.diags(dg).tocsr(), sp.diags(1 / dg), b, 1e-12, 10)
    assert ok and its == 1
    # exact block preconditioner on a block-diagonal matrix -> 1 iteration
    Bd = sp.block_diag([_spd(4, 10.0) for _ in range(15)]).tocsr()
    x, its, ok = O.pcg(Bd, O.block_jacobi_inv(Bd, 4), b, 1e-12, 10)
    assert ok and its == 1


def test_woodbury_block_reg_velocity_block():
    s = configs.CONFIGS["C1"].build()
    eps = configs.eps_for(s)
    P = O.Preconditioner(O.PRECOND_BLOCK_REG, s.M, s.B, eps=eps, inner_rtol=1e-14, inner_maxit=5000)
    nu = s.layout.n_u
    D = np.diag(s.M.diagonal())
    Bd = s.B.toarray()
    ref = np.linalg.inv(D + Bd.T @ Bd / eps)
    v = RNG.normal(size=s.n)
    z = P.apply(v)
    zu_ref = ref @ v[:nu]
    assert np.abs(z[:nu] - zu_ref).max() < 1e-7 * np.abs(zu_ref).max()
    assert np.abs(z[nu:] - v[nu:] / eps).max() == 0.0


@pytest.mark.parametrize("name", ["C2s", "C4s", "C5s", "C3s"])
def test_block_jacobi_lambda_max_bound(name):
    """lambda_max(D_B^-1 S_D) <= 2 (reading R15) by dense eigenvalues, and
    D_B^-1 is the exact inverse of every element block."""
    s = configs.CONFIGS[name].build()
    nb = s.layout.n_p_dof
    SD = O.schur_diag(s.M, s.B)
    Dinv = O.block_jacobi_inv(SD, nb)
    Sd = SD.toarray()
    for e in (0, SD.shape[0] // nb // 2, SD.shape[0] // nb - 1):
        sl = slice(e * nb, (e + 1) * nb)
        assert np.abs(Dinv[sl, sl].toarray() @ Sd[sl, sl] - np.eye(nb)).max() < 1e-9
    n = min(SD.shape[0], 2500)
    lam = np.linalg.eigvals((Dinv @ SD).toarray()[:n, :n] if n < SD.shape[0] else (Dinv @ SD).toarray())
    if n == SD.shape[0]:
        assert np.real(lam).max() <= 2.0 + 1e-10


def test_spmv_definition():
    s = configs.CONFIGS["C1"].build()
    x = RNG.normal(size=s.n)
    A = sp.bmat([[s.M, s.B.T], [s.B, None]]).toarray()
    assert np.abs(O.spmv_saddle(s.M, s.B, x) - A @ x).max() < 1e-13 * np.abs(A @ x).max()


# ---------------------------------------------------------------------------
# aggregation multigrid for S_D (oracle/amg.py, precond kind 3)
# ---------------------------------------------------------------------------
def _c3s_sd():
    s = configs.CONFIGS["C3s"].build()
    return s, O.schur_diag(s.M, s.B)


def test_amg_aggregates_are_a_valid_mis2_partition():
    from oracle import amg
    s, SD = _c3s_sd()
    agg, nc, is_root = amg.aggregate(SD)
    assert agg.min() == 0 and agg.max() == nc - 1 and np.unique(agg).size == nc
    G = amg.strong_graph(SD)
    roots = np.nonzero(is_root)[0]
    assert np.array_equal(agg[roots], np.arange(roots.size))
    # MIS-2: no two roots within strong distance 2
    G2 = (G @ G).tocsr()
    sub = G2[roots][:, roots]
    assert sub.nnz == roots.size  # only the diagonal
    # every non-singleton node is within distance 2 of its aggregate's root
    root_of = np.full(nc, -1)
    root_of[agg[roots]] = roots
    for i in range(0, SD.shape[0], 7):
        r = root_of[agg[i]]
        if r >= 0:
            assert G2[i, r] != 0


def test_amg_galerkin_conserves_row_sums():
    from oracle import amg
    s, SD = _c3s_sd()
    agg, nc, _ = amg.aggregate(SD)
    Ac = amg.galerkin(SD, agg, nc)
    rs = np.asarray(SD.sum(axis=1)).ravel()
    assert np.allclose(np.asarray(Ac.sum(axis=1)).ravel(), np.bincount(agg, weights=rs, minlength=nc),
                       rtol=1e-12, atol=1e-14 * abs(rs).max())
    assert abs(Ac - Ac.T).max() <= 1e-14 * abs(Ac).max()


def test_amg_one_level_is_exact_and_vcycle_symmetric():
    from oracle import amg
    s, SD = _c3s_sd()
    one = amg.AMG(SD, coarse_size=SD.shape[0])
    b = RNG.normal(size=SD.shape[0])
    assert np.abs(SD @ one.vcycle(b) - b).max() < 1e-9 * np.abs(b).max()
    h = amg.AMG(SD)
    assert len(h.levels) >= 2
    u, v = RNG.normal(size=SD.shape[0]), RNG.normal(size=SD.shape[0])
    assert abs(u @ h.vcycle(v) - v @ h.vcycle(u)) <= 1e-10 * abs(u @ h.vcycle(v))


def test_amg_smoothed_prolongator():
    """Level 0 uses the smoothed-aggregation prolongator P = (I - omega D^-1 S) T
    (Vanek, Mandel & Brezina 1996).  Pinned by what the construction implies, not by
    retyping it: P reproduces (I - omega D^-1 S) applied to the constant; damped
    Jacobi with omega = 4 / (3 lmax) < 2 / lambda_max(D^-1 S) lowers the S-energy of
    every coarse basis vector; the Galerkin operator is the S form restricted to
    range(P); the two-grid correction I - P A_c^-1 P^T S is an S-orthogonal projector."""
    from oracle import amg
    s, SD = _c3s_sd()
    h = amg.AMG(SD)
    lev = h.levels[0]
    assert lev.P is not None and amg.SA_LEVELS == 1
    n, nc = SD.shape[0], lev.nc
    d = SD.diagonal()
    one = np.ones(n)
    omega = 4.0 / (3.0 * lev.lmax)
    assert np.abs(lev.P @ np.ones(nc) - (one - omega * (SD @ one) / d)).max() <= 1e-13
    T = sp.csr_matrix((np.ones(n), (np.arange(n), lev.agg)), shape=(n, nc))
    eP = ((lev.P.T @ SD @ lev.P).diagonal())
    eT = ((T.T @ SD @ T).diagonal())
    assert np.all(eP <= eT * (1 + 1e-12)) and eP.sum() < 0.9 * eT.sum()
    Ac = h.levels[1].A
    xc, yc = RNG.normal(size=nc), RNG.normal(size=nc)
    assert abs(xc @ (Ac @ yc) - (lev.P @ xc) @ (SD @ (lev.P @ yc))) <= 1e-12 * abs(xc @ (Ac @ yc))
    Acd = Ac.toarray()
    E = np.eye(n) - lev.P.toarray() @ np.linalg.solve(Acd, lev.P.T.toarray() @ SD.toarray())
    assert np.abs(E @ E - E).max() <= 1e-8
    SE = SD.toarray() @ E
    assert np.abs(SE - SE.T).max() <= 1e-8 * np.abs(SD.toarray()).max()


def test_amg_fp32_vcycle_is_the_fp64_one_to_fp32_accuracy():
    """Kind 4 rounds the hierarchy to FP32 and runs the V-cycle in FP32: its output
    equals the FP64 V-cycle's to a few FP32 units (a dropped cast or a wrong operand
    would show at O(1)), and FGMRES (the FP32 apply is not exactly linear) with it
    reaches the FP64 tolerance in the FP64 preconditioner's iteration count."""
    from oracle import amg
    s, SD = _c3s_sd()
    h = amg.AMG(SD)
    h32 = h.to_float32()
    b = RNG.normal(size=SD.shape[0])
    x64 = h.vcycle(b)
    x32 = h32.vcycle(b.astype(np.float32))
    assert x32.dtype == np.float32
    assert np.abs(x32 - x64).max() <= 1e-5 * np.abs(x64).max()
    r3 = O.solve(s.M, s.B, s.rhs, O.PRECOND_BLOCK_SCHUR_AMG, 1e-10, 50)
    r4 = O.solve(s.M, s.B, s.rhs, O.PRECOND_BLOCK_SCHUR_AMG_F32, 1e-10, 50)
    assert r4.converged and r4.rel_residual_true <= 1e-10 and abs(r4.iterations - r3.iterations) <= 2


def test_block_schur_amg_gmres_vs_lu():
    for name in ("C1", "C3s"):
        s = configs.CONFIGS[name].build()
        xd = O.dense_solve(s.M, s.B, s.rhs) if s.n < 6000 else None
        r = O.solve(s.M, s.B, s.rhs, O.PRECOND_BLOCK_SCHUR_AMG, 1e-10, configs.CONFIGS[name].restart)
        assert r.converged
        if xd is not None:
            assert np.abs(r.x - xd).max() <= 1e-8 * np.abs(xd).max()


# ---------------------------------------------------------------------------
# pins added in round 2: AMG bounds, the Block-Schur sign, the multigrid inner
# PCG of Block-Reg (reading R23) and the M-aware Block-Reg (kind 5, R24)
# ---------------------------------------------------------------------------
def test_amg_gershgorin_bounds_every_level():
    """The Chebyshev smoother interval top on every level is the Gershgorin bound; it
    must be >= lambda_max(D^-1 A_l) (else the smoother diverges on that level)."""
    from oracle import amg
    import scipy.sparse.linalg as spl
    s, SD = _c3s_sd()
    h = amg.AMG(SD)
    for lev in h.levels:
        A = lev.A
        d = A.diagonal()
        Dh = sp.diags(1 / np.sqrt(d))
        lam = spl.eigsh(Dh @ A @ Dh, k=1, which="LA", return_eigenvectors=False, tol=1e-10)[0]
        assert amg.gershgorin(A) >= lam * (1 - 1e-10)
        assert abs(lev.lmax - amg.gershgorin(A)) == 0.0


def test_amg_vcycle_symmetric_with_chebyshev_coarsest():
    """max_levels = 2 leaves a coarsest level above COARSE_SIZE on C3s-sized grids
    only if coarse_size is lowered: force it, so the coarsest is the Chebyshev(32)
    branch (amg.py: coarse_inv None), and check the V-cycle stays symmetric positive
    definite (the Chebyshev polynomial in D^-1 A is D-symmetric)."""
    from oracle import amg
    s, SD = _c3s_sd()
    h = amg.AMG(SD, coarse_size=64, max_levels=2)
    assert len(h.levels) == 2 and h.coarse_inv is None
    n = SD.shape[0]
    u, v = RNG.normal(size=n), RNG.normal(size=n)
    assert abs(u @ h.vcycle(v) - v @ h.vcycle(u)) <= 1e-10 * abs(u @ h.vcycle(v))
    assert v @ h.vcycle(v) > 0 and u @ h.vcycle(u) > 0


def test_block_schur_sign_tends_to_minus_exact_inverse():
    """Kind 1 applies B_2^-1 = S^-1 with S = -S_D: as the Chebyshev degree
    grows the pressure part of the apply tends to -S_D^-1 v_p (a sign error would
    converge to +S_D^-1 v_p)."""
    s = configs.CONFIGS["C1"].build()
    SD = O.schur_diag(s.M, s.B).toarray()
    v = RNG.normal(size=s.n)
    nu = s.layout.n_u
    ref = -np.linalg.solve(SD, v[nu:])
    errs = []
    for deg in (8, 32, 128):
        P = O.Preconditioner(O.PRECOND_BLOCK_SCHUR, s.M, s.B, cheb_degree=deg, cheb_ratio=400.0)
        errs.append(np.abs(P.apply(v)[nu:] - ref).max() / np.abs(ref).max())
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-4
    assert np.abs(P.apply(v)[:nu] - v[:nu] / s.M.diagonal()).max() == 0.0


@pytest.mark.parametrize("name", ["C3s", "C5s"])
def test_block_jacobi_lambda_max_bound_large(name):
    """lambda_max(D_B^-1 S_D) <= 2 (reading R15) on the configs too large for dense
    eigenvalues, by a Lanczos estimate of the symmetric form D_B^-1/2 S_D D_B^-1/2."""
    import scipy.sparse.linalg as spl
    s = configs.CONFIGS[name].build()
    nb = s.layout.n_p_dof
    SD = O.schur_diag(s.M, s.B)
    # symmetric square root of the block inverse, element by element
    ne = SD.shape[0] // nb
    blocks = []
    for e in range(ne):
        sl = slice(e * nb, (e + 1) * nb)
        w, U = np.linalg.eigh(SD[sl, sl].toarray())
        blocks.append((U / np.sqrt(w)) @ U.T)
    R = sp.block_diag(blocks).tocsr()
    lam = spl.eigsh(R @ SD @ R, k=1, which="LA", return_eigenvectors=False, tol=1e-10)[0]
    assert lam <= 2.0 + 1e-9
    assert lam > 1.0   # S_D couples elements: the bound is not vacuous
    # R is the symmetric square root of D_B^-1 (so R S_D R is similar to D_B^-1 S_D)
    Dinv = O.block_jacobi_inv(SD, nb)
    sl = slice(0, 3 * nb)
    assert np.abs((R @ R)[sl, sl].toarray() - Dinv[sl, sl].toarray()).max() <= 1e-10 * abs(Dinv).max()


@pytest.mark.parametrize("name", ["C2s", "C4s", "C3s", "C5t"])
def test_schur_mg_is_symmetric_positive_definite(name):
    """The inner-PCG preconditioner of Block-Reg (reading R23: one V-cycle of
    S_eps = S_D + eps W) must be SPD: probe its matrix column by column (dense) and
    check symmetry and the smallest eigenvalue."""
    from oracle.amg import SchurMG
    s = configs.CONFIGS[name].build()
    nb = s.layout.n_p_dof
    SD = O.schur_diag(s.M, s.B)
    Se = (SD + configs.eps_for(s) * sp.identity(SD.shape[0])).tocsr()
    V = SchurMG(Se, nb)
    n = SD.shape[0]
    Vm = np.stack([V(e) for e in np.eye(n)], axis=1)
    assert np.abs(Vm - Vm.T).max() <= 1e-10 * np.abs(Vm).max()
    assert np.linalg.eigvalsh(0.5 * (Vm + Vm.T)).min() > 0
    if nb > 1:   # the coarse operator is S_eps restricted to the element-mean moments
        assert np.abs((V.Sc - Se[0::nb, 0::nb]).toarray()).max() == 0.0


@pytest.mark.parametrize("name", ["C2s", "C4s", "C3s", "C5s"])
def test_mg_pcg_dense_solve_and_fewer_steps(name):
    """PCG with the V-cycle preconditioner solves S_D + eps W to the dense solution,
    in fewer steps than the element-block Jacobi PCG (the N1 point of the V-cycle);
    on the C5-type mesh, whose low-K blocks put eps W above the local spectrum of S_D,
    the V-cycle must be the one of S_eps: at least 4 times fewer steps than block
    Jacobi to 1e-6, where the V-cycle of S_D alone saves less than half."""
    from oracle.amg import SchurMG
    s = configs.CONFIGS[name].build()
    nb = s.layout.n_p_dof
    eps = configs.eps_for(s)
    SD = O.schur_diag(s.M, s.B)
    Se = (SD + eps * sp.identity(SD.shape[0])).tocsr()
    b = s.B @ (RNG.normal(size=s.layout.n_u) / s.M.diagonal())
    x, its_mg, ok = O.pcg(Se, SchurMG(Se, nb), b, 1e-14, 1000)
    if SD.shape[0] <= 3000:
        xd = np.linalg.solve(Se.toarray(), b)
    else:
        import scipy.sparse.linalg as spl
        xd = spl.splu(Se.tocsc()).solve(b)
    assert ok and np.abs(x - xd).max() <= 1e-10 * np.abs(xd).max()
    _, its_j, ok_j = O.pcg(Se, O.block_jacobi_inv(Se, nb), b, 1e-14, 10000)
    assert ok_j and its_mg < its_j
    if name == "C5s":
        _, m6, _ = O.pcg(Se, SchurMG(Se, nb), b, 1e-6, 1000)
        _, d6, _ = O.pcg(Se, SchurMG(SD, nb), b, 1e-6, 1000)
        _, j6, _ = O.pcg(Se, O.block_jacobi_inv(Se, nb), b, 1e-6, 10000)
        assert 4 * m6 <= j6 and 2 * d6 > j6


def test_pcg_k_exact_preconditioner_and_limit():
    """pcg_k (kind 5, reading R24): with the exact inverse as preconditioner it stops
    after one step with the exact solution; with the Woodbury-diag preconditioner and
    a small tolerance it converges to the dense K^-1 b, K = M + B^T (eps W)^-1 B."""
    s = configs.CONFIGS["C5t"].build()
    eps = configs.eps_for(s)
    P = O.Preconditioner(O.PRECOND_BLOCK_REG_M, s.M, s.B, eps=eps, block=s.layout.n_p_dof)
    K = (s.M + s.B.T @ s.B / eps).toarray()
    b = RNG.normal(size=s.layout.n_u)
    xd = np.linalg.solve(K, b)
    Kinv = np.linalg.inv(K)
    y, its, ok = O.pcg_k(P.kmul, lambda r: Kinv @ r, b, 1e-8, 10)
    assert ok and its == 1 and np.abs(y - xd).max() <= 1e-7 * np.abs(xd).max()
    y, its, ok = O.pcg_k(P.kmul, lambda r: P.woodbury_d(r, 1e-14), b, 1e-9, 2000)
    assert ok and np.abs(y - xd).max() <= 1e-6 * np.abs(xd).max()
    assert np.abs(P.kmul(b) - K @ b).max() <= 1e-12 * np.abs(K @ b).max()


def test_block_reg_m_gmres_vs_lu_c5t():
    """Kind 5 converges on the C5-type mesh where the diag(M) Block-Reg stagnates
    (DESIGN.md §7), to the LU solution."""
    s = configs.CONFIGS["C5t"].build()
    eps = configs.eps_for(s)
    xd = O.dense_solve(s.M, s.B, s.rhs)
    r = O.solve(s.M, s.B, s.rhs, O.PRECOND_BLOCK_REG_M, 1e-10, 50, eps=eps, block=s.layout.n_p_dof)
    assert r.converged and r.rel_residual_true <= 1e-10
    nu = s.layout.n_u
    for sl in (slice(0, nu), slice(nu, None)):
        assert np.abs(r.x[sl] - xd[sl]).max() <= 1e-8 * np.abs(xd[sl]).max()
    r2 = O.solve(s.M, s.B, s.rhs, O.PRECOND_BLOCK_REG, 1e-10, 50, eps=eps, block=s.layout.n_p_dof, maxit=100)
    assert not r2.converged


@pytest.mark.parametrize("name", ["P1s", "P2s"])
def test_paper_mode_gmres_vs_lu(name):
    """Paper mode (the paper's BDM-type space, pressure P_{k-1}): the oracle's
    preconditioned GMRES reaches the LU solution with both preconditioners (and with the
    V-cycle Block-Schur where the pressure block is scalar, k = 1)."""
    s = configs.CONFIGS[name].build()
    eps = configs.eps_for(s)
    nb = s.layout.n_p_dof
    xd = O.dense_solve(s.M, s.B, s.rhs)
    nu = s.layout.n_u
    for kind in (1, 2) + ((3,) if nb == 1 else ()):
        r = O.solve(s.M, s.B, s.rhs, kind, 1e-10, 50, eps=eps, block=nb)
        assert r.converged, (name, kind)
        for sl in (slice(0, nu), slice(nu, None)):
            assert np.abs(r.x[sl] - xd[sl]).max() <= 1e-8 * np.abs(xd[sl]).max(), (name, kind)


@pytest.mark.parametrize("n,k", [(4, 1), (3, 2)])
def test_paper_neumann_gmres_equals_bordered_lu(n, k):
    """The paper's bordered system [M B^T 0; B 0 c; 0 c^T 0] (Neumann data + mean-value
    multiplier) against the way it goes through the solver: the multiplier
    in closed form (ones.f / ones.c), preconditioned GMRES on the consistent singular saddle
    system [M B^T; B 0][u; p] = [g; f - c lambda], then the projection of p onto c.p = 0.  Both of
    the paper's preconditioners reach the LU solution of the bordered system."""
    import scipy.sparse.linalg as spl
    s, N = configs.paper_neumann(n, k)
    x = spl.spsolve(N.bordered().tocsc(), N.bordered_rhs())
    nu = s.layout.n_u
    ub, pb = x[:nu], x[nu:-1]
    eps = 1e-6 * float(N.M.diagonal().mean())
    for kind in (1, 2):
        r = O.solve(N.M, N.B, N.rhs, kind, 1e-10, 50, eps=eps, block=s.layout.n_p_dof, maxit=2000)
        assert r.converged, (n, k, kind)
        u, p = r.x[:nu], N.project(r.x[nu:])
        assert np.abs(u - ub).max() <= 1e-8 * np.abs(ub).max()
        assert np.abs(p - pb).max() <= 1e-8 * np.abs(pb).max()


@pytest.mark.parametrize("name,kind", [("C1", 1), ("C3s", 3), ("C2s", 1)])
def test_compressed_basis_gmres_vs_lu(name, kind):
    """gmres(basis32=True) (the basis vectors are float32 roundings, the
    arithmetic stays float64): the true-residual restart recovers the full accuracy, so the
    solve still reaches the LU solution to 1e-8 and the true residual 1e-10; every stored
    basis vector is exactly representable in float32 times its scale."""
    s = configs.CONFIGS[name].build()
    cfg = configs.CONFIGS[name]
    xd = O.dense_solve(s.M, s.B, s.rhs) if s.n <= 7000 else None
    r = O.solve(s.M, s.B, s.rhs, kind, 1e-10, cfg.restart, block=s.layout.n_p_dof, basis32=True)
    assert r.converged and r.rel_residual_true <= 1e-10
    full = O.solve(s.M, s.B, s.rhs, kind, 1e-10, cfg.restart, block=s.layout.n_p_dof)
    nu = s.layout.n_u
    for ref in ([xd] if xd is not None else []) + [full.x]:
        for sl in (slice(0, nu), slice(nu, None)):
            assert np.abs(r.x[sl] - ref[sl]).max() <= 1e-8 * np.abs(ref[sl]).max()
    assert r.iterations >= full.iterations     # rounding the basis never helps
