"""Pins for the input generator (the assembled mixed-VEM system).

Each test checks the assembler against something the paper or the mathematics
fixes, not against a retyped formula:
  * dimensions of G_k^perp and ker(x ^ .) by numerical rank
  * Props. 1-3 and Prop. inTermsOfGPerpBasis as polynomial identities
  * the paper's own cube DOF totals (Tables 1, 4; tests/golden/paper_cube_dofs.txt)
  * Pi^0_k o interpolation = identity, div o interpolation = analytic divergence
  * the k=0 closed form (two-point flux) on cubes with K jumps
  * symmetry / SPD of M, full row rank of B, local conservation, h^{k+1} rates,
    linear-pressure patch test.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spl

from vemgen import assemble, configs, local, mesh, poly

RNG = np.random.default_rng(1234)


def _grad_monomial(beta, s):
    out = np.zeros(s.shape)
    for d in range(3):
        if beta[d] == 0:
            continue
        b = list(beta)
        b[d] -= 1
        out[:, d] = beta[d] * np.prod(s ** np.array(b), axis=1)
    return out


def _vec_mono(c, a, s):
    v = np.zeros(s.shape)
    v[:, c] = np.prod(s ** np.array(a), axis=1)
    return v


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_gperp_dimension_and_generator_basis(k):
    """rank{m_I ^ g : g in M^{G,+}_{k-1}} = dim G_k^perp = (2k^3+9k^2+7k)/6 and,
    together with grad m_b (1<=|b|<=k+1), spans [P_k]^3 (reading R2)."""
    s = RNG.uniform(-1, 1, size=(400, 3))
    gens = poly.generators(k)
    cols = [np.cross(s, _vec_mono(c, a, s)).reshape(-1) for c, a in gens]
    Gm = np.stack(cols, 1)
    assert np.linalg.matrix_rank(Gm) == len(gens) == poly.dim_gperp(k)
    grads = [_grad_monomial(b, s).reshape(-1) for b in poly.multi_indices_3d(k + 1) if sum(b) > 0]
    full = np.concatenate([np.stack(grads, 1), Gm], 1)
    assert np.linalg.matrix_rank(full) == 3 * poly.dim_pk_3d(k)
    # the printed "0 < |alpha|" set is rank deficient by exactly one
    gens_bad = [(c, a) for c, a in gens if not (c == 0 and sum(a) == 0)]
    Gb = np.stack([np.cross(s, _vec_mono(c, a, s)).reshape(-1) for c, a in gens_bad], 1)
    assert np.linalg.matrix_rank(Gb) == poly.dim_gperp(k) - 1


@pytest.mark.parametrize("k", [1, 2, 3])
def test_kernel_of_x_cross(k):
    """dim ker(x ^ .) on [P_{k-1}]^3 = k(k-1)(k+1)/6 (Corollary)."""
    s = RNG.uniform(-1, 1, size=(400, 3))
    cols = [np.cross(s, _vec_mono(c, a, s)).reshape(-1)
            for c in range(3) for a in poly.multi_indices_3d(k - 1)]
    A = np.stack(cols, 1)
    assert A.shape[1] - np.linalg.matrix_rank(A) == k * (k - 1) * (k + 1) // 6


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_props_1_to_3_identities(k):
    """e_c m_a = (h/(|a|+1)) grad m_b + sum coef m_I ^ (...), evaluated at
    random points (h_P = 1, x_P = 0), then rewritten in the generator basis."""
    s = RNG.uniform(-1, 1, size=(50, 3))
    for c in range(3):
        for a in poly.multi_indices_3d(k):
            gc, beta, cross = poly.decompose_vector_monomial(c, a)
            rhs = gc * _grad_monomial(beta, s)
            rhs2 = rhs.copy()
            for coef, cc, al in cross:
                rhs += coef * np.cross(s, _vec_mono(cc, al, s))
                for coef2, c2, al2 in poly.cross_term_as_generators(cc, al):
                    rhs2 += coef * coef2 * np.cross(s, _vec_mono(c2, al2, s))
            lhs = _vec_mono(c, a, s)
            assert np.abs(lhs - rhs).max() < 1e-12
            assert np.abs(lhs - rhs2).max() < 1e-12


def test_paper_cube_dof_totals():
    """The paper's BDM-type DOF count N_F (k+1)(k+2)/2 + N_P [(dim P_{k-1} - 1)
    + dim G_k^perp + dim P_{k-1}] + 1 with N_F from our cube generator
    reproduces every Cube-mesh header of Tables 1 and 4 exactly."""
    path = os.path.join(os.path.dirname(__file__), "golden", "paper_cube_dofs.txt")
    rows = [l.split()[:3] for l in open(path) if l.strip() and not l.startswith("#")]
    assert len(rows) == 8
    for NP, k, dofs in rows:
        NP, k, dofs = int(NP), int(k), int(dofs)
        n = round(NP ** (1 / 3))
        assert n ** 3 == NP
        nf = 3 * n * n * (n + 1)
        if n <= 12:
            assert mesh.cube_mesh(n).n_faces == nf
        got = nf * poly.dim_pk_2d(k) + NP * ((poly.dim_pk_3d(k - 1) - 1) + len(poly.generators(k))
                                              + poly.dim_pk_3d(k - 1)) + 1
        assert got == dofs


def test_mesh_counts():
    assert mesh.cube_mesh(5).n_faces == 3 * 25 * 6
    for n in (2, 3):
        m = mesh.kuhn_mesh(n)
        assert m.n_faces == 12 * n ** 3 + 6 * n ** 2 and m.n_cells == 6 * n ** 3
        vol = sum(c.vol.sum() for c in m.classes)
        assert abs(vol - 1.0) < 1e-12
    m = mesh.pair_mesh(12, seed=5, block=3)
    cells = m.meta["n_pairs"] * 2
    assert cells >= 12 ** 3 // 2
    assert m.n_cells == 12 ** 3 - m.meta["n_pairs"]
    assert m.n_faces == 3 * 144 * 13 - m.meta["n_pairs"]


def test_config_sizes():
    """SURVEY.md §0 item 4 / BASELINE.json C1 (1728 face + 512 element DOFs)."""
    s = configs.CONFIGS["C1"].build()
    assert (s.layout.n_u, s.layout.n_p) == (1728, 512)
    lay = assemble.Layout(0, 1, 0, 1, 3 * 128 * 128 * 129, 128 ** 3)
    assert (lay.n_u, lay.n_p) == (6340608, 2097152)
    lay = assemble.Layout(2, 6, 20, 10, 3 * 48 * 48 * 49, 48 ** 3)
    assert (lay.n_u, lay.n_p) == (4243968, 1105920)
    lay = assemble.Layout(1, 3, 6, 4, 12 * 16 ** 3 + 6 * 16 ** 2, 6 * 16 ** 3)
    assert (lay.n_u, lay.n_p) == (299520, 98304)


def _meshes():
    return [("cube", mesh.cube_mesh(2)), ("kuhn", mesh.kuhn_mesh(2, seed=7)),
            ("pairs", mesh.pair_mesh(4, seed=5, block=2))]


@pytest.mark.parametrize("k", [0, 1, 2])
def test_projection_reproduces_polynomials(k):
    """Pi^0_k(interp(p)) = p for p in [P_k]^3: Pi @ D = I."""
    for name, m in _meshes():
        for cls in m.classes:
            o = local.local_operators(cls.rep(), k)
            PD = np.einsum("eil,elj->eij", o["Pi"], o["D"])
            assert np.abs(PD - np.eye(PD.shape[1])).max() < 1e-9, (name, cls.name)


@pytest.mark.parametrize("k", [0, 1, 2])
def test_divergence_of_interpolant(k):
    """Div(interp(v)) equals the analytic divergence of v in [P_k]^3 (commuting
    divergence)."""
    for name, m in _meshes():
        cls = m.classes[-1]
        g = cls.rep()
        o = local.local_operators(g, k)
        alphas = poly.multi_indices_3d(k)
        im = poly.index_map_3d(k)
        nk = len(alphas)
        h = g["h"][0]
        coef = RNG.normal(size=3 * nk)
        # analytic divergence coefficients: d/dx_c (m_a) = a_c / h m_{a-e_c}
        dv = np.zeros(nk)
        for c in range(3):
            for a, al in enumerate(alphas):
                if al[c]:
                    am = list(al); am[c] -= 1
                    dv[im[tuple(am)]] += coef[c * nk + a] * al[c] / h
        got = o["Div"][0] @ (o["D"][0] @ coef)
        assert np.abs(got - dv).max() < 1e-9 * max(1, np.abs(dv).max()), name


def test_k0_cube_closed_form():
    """O-K0: M tridiagonal along grid lines with diagonal (3/4)h^3(1/K1+1/K2),
    off-diagonal -(1/4)h^3/K_P; B_{P,f} = -sigma h^2; S_D off-diagonal
    -(4h/3) K1 K2/(K1+K2) and boundary faces add (4/3) h K_P to the diagonal."""
    cfg = configs.CONFIGS["C3s"]
    m = cfg.make_mesh()
    s = assemble.build_system(m, 0)
    n, h = m.meta["n"], m.meta["h"]
    K = m.K[:, 0]
    assert s.M.nnz == 3 * s.layout.n_u - 2 * (3 * n * n)   # 3 per interior row, 2 per boundary row
    M = s.M.tocoo()
    # check every entry against the closed form
    cl = m.classes[0]
    Mref = sp.lil_matrix(s.M.shape)
    Bref = sp.lil_matrix(s.B.shape)
    for e in range(m.n_cells):
        for d in range(3):
            fm, fp = cl.face_ids[e, 2 * d], cl.face_ids[e, 2 * d + 1]
            w = h ** 3 / K[e]
            Mref[fm, fm] += 0.75 * w; Mref[fp, fp] += 0.75 * w
            Mref[fm, fp] += -0.25 * w; Mref[fp, fm] += -0.25 * w
            Bref[e, fm] = h * h; Bref[e, fp] = -h * h
    assert abs(s.M - Mref.tocsr()).max() < 1e-15 * abs(Mref).max() * 10
    assert abs(s.B - Bref.tocsr()).max() < 1e-15
    from oracle.solver import schur_diag
    SD = schur_diag(s.M, s.B).tocsr()
    # off-diagonal across each interior face, boundary contributions on the diagonal
    for e in range(0, m.n_cells, 37):
        i, j, kk = e % n, (e // n) % n, e // (n * n)
        diag = 0.0
        for d, (di, dj, dk) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
            for sgn in (-1, 1):
                a, b, c = i + sgn * di, j + sgn * dj, kk + sgn * dk
                if 0 <= a < n and 0 <= b < n and 0 <= c < n:
                    nb = a + n * (b + n * c)
                    t = 4 * h / 3 * K[e] * K[nb] / (K[e] + K[nb])
                    assert abs(SD[e, nb] + t) < 1e-12 * t
                    diag += t
                else:
                    diag += 4 * h / 3 * K[e]
        assert abs(SD[e, e] - diag) < 1e-12 * diag


def test_rhs_k0_closed_form():
    """int_P 3 pi^2 prod sin(pi x) = 3 pi^2 prod (cos pi a - cos pi b)/pi; f_P = -int_P f."""
    n = 8
    s = assemble.build_system(mesh.cube_mesh(n), 0)
    idx = np.arange(n ** 3)
    ijk = np.stack([idx % n, (idx // n) % n, idx // (n * n)], 1) / n
    ref = 3 * np.pi ** 2 * np.prod((np.cos(np.pi * ijk) - np.cos(np.pi * (ijk + 1 / n))) / np.pi, axis=1)
    assert np.abs(s.f + ref).max() < 1e-13


@pytest.mark.parametrize("name,k", [("kuhn", 1), ("kuhn", 2), ("pairs", 1), ("cube", 2)])
def test_M_symmetric_spd_and_B_full_rank(name, k):
    m = {"kuhn": lambda: mesh.kuhn_mesh(2, seed=3), "pairs": lambda: mesh.pair_mesh(4, seed=5, block=2),
         "cube": lambda: mesh.cube_mesh(3)}[name]()
    s = assemble.build_system(m, k)
    M = s.M.toarray()
    assert np.abs(M - M.T).max() <= 1e-12 * np.abs(M).max()
    np.linalg.cholesky(0.5 * (M + M.T))
    SD = (s.B @ sp.diags(1 / s.M.diagonal()) @ s.B.T).toarray()
    np.linalg.cholesky(SD)      # S_D SPD <=> B full row rank
    assert np.linalg.matrix_rank(s.B.toarray()) == s.layout.n_p


def _direct(s):
    A = sp.bmat([[s.M, s.B.T], [s.B, None]]).tocsc()
    x = spl.spsolve(A, s.rhs)
    return x[:s.layout.n_u], x[s.layout.n_u:]


@pytest.mark.parametrize("kind,k,ns", [("cube", 0, (4, 8, 16)), ("cube", 1, (2, 4, 8)),
                                       ("cube", 2, (2, 4)), ("kuhn", 1, (2, 4)),
                                       ("pairs", 1, (4, 8))])
def test_convergence_rates_and_conservation(kind, k, ns):
    """e_u, e_p ~ h^{k+1} (reading R3; BASELINE north_star) and B u_h = f_h
    element by element (local conservation)."""
    errs = []
    for n in ns:
        m = {"cube": lambda: mesh.cube_mesh(n), "kuhn": lambda: mesh.kuhn_mesh(n, seed=2),
             "pairs": lambda: mesh.pair_mesh(n, seed=5, block=2)}[kind]()
        s = assemble.build_system(m, k, keep_local=True)
        u, p = _direct(s)
        assert np.abs(s.B @ u - s.f).max() <= 1e-10 * np.abs(s.f).max()
        errs.append(assemble.l2_errors(s, u, p))
    errs = np.array(errs)
    rates = np.log2(errs[:-1] / errs[1:])
    lo, hi = k + 1 - 0.25, k + 1 + 0.4
    assert np.all((rates[-1] >= lo) & (rates[-1] <= hi)), rates


@pytest.mark.parametrize("k", [1, 2])
def test_patch_test_linear_pressure(k):
    """p = 1 + 2x - y + 3z with Dirichlet data g_D = p: the discrete solution
    is exact (u = -grad p constant, p_h = p) to round-off."""
    m = mesh.kuhn_mesh(2, seed=11)
    grad = np.array([2.0, -1.0, 3.0])
    pfun = lambda x: 1 + x @ grad  # noqa: E731
    s = assemble.build_system(m, k, source=lambda x: np.zeros(x.shape[:-1]), gD=pfun, keep_local=True)
    u, p = _direct(s)
    cls, ops, L, P = s.local[0]
    nk = poly.dim_pk_3d(k)
    cu = np.einsum("eil,el->ei", ops["Pi"], u[L])
    for c in range(3):
        assert np.abs(cu[:, c * nk] + grad[c]).max() < 1e-8
        assert np.abs(cu[:, c * nk + 1:(c + 1) * nk]).max() < 1e-8
    pc = assemble.pressure_coeffs(s, p)[0][1]
    xP, h = cls.centroid, cls.h
    assert np.abs(pc[:, 0] - pfun(xP)).max() < 1e-8
    assert np.abs(pc[:, 1:4] - h[:, None] * grad[None, :]).max() < 1e-8


def test_class_templates_recombine_to_the_assembled_system():
    """The shape cache handed to the device assembly (class_template) recombines on the
    host into exactly the M, B, f that build_system assembles (C5s: cube and pair
    classes; C4s: k = 2), and Kuhn tetrahedra are refused (not congruent)."""
    import numpy as np
    import scipy.sparse as sp
    from vemgen import configs
    from vemgen.assemble import class_templates
    for name in ("C5s", "C4s"):
        cfg = configs.CONFIGS[name]
        s = cfg.build()
        rows, cols, vals, brows, bcols, bvals = [], [], [], [], [], []
        f = np.zeros(s.layout.n_p)
        for t in class_templates(cfg.make_mesh(), cfg.k):
            c = t["coef"]
            v = (c[:, 0, None] * t["A"][0] + c[:, 1, None] * t["A"][1] + c[:, 2, None] * t["A"][2]
                 + c[:, 3, None] * t["S"])
            rows.append(t["L"][:, t["ii"]].ravel()); cols.append(t["L"][:, t["jj"]].ravel()); vals.append(v.ravel())
            brows.append(t["P"][:, t["bi"]].ravel()); bcols.append(t["L"][:, t["bj"]].ravel())
            bvals.append(np.broadcast_to(t["B"], (t["L"].shape[0], len(t["bi"]))).ravel())
            f[t["P"].ravel()] = (-t["vol"][:, None] * (t["F"] @ t["Hinv"].T)).ravel()
        M = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=s.M.shape).tocsr()
        B = sp.coo_matrix((np.concatenate(bvals), (np.concatenate(brows), np.concatenate(bcols))),
                          shape=s.B.shape).tocsr()
        assert abs(M - s.M).max() <= 1e-15 * abs(s.M).max()
        assert abs(B - s.B).max() == 0.0
        assert np.abs(f - s.f).max() <= 1e-14 * np.abs(s.f).max()
    import pytest
    with pytest.raises(ValueError):
        class_templates(configs.CONFIGS["C2s"].make_mesh(), 1)


# ---------------------------------------------------------------------------
# Paper mode: the paper's own BDM-type space, gradient moments over
# M_{k-1} \ M_0, divergence and pressure in P_{k-1}
# ---------------------------------------------------------------------------
def test_paper_mode_dof_totals_from_the_assembler():
    """The assembler's own layout in paper mode reproduces the paper's Cube-mesh DOF totals
    (Tables 1 and 4, tests/golden/paper_cube_dofs.txt) up to the single mean-value
    multiplier the paper's Neumann problem adds: N_u + N_p + 1 = dofs."""
    path = os.path.join(os.path.dirname(__file__), "golden", "paper_cube_dofs.txt")
    rows = [l.split()[:3] for l in open(path) if l.strip() and not l.startswith("#")]
    for NP, k, dofs in rows:
        NP, k, dofs = int(NP), int(k), int(dofs)
        n = round(NP ** (1 / 3))
        if k > 2:
            continue   # k = 3 is outside BASELINE's orders
        nkd = poly.dim_pk_3d(k - 1)
        lay = assemble.Layout(k, poly.dim_pk_2d(k), (nkd - 1) + len(poly.generators(k)), nkd,
                              3 * n * n * (n + 1), NP)
        assert lay.n_u + lay.n_p + 1 == dofs
    # and the layout formula above is what build_system uses (small meshes, assembled for real)
    for n, k, want in ((8, 2, 19585), (4, 1, None), (3, 2, None)):
        s = assemble.build_system(mesh.cube_mesh(n), k, paper_mode=True)
        nkd = poly.dim_pk_3d(k - 1)
        assert (s.layout.n_int_dof, s.layout.n_p_dof) == ((nkd - 1) + len(poly.generators(k)), nkd)
        assert s.M.shape == (s.layout.n_u, s.layout.n_u) and s.B.shape == (s.layout.n_p, s.layout.n_u)
        if want:
            assert s.n + 1 == want   # Table 4, first row (N_P = 512, k = 2): 19,585


@pytest.mark.parametrize("k", [1, 2])
def test_paper_mode_projection_and_divergence(k):
    """Unisolvence and the commuting divergence of the BDM-type local space: Pi @ D = I on
    [P_k]^3, and Div(interp(v)) = the analytic divergence of v in [P_k]^3 (which lies in P_{k-1})."""
    for name, m in _meshes():
        for cls in m.classes:
            o = local.local_operators(cls.rep(), k, k - 1)
            PD = np.einsum("eil,elj->eij", o["Pi"], o["D"])
            assert np.abs(PD - np.eye(PD.shape[1])).max() < 1e-9, (name, cls.name)
        g = m.classes[-1].rep()
        o = local.local_operators(g, k, k - 1)
        alphas = poly.multi_indices_3d(k)
        im = poly.index_map_3d(k)
        nk, nkd = len(alphas), o["nkd"]
        h = g["h"][0]
        coef = RNG.normal(size=3 * nk)
        dv = np.zeros(nk)
        for c in range(3):
            for a, al in enumerate(alphas):
                if al[c]:
                    am = list(al); am[c] -= 1
                    dv[im[tuple(am)]] += coef[c * nk + a] * al[c] / h
        assert np.abs(dv[nkd:]).max() == 0.0            # div [P_k]^3 is in P_{k-1}
        got = o["Div"][0] @ (o["D"][0] @ coef)
        assert got.shape == (nkd,)
        assert np.abs(got - dv[:nkd]).max() < 1e-9 * max(1, np.abs(dv).max()), name


@pytest.mark.parametrize("name,k", [("kuhn", 1), ("kuhn", 2), ("cube", 2), ("pairs", 1)])
def test_paper_mode_M_spd_B_full_rank(name, k):
    m = {"kuhn": lambda: mesh.kuhn_mesh(2, seed=3), "pairs": lambda: mesh.pair_mesh(4, seed=5, block=2),
         "cube": lambda: mesh.cube_mesh(3)}[name]()
    s = assemble.build_system(m, k, paper_mode=True)
    M = s.M.toarray()
    assert np.abs(M - M.T).max() <= 1e-12 * np.abs(M).max()
    np.linalg.cholesky(0.5 * (M + M.T))
    SD = (s.B @ sp.diags(1 / s.M.diagonal()) @ s.B.T).toarray()
    np.linalg.cholesky(SD)
    assert np.linalg.matrix_rank(s.B.toarray()) == s.layout.n_p


@pytest.mark.parametrize("kind,k,ns", [("cube", 1, (4, 8)), ("cube", 2, (2, 4)), ("kuhn", 1, (2, 4))])
def test_paper_mode_convergence_rates_and_conservation(kind, k, ns):
    """The paper's estimates for its own space (Remark): the pressure in P_{k-1}
    converges like h^k; local conservation B u_h = f_h holds element by element.
    (One more refinement, run once: cube k = 1 rates (e_u, e_p) = (1.99, 1.01), cube k = 2
    (3.03, 1.96), Kuhn k = 1 (1.87, 0.95): Pi^0_k u_h converges like h^{k+1}.)"""
    errs = []
    for n in ns:
        m = {"cube": lambda: mesh.cube_mesh(n), "kuhn": lambda: mesh.kuhn_mesh(n, seed=2)}[kind]()
        s = assemble.build_system(m, k, keep_local=True, paper_mode=True)
        u, p = _direct(s)
        assert np.abs(s.B @ u - s.f).max() <= 1e-10 * np.abs(s.f).max()
        errs.append(assemble.l2_errors(s, u, p))
    errs = np.array(errs)
    rates = np.log2(errs[:-1] / errs[1:])
    assert k - 0.25 <= rates[-1][1] <= k + 0.45, rates        # e_p ~ h^k
    assert rates[-1][0] >= k - 0.25, rates                    # e_u at least h^k


@pytest.mark.parametrize("k,ns", [(1, (2, 4)), (2, (2, 4))])
def test_paper_neumann_problem(k, ns):
    """The paper's own boundary value problem: Neumann data on
    the whole boundary, the mean-zero pressure enforced by one multiplier, the polynomial
    solution.  The DOF total with the multiplier is the paper's formula; B^T annihilates the
    constant pressure; the multiplier of the bordered LU solve equals its closed form
    ones.f / ones.c (zero up to rounding: the data are compatible); int p_h = 0; e_p ~ h^k and
    e_u ~ h^{k+1} for the paper's solution."""
    errs = []
    for n in ns:
        s, N = configs.paper_neumann(n, k)
        nkd = poly.dim_pk_3d(k - 1)
        want = (3 * n * n * (n + 1) * poly.dim_pk_2d(k)
                + n ** 3 * ((nkd - 1) + len(poly.generators(k)) + nkd) + 1)
        assert s.n + 1 == want == N.bordered().shape[0]
        assert np.abs(N.B.T @ N.ones).max() <= 1e-13 * abs(N.B).max()
        x = spl.spsolve(N.bordered().tocsc(), N.bordered_rhs())
        nu = s.layout.n_u
        u, p, lam = x[:nu], x[nu:-1], x[-1]
        scale = np.abs(N.f).max() / np.abs(N.c).max()
        assert abs(lam - N.lam) <= 1e-10 * scale and abs(N.lam) <= 1e-10 * scale
        assert abs(N.c @ p) <= 1e-12 * np.abs(N.c).sum() * np.abs(p).max()
        assert np.abs(u[N.boundary_dofs] - N.u_boundary).max() <= 1e-12 * np.abs(N.u_boundary).max()
        # errors against the exact pair (p with its mean removed)
        old = assemble.exact_u, assemble.exact_p
        assemble.exact_u = lambda pts, K=None: assemble.paper_exact_u(pts)
        assemble.exact_p = lambda pts: assemble.paper_exact_p(pts) - assemble.PAPER_P_MEAN
        try:
            errs.append(assemble.l2_errors(s, u, p))
        finally:
            assemble.exact_u, assemble.exact_p = old
    errs = np.array(errs)
    rates = np.log2(errs[:-1] / errs[1:])
    assert k - 0.25 <= rates[-1][1] <= k + 0.45, rates
    assert rates[-1][0] >= k + 1 - 0.25, rates
