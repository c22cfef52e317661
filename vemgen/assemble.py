"""Global assembly of the mixed-VEM saddle-point system.

    [ M  B^T ] [u]   [g]
    [ B   0  ] [p] = [f]

* M  = sum_P a_{h,P}: consistency nu int Pi v . Pi w plus the dofi-dofi
  stabilisation s_P = nu(x_P)|P| sum dof_i dof_i, with
  nu = K^{-1} (reading R4); for a diagonal tensor K the consistency is
  componentwise and s_P = |P| tr(K^{-1})/3.
* B  = -|P| DivMatrix per cell, pressure unknowns = moments (readings R6, R7):
  row alpha of B u = f states div u_h = Pi^0_k f on every cell (P:58,
  P:805-820).
* g  = -sum_{f in boundary} sigma_f int_f g_D v.n_f (pressure Dirichlet data,
  reading R5); f_P = -|P| Hp^{-1} (int_P f m_a)_a.

Global numbering (O5): face DOF  face*n_f + beta,
                       interior  N_F*n_f + cell*n_i + i,
                       pressure  cell*n_p + alpha.
Local matrix entries |a| <= 1e-14 max|template| are dropped before assembly
(reading R11).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import poly
from .local import local_operators, volume_rule
from .quad import gauss_legendre_01, tet_rule, triangle_rule, parallelogram_rule

DROP_TOL = 1e-14


@dataclass
class Layout:
    k: int
    n_face_dof: int
    n_int_dof: int
    n_p_dof: int
    n_faces: int
    n_elems: int

    @property
    def n_u(self) -> int:
        return self.n_faces * self.n_face_dof + self.n_elems * self.n_int_dof

    @property
    def n_p(self) -> int:
        return self.n_elems * self.n_p_dof


@dataclass
class System:
    M: sp.csr_matrix
    B: sp.csr_matrix
    g: np.ndarray
    f: np.ndarray
    layout: Layout
    mesh: object
    k: int
    local: list = field(default_factory=list)  # per class: (class, ops)

    @property
    def rhs(self) -> np.ndarray:
        return np.concatenate([self.g, self.f])

    @property
    def n(self) -> int:
        return self.layout.n_u + self.layout.n_p


def _drop(T):
    T = np.array(T, copy=True)
    mx = np.abs(T).reshape(T.shape[0], -1).max(axis=1)
    T[np.abs(T) <= DROP_TOL * mx.reshape((-1,) + (1,) * (T.ndim - 1))] = 0.0
    return T


def sin_source(x):
    """f = 3 pi^2 prod sin(pi x_d): the source of p = prod sin(pi x_d), K = I."""
    return 3 * np.pi ** 2 * np.prod(np.sin(np.pi * x), axis=-1)


def exact_p(x):
    return np.prod(np.sin(np.pi * x), axis=-1)


def exact_u(x, K=None):
    """u = -K grad p (reading R4); K diagonal (3,) or None."""
    s, c = np.sin(np.pi * x), np.cos(np.pi * x)
    gp = np.pi * np.stack([c[..., 0] * s[..., 1] * s[..., 2], s[..., 0] * c[..., 1] * s[..., 2],
                           s[..., 0] * s[..., 1] * c[..., 2]], axis=-1)
    return -gp if K is None else -gp * K


def _box_source_moments(lo, hi, xP, hP, k, nq=16):
    """int over the union of boxes of f m_a for f = 3pi^2 prod sin(pi x_d),
    separable in 1D (lo, hi (E, nb, 3)) -> (E, n_k)."""
    x, w = gauss_legendre_01(nq)
    E, nb = lo.shape[:2]
    alphas = poly.multi_indices_3d(k)
    out = np.zeros((E, len(alphas)))
    for b in range(nb):
        I = []
        for d in range(3):
            a, bb = lo[:, b, d], hi[:, b, d]
            pts = a[:, None] + x[None, :] * (bb - a)[:, None]
            ww = w[None, :] * (bb - a)[:, None]
            t = (pts - xP[:, d, None]) / hP[:, None]
            base = ww * np.sin(np.pi * pts)
            I.append(np.stack([(base * t ** p).sum(1) for p in range(k + 1)], 1))
        for i, (a1, a2, a3) in enumerate(alphas):
            out[:, i] += I[0][:, a1] * I[1][:, a2] * I[2][:, a3]
    return 3 * np.pi ** 2 * out


def source_moments(cls, k, source=None, chunk=200000):
    """F (E, n_k) = int_P f m_a for every cell of the class."""
    if source is None and cls.vol_kind == "boxes":
        return _box_source_moments(cls.box_lo, cls.box_hi, cls.centroid, cls.h, k)
    src = source or sin_source
    out = []
    E = cls.centroid.shape[0]
    for s0 in range(0, E, chunk):
        sl = slice(s0, min(E, s0 + chunk))
        g = dict(vol_kind=cls.vol_kind)
        if cls.vol_kind == "boxes":
            g["box_lo"], g["box_hi"] = cls.box_lo[sl], cls.box_hi[sl]
        else:
            g["tet_verts"] = cls.tet_verts[sl]
        pts, w = volume_rule(g, 2 * k + 8)
        m = poly.eval_monomials_3d((pts - cls.centroid[sl, None, :]) / cls.h[sl, None, None], k)
        out.append(np.einsum("eq,eq,eqa->ea", w, src(pts), m))
    return np.concatenate(out, axis=0)


def boundary_term(mesh, k, gD):
    """g_(f,beta) = -sigma_f sum_gamma CF[gamma, beta] int_f g_D m^f_gamma on
    boundary faces (natural pressure BC).  Returns (dof ids, values)."""
    fg = mesh.boundary_geom
    nf = poly.dim_pk_2d(k)
    q = 2 * k + 8
    if fg.kind == "para":
        fp, fw = parallelogram_rule(fg.v0, fg.v1, fg.v2, q)
    else:
        fp, fw = triangle_rule(fg.v0, fg.v1, fg.v2, q)
    from .local import face_coords
    mf = poly.eval_monomials_2d(face_coords(fg, fp), k)
    Hf = np.einsum("eq,eqa,eqb->eab", fw, mf, mf)
    CF = fg.area[:, None, None] * np.linalg.inv(Hf)
    G = np.einsum("eq,eq,eqa->ea", fw, gD(fp), mf)
    val = -mesh.boundary_sign[:, None] * np.einsum("eab,ea->eb", CF, G)
    dofs = mesh.boundary_faces[:, None] * nf + np.arange(nf)[None, :]
    return dofs.reshape(-1), val.reshape(-1)


def class_template(mesh, cls, ops, k: int, source=None) -> dict:
    """Shape cache of one congruent cell class (the host half of the element-parallel
    GPU assembly, vem_mixed_assemble): local DOF maps, the K-independent local
    templates after the R11 drop, their nonzero pattern (ii, jj) / (bi, bj) and the
    per-cell coefficients, such that cell e contributes
        M_e[ii, jj] = ((c_e0 A0 + c_e1 A1) + c_e2 A2) + c_e3 S,   c_e = (1/K_e0, 1/K_e1, 1/K_e2, s_P)
        B_e[bi, bj] = Bt[bi, bj]
        f_e = -|P| Hinv F_e."""
    nf = poly.dim_pk_2d(k)
    nk = ops["nkd"]                      # pressure / divergence space P_kd (kd = k, or k - 1 in paper mode)
    n_int = (nk - 1) + poly.dim_gperp(k)
    E = cls.cell_ids.shape[0]
    fd = (cls.face_ids[:, :, None] * nf + np.arange(nf)[None, None, :]).reshape(E, -1)
    idofs = mesh.n_faces * nf + cls.cell_ids[:, None] * n_int + np.arange(n_int)[None, :]
    L = np.concatenate([fd, idofs], axis=1)
    assert L.shape[1] == ops["nloc"]
    P = cls.cell_ids[:, None] * nk + np.arange(nk)[None, :]
    Kc = mesh.K[cls.cell_ids]
    invK = 1.0 / Kc
    sP = cls.vol * invK.mean(axis=1)
    A = np.stack([_drop(ops["A"][:, c]) for c in range(3)], axis=1)
    S = _drop(ops["S"])
    Bt = _drop(-ops["vol"][:, None, None] * ops["Div"])
    mask = (A[0] != 0).any(axis=0) | (S[0] != 0)
    ii, jj = np.nonzero(mask)
    bi, bj = np.nonzero(Bt[0])
    F = source_moments(cls, k, source)[:, :nk]
    Hinv = np.linalg.inv(ops["Hp"][:, :nk, :nk])
    return dict(L=L, P=P, ii=ii, jj=jj, A=np.stack([A[0, c][ii, jj] for c in range(3)]), S=S[0][ii, jj],
                coef=np.concatenate([invK, sP[:, None]], axis=1), bi=bi, bj=bj, B=Bt[0][bi, bj],
                F=F, Hinv=np.broadcast_to(Hinv, (E, nk, nk))[0], vol=cls.vol)


def tet_class_input(mesh, cls, k: int, source=None) -> dict:
    """Per-cell input of the device computation of the local operators for a class of
    single tetrahedra (Kuhn meshes, C2; vem_mixed_assemble_tets): geometry, the
    reference quadrature rules, the symbolic tables of Props. 1-3 / P:478-490 and the
    generator basis, DOF maps, per-cell coefficients and source moments.  The local
    matrices themselves (the batched small dense Pi / Div solves of local_operators)
    are then computed on the device, one thread per cell."""
    assert cls.vol_kind == "tet" and not cls.congruent and cls.n_faces == 4
    nf = poly.dim_pk_2d(k)
    nk = poly.dim_pk_3d(k)
    n_int = (nk - 1) + poly.dim_gperp(k)
    E = cls.cell_ids.shape[0]
    fd = (cls.face_ids[:, :, None] * nf + np.arange(nf)[None, None, :]).reshape(E, -1)
    idofs = mesh.n_faces * nf + cls.cell_ids[:, None] * n_int + np.arange(n_int)[None, :]
    L = np.concatenate([fd, idofs], axis=1)
    P = cls.cell_ids[:, None] * nk + np.arange(nk)[None, :]
    invK = 1.0 / mesh.K[cls.cell_ids]
    sP = cls.vol * invK.mean(axis=1)
    # faces: v0, v1, v2, normal, e1, e2, centroid (3 each), area, h
    fg = np.zeros((E, 4, 23))
    for lf, f in enumerate(cls.faces):
        fg[:, lf, :] = np.concatenate([f.v0, f.v1, f.v2, f.normal, f.e1, f.e2, f.centroid,
                                       f.area[:, None], f.h[:, None]], axis=1)
    cell = np.concatenate([cls.centroid, cls.h[:, None], cls.vol[:, None], cls.tet_verts.reshape(E, 12)], axis=1)
    # reference rules (the same collapsed Gauss-Legendre rules as quad.tet_rule / triangle_rule)
    from .quad import gauss_legendre_01, npts_for_degree
    q = 2 * k + 2
    n3 = npts_for_degree(q, 2)
    x, w = gauss_legendre_01(n3)
    U, V, Wc = (a.reshape(-1) for a in np.meshgrid(x, x, x, indexing="ij"))
    Wt = (w[:, None, None] * w[None, :, None] * w[None, None, :]).reshape(-1) * (1.0 - U) ** 2 * (1.0 - V)
    vref = np.stack([U, (1.0 - U) * V, (1.0 - U) * (1.0 - V) * Wc, Wt], axis=1)
    n2 = npts_for_degree(q, 1)
    x2, w2 = gauss_legendre_01(n2)
    U2, V2 = (a.reshape(-1) for a in np.meshgrid(x2, x2, indexing="ij"))
    W2 = (w2[:, None] * w2[None, :]).reshape(-1) * (1.0 - U2)
    fref = np.stack([U2, (1.0 - U2) * V2, W2], axis=1)
    # symbolic tables
    alphas = poly.multi_indices_3d(k)
    alphas1 = poly.multi_indices_3d(k + 1)
    idx1 = poly.index_map_3d(k + 1)
    imap = poly.index_map_3d(k)
    gens = poly.generators(k)
    gen_idx = {gg: i for i, gg in enumerate(gens)}
    rgrad = np.zeros((3 * nk, 2))                   # (gc, index of beta in M_{k+1}) per R row
    rcross = np.zeros((3 * nk, 4, 2))               # up to 4 (generator, coef) per R row; generator -1 = none
    rcross[..., 0] = -1
    for c in range(3):
        for a, alpha in enumerate(alphas):
            gc, beta, cross = poly.decompose_vector_monomial(c, alpha)
            rgrad[c * nk + a] = (gc, idx1[beta])
            terms = {}
            for coef, cc, al in cross:
                for coef2, c2, al2 in poly.cross_term_as_generators(cc, al):
                    g = gen_idx[(c2, al2)]
                    terms[g] = terms.get(g, 0.0) + coef * coef2
            assert len(terms) <= 4
            for t, (g, v) in enumerate(sorted(terms.items())):
                rcross[c * nk + a, t] = (g, v)
    dgrad = np.full((max(nk - 1, 1), 3, 2), -1.0)   # per gradient DOF a >= 1, component c: (alpha_c, imap[a - e_c])
    for a in range(1, nk):
        for c in range(3):
            if alphas[a][c] > 0:
                am = list(alphas[a])
                am[c] -= 1
                dgrad[a - 1, c] = (alphas[a][c], imap[tuple(am)])
    gtab = np.array([(c2, imap[al]) for c2, al in gens], dtype=np.float64).reshape(-1, 2)
    return dict(k=k, L=L, P=P, coef=np.concatenate([invK, sP[:, None]], axis=1), cell=cell, faces=fg,
                signs=cls.face_signs.astype(np.float64), F=source_moments(cls, k, source), vref=vref, fref=fref,
                alphas1=np.array(alphas1, dtype=np.float64), betas=np.array(poly.multi_indices_2d(k), dtype=np.float64),
                rgrad=rgrad, rcross=rcross, dgrad=dgrad, gens=gtab)


def class_templates(mesh, k: int, source=None) -> list:
    """Shape caches of every cell class (the input of vem_mixed_assemble); all
    classes must be congruent (cube grids, cube pairs).  Kuhn tetrahedra (C2) are
    not: every cell has its own local matrices, assembled on the host."""
    out = []
    for cls in mesh.classes:
        if not cls.congruent:
            raise ValueError("device assembly needs congruent cell classes (cubes, cube pairs)")
        out.append(class_template(mesh, cls, local_operators(cls.rep(), k), k, source))
    return out


def build_system(mesh, k: int, source=None, gD=None, keep_local=False, paper_mode=False) -> System:
    """Assemble M, B, g, f for mesh at order k (RT-type, reading R1).  paper_mode: the
    paper's own BDM-type space (gradient moments over M_{k-1} \\ M_0, divergence and pressure
    in P_{k-1}, k >= 1) with this build's pressure-Dirichlet
    boundary condition (R5): the paper's DOF total minus its mean-value multiplier."""
    nf = poly.dim_pk_2d(k)
    kd = k - 1 if paper_mode else k
    if kd < 0:
        raise ValueError("paper mode needs k >= 1")
    nk = poly.dim_pk_3d(kd)
    n_int = (nk - 1) + poly.dim_gperp(k)
    lay = Layout(k, nf, n_int, nk, mesh.n_faces, mesh.n_cells)
    Nu, Np = lay.n_u, lay.n_p
    mr, mc, mv, br, bc, bv = [], [], [], [], [], []
    f = np.zeros(Np)
    local_keep = []
    for cls in mesh.classes:
        E = cls.cell_ids.shape[0]
        ops = local_operators(cls.rep(), k, kd)
        if cls.congruent:
            t = class_template(mesh, cls, ops, k, source)
            L, P, ii, jj, bi, bj = t["L"], t["P"], t["ii"], t["jj"], t["bi"], t["bj"]
            c = t["coef"]
            vals = (c[:, 0, None] * t["A"][0] + c[:, 1, None] * t["A"][1] + c[:, 2, None] * t["A"][2]
                    + c[:, 3, None] * t["S"])
            mr.append(L[:, ii].reshape(-1)); mc.append(L[:, jj].reshape(-1)); mv.append(vals.reshape(-1))
            br.append(P[:, bi].reshape(-1)); bc.append(L[:, bj].reshape(-1))
            bv.append(np.broadcast_to(t["B"], (E, bi.size)).reshape(-1))
            fP = -cls.vol[:, None] * np.einsum("ab,eb->ea", t["Hinv"], t["F"])
        else:
            nloc = ops["nloc"]
            fd = (cls.face_ids[:, :, None] * nf + np.arange(nf)[None, None, :]).reshape(E, -1)
            idofs = mesh.n_faces * nf + cls.cell_ids[:, None] * n_int + np.arange(n_int)[None, :]
            L = np.concatenate([fd, idofs], axis=1)
            assert L.shape[1] == nloc
            P = cls.cell_ids[:, None] * nk + np.arange(nk)[None, :]
            invK = 1.0 / mesh.K[cls.cell_ids]
            sP = cls.vol * invK.mean(axis=1)
            A = np.stack([_drop(ops["A"][:, c]) for c in range(3)], axis=1)
            S = _drop(ops["S"])
            Bt = _drop(-ops["vol"][:, None, None] * ops["Div"])
            Ml = np.einsum("ec,ecij->eij", invK, A) + sP[:, None, None] * S
            nz = Ml != 0
            mr.append(np.broadcast_to(L[:, :, None], Ml.shape)[nz])
            mc.append(np.broadcast_to(L[:, None, :], Ml.shape)[nz])
            mv.append(Ml[nz])
            nzb = Bt != 0
            br.append(np.broadcast_to(P[:, :, None], Bt.shape)[nzb])
            bc.append(np.broadcast_to(L[:, None, :], Bt.shape)[nzb])
            bv.append(Bt[nzb])
            F = source_moments(cls, k, source)[:, :nk]
            Hinv = np.linalg.inv(ops["Hp"][:, :nk, :nk])
            fP = -cls.vol[:, None] * np.einsum("eab,eb->ea", np.broadcast_to(Hinv, (E, nk, nk)), F)
        f[P.reshape(-1)] = fP.reshape(-1)
        if keep_local:
            local_keep.append((cls, ops, L, P))
    M = _to_csr(np.concatenate(mr), np.concatenate(mc), np.concatenate(mv), Nu, Nu)
    B = _to_csr(np.concatenate(br), np.concatenate(bc), np.concatenate(bv), Np, Nu)
    g = np.zeros(Nu)
    if gD is not None:
        dofs, vals = boundary_term(mesh, k, gD)
        np.add.at(g, dofs, vals)
    return System(M, B, g, f, lay, mesh, k, local_keep)


def _to_csr(r, c, v, nr, nc):
    A = sp.coo_matrix((v, (r.astype(np.int64), c.astype(np.int64))), shape=(nr, nc)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A


def pressure_coeffs(system: System, p_mom: np.ndarray):
    """Monomial coefficients of p_h from moment unknowns: q = |P| Hp^{-1} mu."""
    out = []
    for cls, ops, L, P in system.local:
        E = cls.cell_ids.shape[0]
        nkd = ops["nkd"]
        Hinv = np.broadcast_to(np.linalg.inv(ops["Hp"][:, :nkd, :nkd]), (E, nkd, nkd))
        out.append((cls, cls.vol[:, None] * np.einsum("eab,eb->ea", Hinv, p_mom[P])))
    return out


def l2_errors(system: System, u: np.ndarray, p: np.ndarray, K=None):
    """Relative errors e_u = ||u - Pi^0_k u_h|| / ||u||, e_p = ||p - p_h|| / ||p||
    (with Pi^0_k u_h for the velocity)."""
    k = system.k
    nk = poly.dim_pk_3d(k)
    eu2 = nu2 = ep2 = np2 = 0.0
    for cls, ops, L, P in system.local:
        E = cls.cell_ids.shape[0]
        g = dict(vol_kind=cls.vol_kind)
        if cls.vol_kind == "boxes":
            g["box_lo"], g["box_hi"] = cls.box_lo, cls.box_hi
        else:
            g["tet_verts"] = cls.tet_verts
        pts, w = volume_rule(g, 2 * k + 8)
        m = poly.eval_monomials_3d((pts - cls.centroid[:, None, :]) / cls.h[:, None, None], k)
        Pi = np.broadcast_to(ops["Pi"], (E,) + ops["Pi"].shape[1:])
        cu = np.einsum("eil,el->ei", Pi, u[L])                     # (E, 3 nk)
        uh = np.stack([np.einsum("eqa,ea->eq", m, cu[:, c * nk:(c + 1) * nk]) for c in range(3)], -1)
        nkd = ops["nkd"]
        Hinv = np.broadcast_to(np.linalg.inv(ops["Hp"][:, :nkd, :nkd]), (E, nkd, nkd))
        cp = cls.vol[:, None] * np.einsum("eab,eb->ea", Hinv, p[P])
        ph = np.einsum("eqa,ea->eq", m[..., :nkd], cp)
        ue = exact_u(pts, K)
        pe = exact_p(pts)
        eu2 += float(np.einsum("eq,eqd->", w, (ue - uh) ** 2))
        nu2 += float(np.einsum("eq,eqd->", w, ue ** 2))
        ep2 += float(np.einsum("eq,eq->", w, (pe - ph) ** 2))
        np2 += float(np.einsum("eq,eq->", w, pe ** 2))
    return np.sqrt(eu2 / nu2), np.sqrt(ep2 / np2)


# ---------------------------------------------------------------------------
# The paper's own boundary value problem: Neumann data u.n = u_N on the whole
# boundary and the mean-zero pressure enforced by one multiplier (PAPER.md P:562-566,
# P:764-765), with the paper's polynomial solution
# ---------------------------------------------------------------------------
def paper_exact_p(x):
    """q = x^5 + 6 y^4 + 9 z^3 + x y^2 z^3, before the mean is removed."""
    X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
    return X ** 5 + 6 * Y ** 4 + 9 * Z ** 3 + X * Y ** 2 * Z ** 3


PAPER_P_MEAN = 1.0 / 6 + 6.0 / 5 + 9.0 / 4 + (1.0 / 2) * (1.0 / 3) * (1.0 / 4)   # int over [0,1]^3


def paper_exact_u(x):
    """v = -grad q = (-5x^4 - y^2 z^3, -24 y^3 - 2 x y z^3, -27 z^2 - 3 x y^2 z^2) (nu = 1)."""
    X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
    return np.stack([-5 * X ** 4 - Y ** 2 * Z ** 3, -24 * Y ** 3 - 2 * X * Y * Z ** 3,
                     -27 * Z ** 2 - 3 * X * Y ** 2 * Z ** 2], axis=-1)


def paper_source(x):
    """f = div v = -20 x^3 - 72 y^2 - 2 x z^3 - 54 z - 6 x y^2 z."""
    X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
    return -20 * X ** 3 - 72 * Y ** 2 - 2 * X * Z ** 3 - 54 * Z - 6 * X * Y ** 2 * Z


@dataclass
class NeumannSystem:
    """The bordered system of the paper's problem,
        [ M   B^T  0 ] [u]        [g]
        [ B   0    c ] [p]      = [f]          c_i = int q_i  (mean-value functional),
        [ 0   c^T  0 ] [lambda]   [0]
    after the boundary face DOFs were set to the data (their rows of M are diag(M), their columns
    of M and B moved to the right-hand side).  `ones` holds the moments of the constant pressure 1
    (B^T ones = 0: the pressure is determined up to it, which the multiplier row removes)."""
    M: sp.csr_matrix
    B: sp.csr_matrix
    g: np.ndarray
    f: np.ndarray
    c: np.ndarray
    ones: np.ndarray
    layout: Layout
    boundary_dofs: np.ndarray
    u_boundary: np.ndarray

    @property
    def lam(self) -> float:
        """The multiplier in closed form: ones^T (B u + c lambda) = ones^T f and B^T ones = 0."""
        return float(self.ones @ self.f) / float(self.ones @ self.c)

    @property
    def rhs(self) -> np.ndarray:
        """Right-hand side of the consistent singular saddle system [M B^T; B 0][u; p] = [g; f - c lambda]
        that goes through the C ABI; project() then picks the mean-zero pressure."""
        return np.concatenate([self.g, self.f - self.lam * self.c])

    def project(self, p: np.ndarray) -> np.ndarray:
        """The pressure of the bordered system: p - (c.p / c.ones) ones."""
        return p - (self.c @ p) / (self.c @ self.ones) * self.ones

    def bordered(self) -> sp.csr_matrix:
        c = sp.csr_matrix(self.c.reshape(-1, 1))
        return sp.bmat([[self.M, self.B.T, None], [self.B, None, c], [None, c.T, None]]).tocsr()

    def bordered_rhs(self) -> np.ndarray:
        return np.concatenate([self.g, self.f, [0.0]])


def neumann_system(system: System, u_exact) -> NeumannSystem:
    """Impose u.n = u_exact.n on every boundary face of `system` (assembled with keep_local=True)
    and add the mean-value multiplier data."""
    mesh, k = system.mesh, system.k
    nf = poly.dim_pk_2d(k)
    fg = mesh.boundary_geom
    q = 2 * k + 8
    if fg.kind == "para":
        fp, fw = parallelogram_rule(fg.v0, fg.v1, fg.v2, q)
    else:
        fp, fw = triangle_rule(fg.v0, fg.v1, fg.v2, q)
    from .local import face_coords
    mf = poly.eval_monomials_2d(face_coords(fg, fp), k)
    un = np.einsum("eqd,ed->eq", u_exact(fp), fg.normal)            # u . n_f (global face normal)
    uB = (np.einsum("eq,eq,eqa->ea", fw, un, mf) / fg.area[:, None]).reshape(-1)   # face moments
    bd = (mesh.boundary_faces[:, None] * nf + np.arange(nf)[None, :]).reshape(-1)
    nu = system.layout.n_u
    xb = np.zeros(nu)
    xb[bd] = uB
    g = system.g - system.M @ xb
    f = system.f - system.B @ xb
    keep = np.ones(nu)
    keep[bd] = 0.0
    Dk = sp.diags(keep)
    dM = system.M.diagonal()
    M = (Dk @ system.M @ Dk + sp.diags((1 - keep) * dM)).tocsr()
    B = (system.B @ Dk).tocsr()
    for A_ in (M, B):      # the C ABI wants sorted, duplicate-free rows
        A_.eliminate_zeros()
        A_.sum_duplicates()
        A_.sort_indices()
    g[bd] = dM[bd] * uB
    # mean-value functional and the constant pressure in moment unknowns
    c = np.zeros(system.layout.n_p)
    ones = np.zeros(system.layout.n_p)
    for cls, ops, L, P in system.local:
        nkd = ops["nkd"]
        E = cls.cell_ids.shape[0]
        Hp = np.broadcast_to(ops["Hp"], (E,) + ops["Hp"].shape[1:])
        c[P[:, 0]] = cls.vol                                     # int q = |P| * (mean moment)
        ones[P.reshape(-1)] = (Hp[:, 0, :nkd] / cls.vol[:, None]).reshape(-1)   # (1/|P|) int m_a
    return NeumannSystem(M, B, g, f, c, ones, system.layout, bd, uB)
