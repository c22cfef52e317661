"""Local RT-type mixed VEM operators, batched over cells.

PAPER.md §4 with the order convention of DESIGN.md reading R1
(face moments in P_k(f), gradient moments over M_k \\ M_0, cross moments over
M^{G,+}_{k-1}, divergence and pressure in P_k).  Local DOF vector
    chi = [ face moments, face by face (n_f each) | gradient moments | cross moments ]
with the paper's scalings 1/|f| (eqn:facePoly), h_P/|P| (eqn:gradMom,
P:632) and 1/|P| (eqn:crossMom).  Face moments use the face's global
normal, so a face DOF is single-valued across the two cells sharing it.

Every array carries a leading batch axis E.
"""
from __future__ import annotations

import numpy as np

from . import poly
from .quad import box_rule, parallelogram_rule, tet_rule, triangle_rule


def volume_rule(g: dict, q: int):
    if g["vol_kind"] == "boxes":
        lo, hi = g["box_lo"], g["box_hi"]
        E, nb = lo.shape[:2]
        pts, w = box_rule(lo.reshape(-1, 3), hi.reshape(-1, 3), q)
        return pts.reshape(E, -1, 3), w.reshape(E, -1)
    tv = g["tet_verts"]
    return tet_rule(tv[:, 0], tv[:, 1], tv[:, 2], tv[:, 3], q)


def face_rule(f, q: int):
    if f.kind == "para":
        return parallelogram_rule(f.v0, f.v1, f.v2, q)
    return triangle_rule(f.v0, f.v1, f.v2, q)


def face_coords(f, pts):
    """Scaled face-local coordinates ((x - x_f).e1, (x - x_f).e2)/h_f."""
    d = pts - f.centroid[:, None, :]
    return np.stack([np.einsum("eqd,ed->eq", d, f.e1), np.einsum("eqd,ed->eq", d, f.e2)],
                    axis=-1) / f.h[:, None, None]


def local_operators(g: dict, k: int, kd: int | None = None) -> dict:
    """kd = order of the divergence / pressure space: k (RT-type, reading R1, the default) or
    k - 1 (the paper's own BDM-type space: gradient moments over M_{k-1} \\ M_0, div v and
    pressure in P_{k-1}; SURVEY.md N3 "paper mode").

    Compute, for the batch of cells described by g (see CellClass.rep):
      Hp    (E, n_k, n_k)     int_P m_a m_b                       (monomial mass)
      Div   (E, n_k, n_loc)   chi -> coefficients of div v in M_k
      Pi    (E, 3 n_k, n_loc) chi -> coefficients of Pi^0_k v in [M_k]^3
      D     (E, n_loc, 3 n_k) dof_i(m_j) for vector monomials m_j
      A     (E, 3, n_loc, n_loc) consistency per component: Pi_c^T Hp Pi_c
      S     (E, n_loc, n_loc) (I - D Pi)^T (I - D Pi)  (stabilisation)
    """
    alphas = poly.multi_indices_3d(k)
    alphas1 = poly.multi_indices_3d(k + 1)
    idx1 = poly.index_map_3d(k + 1)
    betas = poly.multi_indices_2d(k)
    nk, nk1, nf = len(alphas), len(alphas1), len(betas)
    kd = k if kd is None else kd
    assert kd in (k, k - 1) and kd >= 0
    nkd = poly.dim_pk_3d(kd)          # graded-lex order: the first nkd monomials span P_kd
    gens = poly.generators(k)
    gen_idx = {gg: i for i, gg in enumerate(gens)}
    nF = len(g["faces"])
    ngrad = nkd - 1
    ncross = len(gens)
    nloc = nF * nf + ngrad + ncross
    off_grad = nF * nf
    off_cross = off_grad + ngrad

    xP, hP, vol = g["centroid"], g["h"], g["vol"]
    E = xP.shape[0]
    q = 2 * k + 2
    pts, w = volume_rule(g, q)
    s = (pts - xP[:, None, :]) / hP[:, None, None]
    mv = poly.eval_monomials_3d(s, k + 1)          # (E, nq, nk1)
    Hp = np.einsum("eq,eqa,eqb->eab", w, mv[..., :nk], mv[..., :nk])
    Hk_k1 = np.einsum("eq,eqa,eqb->eab", w, mv[..., :nk], mv)   # (E, nk, nk1)

    # boundary flux rows: Bnd[b] . chi = sum_f sigma_f int_f (v.n_f) m_b, b in M_{k+1}
    Bnd = np.zeros((E, nk1, nloc))
    facedata = []
    for lf, f in enumerate(g["faces"]):
        fp, fw = face_rule(f, q)
        if fp.shape[0] != E:       # congruent faces shared by batch (E == 1 anyway)
            fp, fw = np.broadcast_to(fp, (E,) + fp.shape[1:]), np.broadcast_to(fw, (E,) + fw.shape[1:])
        t = face_coords(f, fp) if f.centroid.shape[0] == E else face_coords(
            _bcast_face(f, E), fp)
        mf = poly.eval_monomials_2d(t, k)                          # (E, nqf, nf)
        Hf = np.einsum("eq,eqa,eqb->eab", fw, mf, mf)
        area = np.broadcast_to(f.area, (E,))
        CF = area[:, None, None] * np.linalg.inv(Hf)               # chi_f -> c^f
        m3 = poly.eval_monomials_3d((fp - xP[:, None, :]) / hP[:, None, None], k + 1)
        Phi = np.einsum("eq,eqa,eqb->eab", fw, mf, m3)             # (E, nf, nk1)
        sig = g["face_signs"][:, lf].astype(np.float64)
        Bnd[:, :, lf * nf:(lf + 1) * nf] += sig[:, None, None] * np.einsum("eab,eac->ebc", Phi, CF)
        facedata.append((fp, fw, mf, np.broadcast_to(f.normal, (E, 3)), area))

    # divergence in P_kd: Hp d = r, r_a = -[a != 0] (|P|/h_P) chi^grad_a + Bnd[a], a in M_kd
    r = Bnd[:, :nkd, :].copy()
    for a in range(1, nkd):
        r[:, a, off_grad + a - 1] -= vol / hP
    Div = np.linalg.solve(Hp[:, :nkd, :nkd], r)

    # G[b] . chi = int_P v . grad m_b, b in M_{k+1}, |b| >= 1
    G = np.zeros((E, nk1, nloc))
    for b, beta in enumerate(alphas1):
        if sum(beta) == 0:
            continue
        if sum(beta) <= kd:
            G[:, b, off_grad + b - 1] = vol / hP
        else:   # by parts with div v in P_kd
            G[:, b] = -np.einsum("ea,eal->el", Hk_k1[:, :nkd, b], Div) + Bnd[:, b]

    # R rows: int_P v . (e_c m_a) via Props 1-3 and Prop. inTermsOfGPerpBasis
    R = np.zeros((E, 3 * nk, nloc))
    for c in range(3):
        for a, alpha in enumerate(alphas):
            gc, beta, cross = poly.decompose_vector_monomial(c, alpha)
            row = c * nk + a
            R[:, row] += (gc * hP)[:, None] * G[:, idx1[beta]]
            for coef, cc, al in cross:
                for coef2, c2, al2 in poly.cross_term_as_generators(cc, al):
                    R[:, row, off_cross + gen_idx[(c2, al2)]] += coef * coef2 * vol
    Pi = np.concatenate([np.linalg.solve(Hp, R[:, c * nk:(c + 1) * nk]) for c in range(3)], axis=1)

    # D: dofs of the vector monomials e_c m_j
    D = np.zeros((E, nloc, 3 * nk))
    for lf, (fp, fw, mf, nrm, area) in enumerate(facedata):
        m3 = poly.eval_monomials_3d((fp - xP[:, None, :]) / hP[:, None, None], k)
        base = np.einsum("eq,eqb,eqj->ebj", fw, mf, m3) / area[:, None, None]
        for c in range(3):
            D[:, lf * nf:(lf + 1) * nf, c * nk:(c + 1) * nk] = nrm[:, c, None, None] * base
    imap = poly.index_map_3d(k)
    mvk = mv[..., :nk]
    for a in range(1, nkd):
        alpha = alphas[a]
        for c in range(3):
            if alpha[c] == 0:
                continue
            am = list(alpha)
            am[c] -= 1
            # (h_P/|P|) int m_j d_c m_a = (1/|P|) a_c int m_j m_{a - e_c}
            D[:, off_grad + a - 1, c * nk:(c + 1) * nk] = alpha[c] * Hp[:, :, imap[tuple(am)]] / vol[:, None]
    for gi, (c2, al) in enumerate(gens):
        e = np.zeros(3)
        e[c2] = 1.0
        field = np.cross(s, e) * mv[..., imap[al]][..., None]          # (E, nq, 3)
        for c in range(3):
            D[:, off_cross + gi, c * nk:(c + 1) * nk] = np.einsum(
                "eq,eqj,eq->ej", w, mvk, field[..., c]) / vol[:, None]

    A = np.stack([np.einsum("eai,eab,ebj->eij", Pi[:, c * nk:(c + 1) * nk], Hp,
                            Pi[:, c * nk:(c + 1) * nk]) for c in range(3)], axis=1)
    IDP = np.eye(nloc)[None] - np.einsum("eij,ejl->eil", D, Pi)
    S = np.einsum("eki,ekj->eij", IDP, IDP)
    return dict(Hp=Hp, Div=Div, Pi=Pi, D=D, A=A, S=S, nloc=nloc, nk=nk, nkd=nkd, nf=nf,
                n_int=ngrad + ncross, vol=vol, h=hP)


def _bcast_face(f, E):
    from .mesh import FaceGeom
    return FaceGeom(f.kind, *(np.broadcast_to(getattr(f, a), (E,) + getattr(f, a).shape[1:])
                              for a in ("v0", "v1", "v2", "normal", "e1", "e2", "centroid", "area", "h")))
