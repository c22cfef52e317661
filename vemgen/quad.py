"""Quadrature rules used by the assembler (reading R10).

PAPER.md only says the discrete forms reduce to "the computation of integrals"
(P:799-802).  We use Gauss-Legendre products: tensor rules on boxes and
rectangles, collapsed (Duffy / conical-product) rules on tetrahedra and
triangles.  All rules are exact for polynomials of the requested degree.
"""
from __future__ import annotations

import numpy as np


def gauss_legendre_01(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def npts_for_degree(q: int, extra: int = 0) -> int:
    """Points per direction so that degree q + extra is integrated exactly."""
    return max(1, (q + extra + 2) // 2)


def box_rule(lo: np.ndarray, hi: np.ndarray, q: int):
    """Tensor GL on axis-aligned boxes. lo, hi (E, 3) -> pts (E, n^3, 3), w (E, n^3)."""
    n = npts_for_degree(q)
    x, w = gauss_legendre_01(n)
    X = np.stack(np.meshgrid(x, x, x, indexing="ij"), axis=-1).reshape(-1, 3)
    W = (w[:, None, None] * w[None, :, None] * w[None, None, :]).reshape(-1)
    ext = hi - lo
    pts = lo[:, None, :] + X[None, :, :] * ext[:, None, :]
    wts = W[None, :] * np.prod(ext, axis=1)[:, None]
    return pts, wts


def parallelogram_rule(v0: np.ndarray, v1: np.ndarray, v3: np.ndarray, q: int):
    """p = v0 + u (v1 - v0) + v (v3 - v0), (u, v) in [0,1]^2. (E,3) each."""
    n = npts_for_degree(q)
    x, w = gauss_legendre_01(n)
    U, V = np.meshgrid(x, x, indexing="ij")
    U, V = U.reshape(-1), V.reshape(-1)
    W = (w[:, None] * w[None, :]).reshape(-1)
    a = v1 - v0
    b = v3 - v0
    area = np.linalg.norm(np.cross(a, b), axis=1)
    pts = v0[:, None, :] + U[None, :, None] * a[:, None, :] + V[None, :, None] * b[:, None, :]
    return pts, W[None, :] * area[:, None]


def triangle_rule(v0: np.ndarray, v1: np.ndarray, v2: np.ndarray, q: int):
    """Collapsed GL on triangles: s = u, t = (1-u) v, Jacobian (1-u) * 2|T|."""
    n = npts_for_degree(q, 1)
    x, w = gauss_legendre_01(n)
    U, V = np.meshgrid(x, x, indexing="ij")
    U, V = U.reshape(-1), V.reshape(-1)
    W = (w[:, None] * w[None, :]).reshape(-1) * (1.0 - U)
    S, T = U, (1.0 - U) * V
    a = v1 - v0
    b = v2 - v0
    area2 = np.linalg.norm(np.cross(a, b), axis=1)
    pts = v0[:, None, :] + S[None, :, None] * a[:, None, :] + T[None, :, None] * b[:, None, :]
    return pts, W[None, :] * area2[:, None]


def tet_rule(v0, v1, v2, v3, q: int):
    """Collapsed GL on tetrahedra: s = u, t = (1-u) v, r = (1-u)(1-v) w,
    Jacobian (1-u)^2 (1-v) * 6|T|.  Returns pts (E, n^3, 3), w (E, n^3)."""
    n = npts_for_degree(q, 2)
    x, w = gauss_legendre_01(n)
    U, V, Wc = np.meshgrid(x, x, x, indexing="ij")
    U, V, Wc = U.reshape(-1), V.reshape(-1), Wc.reshape(-1)
    W = (w[:, None, None] * w[None, :, None] * w[None, None, :]).reshape(-1)
    W = W * (1.0 - U) ** 2 * (1.0 - V)
    S = U
    T = (1.0 - U) * V
    R = (1.0 - U) * (1.0 - V) * Wc
    a, b, c = v1 - v0, v2 - v0, v3 - v0
    vol6 = np.abs(np.einsum("ij,ij->i", a, np.cross(b, c)))
    pts = (v0[:, None, :] + S[None, :, None] * a[:, None, :] + T[None, :, None] * b[:, None, :]
           + R[None, :, None] * c[:, None, :])
    return pts, W[None, :] * vol6[:, None]
