"""Scaled monomial bases and the G_k (+) G_k^perp machinery of PAPER.md §2.

Input-generator code (see vemgen/__init__.py): shared by the oracle tests and
the CUDA-path tests as the definition of the assembled system, never called by
the GPU solve itself.

Citations are PAPER.md line numbers (P:n):
  * scaled monomials m_alpha = ((x - x_P)/h_P)^alpha, eqn:monoBasis
  * face monomials m^f_beta
  * Props. 1-3 (decomposition of vector monomials)
  * Prop. inTermsOfGPerpBasis
  * generator set M^{G,+}_{k-1} and N_k (eqn:NDef), read with
    "0 <= |alpha|" (reading R2: the printed "0<|alpha|" contradicts
    the paper's own count at P:548).
"""
from __future__ import annotations

import numpy as np


def multi_indices_3d(k: int) -> list[tuple[int, int, int]]:
    """Graded-lex list of alpha with 0 <= |alpha| <= k (M_k(P))."""
    out = []
    for d in range(k + 1):
        for a1 in range(d, -1, -1):
            for a2 in range(d - a1, -1, -1):
                out.append((a1, a2, d - a1 - a2))
    return out


def multi_indices_2d(k: int) -> list[tuple[int, int]]:
    """Graded-lex list of beta with 0 <= |beta| <= k (M_k(f))."""
    out = []
    for d in range(k + 1):
        for b1 in range(d, -1, -1):
            out.append((b1, d - b1))
    return out


def dim_pk_3d(k: int) -> int:
    return 0 if k < 0 else (k + 1) * (k + 2) * (k + 3) // 6


def dim_pk_2d(k: int) -> int:
    return 0 if k < 0 else (k + 1) * (k + 2) // 2


def dim_gperp(k: int) -> int:
    """dim G_k^perp = (2k^3 + 9k^2 + 7k)/6, eqn:dimGperp."""
    return (2 * k ** 3 + 9 * k ** 2 + 7 * k) // 6


def index_map_3d(k: int) -> dict:
    return {a: i for i, a in enumerate(multi_indices_3d(k))}


def eval_monomials_3d(s: np.ndarray, k: int) -> np.ndarray:
    """m_alpha at scaled coordinates s = (x - x_P)/h_P; s (..., 3) -> (..., n_k)."""
    alphas = multi_indices_3d(k)
    pw = [np.stack([s[..., d] ** p for p in range(k + 2)], axis=-1) for d in range(3)]
    out = np.empty(s.shape[:-1] + (len(alphas),))
    for i, (a1, a2, a3) in enumerate(alphas):
        out[..., i] = pw[0][..., a1] * pw[1][..., a2] * pw[2][..., a3]
    return out


def eval_monomials_2d(t: np.ndarray, k: int) -> np.ndarray:
    """m^f_beta at scaled face coordinates t (..., 2) -> (..., n_f)."""
    betas = multi_indices_2d(k)
    out = np.empty(t.shape[:-1] + (len(betas),))
    for i, (b1, b2) in enumerate(betas):
        out[..., i] = t[..., 0] ** b1 * t[..., 1] ** b2
    return out


def generators(k: int) -> list[tuple[int, tuple[int, int, int]]]:
    """M^{G,+}_{k-1}(P): list of (component c, alpha) meaning the vector
    monomial with m_alpha in component c.

    Component 0 takes alpha in N_{k-1} = {alpha_1 = 0, 0 <= |alpha| <= k-1}
    (reading R2 of eqn:NDef); components 1 and 2 take all of M_{k-1}(P).
    """
    if k <= 0:
        return []
    out = [(0, a) for a in multi_indices_3d(k - 1) if a[0] == 0]
    out += [(1, a) for a in multi_indices_3d(k - 1)]
    out += [(2, a) for a in multi_indices_3d(k - 1)]
    assert len(out) == dim_gperp(k)
    return out


def cross_term_as_generators(c: int, alpha: tuple[int, int, int]) -> list[tuple[float, int, tuple]]:
    """Express m_I ^ (e_c m_alpha) as a combination of m_I ^ generator.

    Components 1, 2 and component 0 with alpha_1 = 0 are generators already.
    Component 0 with alpha_1 >= 1 uses Prop. inTermsOfGPerpBasis:
      m_I ^ (m_a,0,0) = - m_I ^ (0,m_b,0) - m_I ^ (0,0,m_g),
      b = (a1-1, a2+1, a3), g = (a1-1, a2, a3+1).
    Returns [(coef, c', alpha')].
    """
    a1, a2, a3 = alpha
    if c != 0 or a1 == 0:
        return [(1.0, c, alpha)]
    return [(-1.0, 1, (a1 - 1, a2 + 1, a3)), (-1.0, 2, (a1 - 1, a2, a3 + 1))]


def decompose_vector_monomial(c: int, alpha: tuple[int, int, int], h: float = 1.0):
    """Props. 1-3: e_c m_alpha = (h_P/(|a|+1)) grad m_beta + sum of
    coef * m_I ^ (e_c' m_alpha').

    Returns (grad_coef, beta, [(coef, c', alpha'), ...]) where grad_coef is the
    multiplier of grad m_beta *including* h_P; the cross terms are not yet
    rewritten in the generator basis.
    """
    a = list(alpha)
    n1 = sum(a) + 1.0
    beta = list(a)
    beta[c] += 1
    cross = []

    def sub(idx, d):
        b = list(a)
        b[d] -= 1
        return tuple(b)

    if c == 0:
        # Prop. 1: - a3/(|a|+1) m_I ^ (0, m_{a-e3}, 0) + a2/(|a|+1) m_I ^ (0,0,m_{a-e2})
        if a[2] > 0:
            cross.append((-a[2] / n1, 1, sub(a, 2)))
        if a[1] > 0:
            cross.append((a[1] / n1, 2, sub(a, 1)))
    elif c == 1:
        # Prop. 2: + a3/(|a|+1) m_I ^ (m_{a-e3},0,0) - a1/(|a|+1) m_I ^ (0,0,m_{a-e1})
        if a[2] > 0:
            cross.append((a[2] / n1, 0, sub(a, 2)))
        if a[0] > 0:
            cross.append((-a[0] / n1, 2, sub(a, 0)))
    else:
        # Prop. 3: + a1/(|a|+1) m_I ^ (0,m_{a-e1},0) - a2/(|a|+1) m_I ^ (m_{a-e2},0,0)
        if a[0] > 0:
            cross.append((a[0] / n1, 1, sub(a, 0)))
        if a[1] > 0:
            cross.append((-a[1] / n1, 0, sub(a, 1)))
    return h / n1, tuple(beta), cross


def cross_mI(s: np.ndarray, vec: np.ndarray) -> np.ndarray:
    """m_I ^ vec where m_I = s (scaled coordinates), both (..., 3)."""
    return np.cross(s, vec)
