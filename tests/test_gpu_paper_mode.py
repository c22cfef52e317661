"""GPU-vs-oracle parity in paper mode: the paper's own BDM-type space
(gradient moments over M_{k-1} \\ M_0, divergence and pressure in P_{k-1}; PAPER.md
P:612-652) assembled by vemgen (paper_mode=True) on cube grids, solved through
the same C ABI with both of the paper's preconditioners."""
import numpy as np
import pytest

from oracle import solver as O
from vemgen import configs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_02330_b200 as pkg  # noqa: E402

RNG = np.random.default_rng(77)


def rel_inf(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name,kind", [("P1s", 1), ("P1s", 2), ("P1s", 3), ("P2s", 1), ("P2s", 2)])
def test_paper_mode_solve_parity(name, kind):
    cfg = configs.CONFIGS[name]
    s = cfg.build()
    eps = configs.eps_for(s)
    nb = s.layout.n_p_dof
    assert nb == (1 if cfg.k == 1 else 4)
    ref = O.solve(s.M, s.B, s.rhs, kind, 1e-10, cfg.restart, eps=eps, block=nb)
    assert ref.converged
    lo = hi = ref.iterations
    if (name, kind) == ("P2s", 1):
        # k = 2 cubes with K = I and Block-Schur: the count is ill-conditioned in the oracle itself
        # (R20, the C4s case): band over 8 RHS perturbations of 1e-15 relative
        rng = np.random.default_rng(99)
        its = [O.solve(s.M, s.B, s.rhs * (1 + 1e-15 * rng.normal(size=s.n)), kind, 1e-10, cfg.restart, eps=eps,
                       block=nb).iterations for _ in range(8)]
        lo, hi = min(its + [lo]), max(its + [hi])
    sv = pkg.VemMixed(s.M, s.B, eps=eps, layout=s.layout, opts=pkg.default_options(restart=cfg.restart))
    x = RNG.normal(size=s.n)
    y = sv.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel_inf(y, O.spmv_saddle(s.M, s.B, x)) <= 1e-12
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, kind)
    r = res.report
    print(f"{name} precond={kind}: gpu {r['iterations']} oracle {ref.iterations} band [{lo}, {hi}]")
    assert r["converged"] == 1 and lo - 2 <= r["iterations"] <= hi + 2, (r["iterations"], lo, hi)
    nu = s.layout.n_u
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8
    assert rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    u = res.u.cpu().numpy()
    assert np.abs(s.B @ u - s.f).max() <= 1e-8 * np.abs(s.f).max()   # local conservation
    sv.close()


@pytest.mark.parametrize("n,k,kind", [(4, 1, 1), (4, 1, 2), (3, 2, 1), (3, 2, 2)])
def test_paper_neumann_solve_parity(n, k, kind):
    """The paper's own boundary value problem (Neumann data, mean-value multiplier, polynomial
    solution; vemgen.configs.paper_neumann) through the C ABI: the multiplier in closed form, the
    consistent singular saddle system solved on the GPU, the pressure projected onto mean zero.
    Against the oracle's solve of the same system (u and p to 1e-8; count +-2 for Block-Schur, +-5
    for Block-Reg: on this singular system S_D + eps W has the eigenvalue eps on the constant
    pressure, the inner solves amplify rounding along it by 1 / eps, and the oracle's own count
    spreads 87..89 / 75..76 under 1e-15 RHS perturbations) and against the sparse LU solution of
    the bordered system with the multiplier (u, p to 1e-7)."""
    import scipy.sparse.linalg as spl
    s, N = configs.paper_neumann(n, k)
    nb = s.layout.n_p_dof
    eps = 1e-6 * float(N.M.diagonal().mean())
    ref = O.solve(N.M, N.B, N.rhs, kind, 1e-10, 50, eps=eps, block=nb, maxit=5000)
    assert ref.converged
    sv = pkg.VemMixed(N.M, N.B, eps=eps, layout=s.layout, opts=pkg.default_options(restart=50))
    res = sv.solve(torch.from_numpy(N.rhs).cuda(), 1e-10, 10000, kind)
    r = res.report
    print(f"paper Neumann n={n} k={k} precond={kind}: gpu {r['iterations']} oracle {ref.iterations}")
    assert r["converged"] == 1 and abs(r["iterations"] - ref.iterations) <= (2 if kind == 1 else 5), (
        r["iterations"], ref.iterations)
    nu = s.layout.n_u
    u, p = res.u.cpu().numpy(), N.project(res.p.cpu().numpy())
    assert rel_inf(u, ref.x[:nu]) <= 1e-8 and rel_inf(p, N.project(ref.x[nu:])) <= 1e-8
    x = spl.spsolve(N.bordered().tocsc(), N.bordered_rhs())
    assert rel_inf(u, x[:nu]) <= 1e-7 and rel_inf(p, x[nu:-1]) <= 1e-7
    assert abs(N.c @ p) <= 1e-12 * np.abs(N.c).sum() * np.abs(p).max()
    sv.close()
