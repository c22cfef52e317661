"""GPU-vs-oracle parity through the C ABI (libvem_mixed.so, sm_100a).

Tolerances (BASELINE.json north_star, reading R20):
  * SpMV / S_D product: ||y_gpu - y_oracle||_inf <= 1e-12 ||y_oracle||_inf
  * solution: u and p separately, ||.||_inf relative <= 1e-8 at rtol 1e-10
  * GMRES iteration counts within +-2 of the oracle's (FGMRES: outer count)
Full-size configs are checked on sampled rows and by properties that hold at
any size (true residual, local conservation B u = f).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import solver as O
from vemgen import configs, mesh
from vemgen.assemble import build_system

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_02330_b200 as pkg  # noqa: E402

RNG = np.random.default_rng(2024)
_CACHE = {}


def system(name):
    if name not in _CACHE:
        _CACHE[name] = configs.CONFIGS[name].build()
    return _CACHE[name]


def solver_for(s, eps=None, **opts):
    o = pkg.default_options(**opts) if opts else None
    return pkg.VemMixed(s.M, s.B, eps=configs.eps_for(s) if eps is None else eps, layout=s.layout, opts=o)


def rel_inf(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s", "C5s"])
def test_spmv_parity(name):
    s = system(name)
    sv = solver_for(s)
    for _ in range(3):
        x = RNG.normal(size=s.n)
        y = sv.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_inf(y, O.spmv_saddle(s.M, s.B, x)) <= 1e-12
    sv.close()


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s", "C5s"])
def test_schur_product_parity(name):
    s = system(name)
    sv = solver_for(s)
    Sg = sv.get_schur()
    So = O.schur_diag(s.M, s.B)
    d = abs(Sg - So)
    assert d.max() <= 1e-12 * abs(So).max()
    x = RNG.normal(size=s.layout.n_p)
    y = sv.schur_spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel_inf(y, So @ x) <= 1e-12
    info = sv.info()
    assert abs(info["lambda_max"] - O.gershgorin_lmax(So)) <= 1e-12 * info["lambda_max"]
    sv.close()


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s"])
def test_block_schur_apply_parity(name):
    s = system(name)
    sv = solver_for(s)
    P = O.Preconditioner(O.PRECOND_BLOCK_SCHUR, s.M, s.B, block=s.layout.n_p_dof)
    v = RNG.normal(size=s.n)
    z, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR, torch.from_numpy(v).cuda())
    zo = P.apply(v)
    nu = s.layout.n_u
    assert rel_inf(z.cpu().numpy()[:nu], zo[:nu]) <= 1e-12
    assert rel_inf(z.cpu().numpy()[nu:], zo[nu:]) <= 1e-10
    sv.close()


@pytest.mark.parametrize("name", ["C1", "C3s", "C2s", "C4s"])
def test_block_reg_apply_parity(name):
    s = system(name)
    eps = configs.eps_for(s)
    sv = solver_for(s)
    P = O.Preconditioner(O.PRECOND_BLOCK_REG, s.M, s.B, eps=eps, block=s.layout.n_p_dof)
    v = RNG.normal(size=s.n)
    z, its = sv.precond_apply(pkg.PRECOND_BLOCK_REG, torch.from_numpy(v).cuda())
    zo = P.apply(v)
    nu = s.layout.n_u
    assert abs(its - P.inner_iterations) <= 2
    assert rel_inf(z.cpu().numpy()[:nu], zo[:nu]) <= 1e-8
    assert rel_inf(z.cpu().numpy()[nu:], zo[nu:]) <= 1e-14
    sv.close()


# (config, preconditioner) pairs of BASELINE.json at reduced size, plus C1/C3s Block-Reg.
SOLVE_CASES = [("C1", 1), ("C1", 2), ("C3s", 1), ("C3s", 2), ("C2s", 1), ("C2s", 2), ("C4s", 1), ("C4s", 2)]


# Oracle counts under 8 RHS perturbations of 1e-15 relative (a few ulps), /tmp-measured with the
# oracle alone and recorded in DESIGN.md R20: every case below has a spread of at most 1 except
# C4s Block-Schur (198..216: GMRES(50) on the k = 2 cube ends cycles with the estimate within
# rounding of rtol).  Only that case is compared with a band; the others are strict +-2.
BAND_CASES = {("C4s", 1): 8}


def log_counts(**kw):
    """Per-case iteration counts, appended to gpurun_out/parity_counts.jsonl (copied to
    profiles/ after a GPU run): the record `pytest -q` does not keep."""
    import json
    import os
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    try:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "parity_counts.jsonl"), "a") as f:
            f.write(json.dumps(kw) + "\n")
    except OSError:
        pass


def oracle_iteration_band(s, kind, restart, eps, trials=0):
    """The oracle's solve and its iteration count.  trials > 0 (BAND_CASES only, DESIGN.md
    reading R20): the count is the set over the unperturbed RHS and `trials` RHS perturbed
    by 1e-15 relative, for the one case whose restarted-GMRES count is ill-conditioned in
    the oracle itself; trials = 0: the band is the single unperturbed count (strict +-2)."""
    rng = np.random.default_rng(99)
    its = []
    ref = None
    for t in range(trials + 1):
        rhs = s.rhs if t == 0 else s.rhs * (1 + 1e-15 * rng.normal(size=s.rhs.size))
        r = O.solve(s.M, s.B, rhs, kind, 1e-10, restart, eps=eps, block=s.layout.n_p_dof)
        assert r.converged
        its.append(r.iterations)
        ref = ref or r
    return ref, min(its), max(its)


@pytest.mark.parametrize("name,kind", SOLVE_CASES)
def test_solve_parity(name, kind):
    s = system(name)
    cfg = configs.CONFIGS[name]
    eps = configs.eps_for(s)
    ref, lo, hi = oracle_iteration_band(s, kind, cfg.restart, eps, BAND_CASES.get((name, kind), 0))
    sv = solver_for(s, restart=cfg.restart)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, kind)
    r = res.report
    assert r["status"] == 0 and r["converged"] == 1, r
    print(f"{name} precond={kind}: gpu {r['iterations']} oracle {ref.iterations} band [{lo}, {hi}] its")
    log_counts(test="solve_parity", config=name, precond=kind, gpu=r["iterations"], oracle=ref.iterations,
               band=[lo, hi], gpu_inner=r["inner_iterations"], oracle_inner=ref.inner_iterations)
    assert lo - 2 <= r["iterations"] <= hi + 2, (r["iterations"], lo, hi)
    nu = s.layout.n_u
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8
    assert rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    # true residual and local conservation, recomputed on the host
    x = np.concatenate([res.u.cpu().numpy(), res.p.cpu().numpy()])
    assert np.linalg.norm(s.rhs - O.spmv_saddle(s.M, s.B, x)) <= 1e-10 * np.linalg.norm(s.rhs) * 1.0001
    sv.close()


@pytest.mark.parametrize("name,kind,nsteps", [("C1", 1, 50), ("C3s", 1, 50), ("C3s", 3, 50), ("C2s", 1, 30),
                                              ("C4s", 1, 20), ("C3s", 2, 50)])
def test_first_cycle_residual_history(name, kind, nsteps):
    """Element-wise parity of the Givens residual history |g_{j+1}| / ||b|| of the first
    GMRES(m) cycle (one cycle from x0 = 0 on both sides): every Arnoldi step of the cycle,
    not only the count.  The estimates agree to 1e-5 relative while they are above 1e-8 (the
    rounding of ~1e-16 ||b|| in w is amplified by 1 / est: 1e-14 at the first steps, 1e-6 near
    est = 1e-8), and to 1e-2 below.  C4s Block-Schur, the case whose count is ill-conditioned in the
    oracle itself (R20: CGS1 on a nearly invariant Krylov space), is held to this over its first 20
    steps; its later steps differ by up to 5e-2 and are only logged.  Block-Reg at k >= 1 (C2s) is
    not held to it: its estimates sit at 1 - O(1e-4) for most of the cycle (the (eps W)^-1 block
    scales the pressure part by 1e6), so est-relative differences of 1e-4..0.5 between two inner
    PCG solves that both stop at 1e-14 say nothing; its count, solution and inner step counts are
    compared in test_solve_parity and tests/test_gpu_blockreg_m.py."""
    s = system(name)
    cfg = configs.CONFIGS[name]
    eps = configs.eps_for(s)
    m = cfg.restart
    ref = O.solve(s.M, s.B, s.rhs, kind, 1e-10, m, maxit=m, eps=eps, block=s.layout.n_p_dof)
    sv = solver_for(s, restart=m)
    sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, m, kind)
    h = sv.last_cycle_history()
    ho = np.array(ref.history[:len(h)])
    assert len(h) == min(m, ref.iterations) == len(ho)
    big = ho > 1e-8
    err = np.abs(h - ho) / ho
    log_counts(test="first_cycle_history", config=name, precond=kind, steps=len(h),
               max_rel_err_above_1em8=float(err[big].max()) if big.any() else 0.0, max_rel_err=float(err.max()),
               last=float(h[-1]), oracle_last=float(ho[-1]))
    big[nsteps:] = False
    assert err[big].max() <= 1e-5, (err.max(), int(err.argmax()))
    assert np.all(err[:nsteps][~big[:nsteps]] <= 1e-2)
    sv.close()


def test_block_reg_fixed_budget_c5s():
    """C5 (pairs, anisotropic K with 1e-3 jumps) stagnates with the diag(M)-Woodbury
    Block-Reg (kind 2; kind 5 is the converging form, tests/test_gpu_blockreg_m.py), so
    kind-2 parity on this mesh is checked on a fixed budget: one FGMRES(50) cycle from
    x0 = 0 on both sides."""
    s = system("C5s")
    eps = configs.eps_for(s)
    ref = O.solve(s.M, s.B, s.rhs, 2, 1e-10, 50, maxit=50, eps=eps, block=s.layout.n_p_dof)
    sv = solver_for(s, restart=50)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 50, 2)
    assert res.report["iterations"] == ref.iterations == 50
    assert abs(res.report["rel_residual_true"] - ref.rel_residual_true) <= 1e-6 * ref.rel_residual_true
    nu = s.layout.n_u
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-6
    assert rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-6
    sv.close()


@pytest.mark.parametrize("name", ["C4s", "C5s", "C2s"])
def test_sell_sigma_reordering(name):
    """SELL-C-sigma reordering (opts.reorder, k >= 1): active where it removes
    slice padding (C4s, C5s mix row lengths), invisible to the caller: every
    entry point returns the same numbers as the identity numbering up to the
    summation order, and a solve lands in the same iteration band."""
    s = system(name)
    cfg = configs.CONFIGS[name]
    a = solver_for(s, restart=cfg.restart)
    b = solver_for(s, restart=cfg.restart, reorder=0)
    ia, ib = a.info(), b.info()
    assert ib["reordered"] == 0
    if name != "C2s":
        assert ia["reordered"] == 1
        assert ia["nnz_A_stored"] + ia["nnz_S_stored"] < 0.95 * (ib["nnz_A_stored"] + ib["nnz_S_stored"])
    x = RNG.normal(size=s.n)
    ya = a.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel_inf(ya, O.spmv_saddle(s.M, s.B, x)) <= 1e-12
    xp = RNG.normal(size=s.layout.n_p)
    ysa = a.schur_spmv(torch.from_numpy(xp).cuda()).cpu().numpy()
    assert rel_inf(ysa, O.schur_diag(s.M, s.B) @ xp) <= 1e-12
    for kind in cfg.precs:
        za, _ = a.precond_apply(kind, torch.from_numpy(x).cuda())
        zb, _ = b.precond_apply(kind, torch.from_numpy(x).cuda())
        assert rel_inf(za.cpu().numpy(), zb.cpu().numpy()) <= 1e-8
    kind = cfg.precs[0]
    if name == "C5s":   # fixed budget (see test_block_reg_fixed_budget_c5s)
        ra = a.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 50, kind)
        rb = b.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 50, kind)
        assert rel_inf(ra.u.cpu().numpy(), rb.u.cpu().numpy()) <= 1e-6
        assert rel_inf(ra.p.cpu().numpy(), rb.p.cpu().numpy()) <= 1e-6
    else:               # a reordering is an ulp-level perturbation: compare with the oracle band (R20)
        ref, lo, hi = oracle_iteration_band(s, kind, cfg.restart, configs.eps_for(s))
        ra = a.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, kind)
        assert ra.report["converged"] == 1
        assert lo - 2 <= ra.report["iterations"] <= hi + 2, (ra.report["iterations"], lo, hi)
        nu = s.layout.n_u
        assert rel_inf(ra.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(ra.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["C1", "C3s", "C2s"])
def test_cgs2_option_parity(name):
    """opts.reorth = 1 (CGS2 for every preconditioner) against the oracle's CGS2."""
    s = system(name)
    cfg = configs.CONFIGS[name]
    ref = O.solve(s.M, s.B, s.rhs, 1, 1e-10, cfg.restart, block=s.layout.n_p_dof, reorth=1)
    sv = solver_for(s, restart=cfg.restart, reorth=1)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 1)
    assert res.report["converged"] == 1 and abs(res.report["iterations"] - ref.iterations) <= 2
    nu = s.layout.n_u
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


@pytest.mark.parametrize("name", ["C1", "C3s"])
def test_amg_hierarchy_matches_oracle(name):
    """Block-Schur-AMG (kind 3): the device aggregation reproduces the oracle's
    hierarchy (rows and nnz of every level, integers), the V-cycle apply agrees
    to 1e-10, and the solve is within the iteration band."""
    from oracle.amg import AMG
    s = system(name)
    cfg = configs.CONFIGS[name]
    SD = O.schur_diag(s.M, s.B)
    h = AMG(SD)
    sv = solver_for(s, restart=cfg.restart)
    assert sv.amg_levels() == [(lev.A.shape[0], lev.A.nnz) for lev in h.levels]
    v = RNG.normal(size=s.n)
    z, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR_AMG, torch.from_numpy(v).cuda())
    nu = s.layout.n_u
    zo = np.concatenate([v[:nu] / s.M.diagonal(), -h.vcycle(v[nu:])])
    assert rel_inf(z.cpu().numpy()[:nu], zo[:nu]) <= 1e-12
    assert rel_inf(z.cpu().numpy()[nu:], zo[nu:]) <= 1e-10
    ref, lo, hi = oracle_iteration_band(s, 3, cfg.restart, 0.0)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 3)
    assert res.report["converged"] == 1
    assert lo - 2 <= res.report["iterations"] <= hi + 2, (res.report["iterations"], lo, hi)
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


@pytest.mark.parametrize("name", ["C1", "C3s"])
def test_amg_fp32_vcycle_parity(name):
    """Precond kind 4: the same hierarchy with the V-cycle in
    FP32 inside FP64 FGMRES.  The apply agrees with the oracle's float32 V-cycle to
    FP32 accuracy, and the solve reaches the FP64 tolerance with the oracle's count."""
    s = system(name)
    cfg = configs.CONFIGS[name]
    sv = solver_for(s, restart=cfg.restart)
    P = O.Preconditioner(O.PRECOND_BLOCK_SCHUR_AMG_F32, s.M, s.B)
    v = RNG.normal(size=s.n)
    z, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR_AMG_F32, torch.from_numpy(v).cuda())
    zo = P.apply(v)
    nu = s.layout.n_u
    assert rel_inf(z.cpu().numpy()[:nu], zo[:nu]) <= 1e-12
    assert rel_inf(z.cpu().numpy()[nu:], zo[nu:]) <= 2e-5
    ref, lo, hi = oracle_iteration_band(s, 4, cfg.restart, 0.0)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 4)
    assert res.report["converged"] == 1
    assert lo - 2 <= res.report["iterations"] <= hi + 2, (res.report["iterations"], lo, hi)
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


# 32^3 C3-type cube system: with VEM_AMG_MAX_LEVELS=2 its coarsest level (the SA
# Galerkin level, 3,643 rows, 33 nnz/row) is above the dense-inverse size, so the
# V-cycle ends in the degree-32 Chebyshev coarse smoother (oracle/amg.py AMG.vcycle)
C3M = configs.Config("C3m", "cube", 32, 0, (3,), 50, block=4, seed=3)


@pytest.mark.parametrize("cluster", [1, 0])
def test_amg_cluster_coarsest(monkeypatch, cluster):
    """The non-dense coarsest level smoothed by ONE 16-CTA thread-block-cluster launch
    (k_vc_coarse_cluster: CSR slices in shared memory, directions read through
    distributed shared memory) against the oracle's Chebyshev(32) coarse solve, FP64
    and FP32, and against the per-step warp kernels (cluster = 0)."""
    from oracle.amg import AMG
    monkeypatch.setenv("VEM_AMG_MAX_LEVELS", "2")
    monkeypatch.setenv("VEM_AMG_CLUSTER", str(cluster))
    if "C3m" not in _CACHE:
        _CACHE["C3m"] = C3M.build()
    s = _CACHE["C3m"]
    SD = O.schur_diag(s.M, s.B)
    h = AMG(SD, max_levels=2)
    assert h.coarse_inv is None
    sv = solver_for(s, restart=50)
    assert sv.amg_levels() == [(lev.A.shape[0], lev.A.nnz) for lev in h.levels]
    assert sv.info()["amg_coarse_cluster"] == cluster
    nu = s.layout.n_u
    v = RNG.normal(size=s.n)
    z, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR_AMG, torch.from_numpy(v).cuda())
    zo = -h.vcycle(v[nu:])
    assert rel_inf(z.cpu().numpy()[nu:], zo) <= 1e-10
    z32, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR_AMG_F32, torch.from_numpy(v).cuda())
    zo32 = -h.to_float32().vcycle(v[nu:].astype(np.float32)).astype(np.float64)
    assert rel_inf(z32.cpu().numpy()[nu:], zo32) <= 2e-5
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 3)
    assert res.report["converged"] == 1 and res.report["rel_residual_true"] <= 1e-10
    sv.close()


@pytest.mark.parametrize("group", [4, 8, 16, 32])
def test_amg_three_level_group_csr(monkeypatch, group):
    """Default hierarchy of the 32^3 C3-type system: 32768 -> 3643 -> 867 (dense)
    rows, so the middle level runs the coarse CSR kernels (pre/post Chebyshev(3)
    smoothing, residuals) with G lanes per row (VEM_AMG_GROUP; default 8).  The
    V-cycle matches the oracle in FP64 and FP32 and the solve lands in the
    oracle's iteration band for every G."""
    from oracle.amg import AMG
    monkeypatch.setenv("VEM_AMG_GROUP", str(group))
    if "C3m" not in _CACHE:
        _CACHE["C3m"] = C3M.build()
    s = _CACHE["C3m"]
    SD = O.schur_diag(s.M, s.B)
    h = AMG(SD)
    assert len(h.levels) == 3 and h.coarse_inv is not None
    sv = solver_for(s, restart=50)
    assert sv.amg_levels() == [(lev.A.shape[0], lev.A.nnz) for lev in h.levels]
    nu = s.layout.n_u
    v = RNG.normal(size=s.n)
    z, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR_AMG, torch.from_numpy(v).cuda())
    assert rel_inf(z.cpu().numpy()[nu:], -h.vcycle(v[nu:])) <= 1e-10
    z32, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR_AMG_F32, torch.from_numpy(v).cuda())
    zo32 = -h.to_float32().vcycle(v[nu:].astype(np.float32)).astype(np.float64)
    assert rel_inf(z32.cpu().numpy()[nu:], zo32) <= 2e-5
    if group == 8:
        ref, lo, hi = oracle_iteration_band(s, 3, 50, 0.0)
        res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 3)
        assert res.report["converged"] == 1
        assert lo - 2 <= res.report["iterations"] <= hi + 2, (res.report["iterations"], lo, hi)
        assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


@pytest.mark.parametrize("name,kind", [("C1", 1), ("C3s", 1), ("C3s", 3), ("C2s", 2)])
def test_random_rhs_parity(name, kind):
    """the same matrices with the seeded N(0, 1) right-hand side
    (vemgen.configs.random_rhs, seed 7) -- representative iteration counts; GPU within
    the oracle's band, u and p within 1e-8."""
    s = system(name)
    cfg = configs.CONFIGS[name]
    eps = configs.eps_for(s)
    rhs = configs.random_rhs(s.n)

    class _S:   # the system with the random RHS (same matrices)
        M, B, layout = s.M, s.B, s.layout
    _S.rhs = rhs
    ref, lo, hi = oracle_iteration_band(_S, kind, cfg.restart, eps)
    sv = solver_for(s, restart=cfg.restart)
    res = sv.solve(torch.from_numpy(rhs).cuda(), 1e-10, 10000, kind)
    assert res.report["converged"] == 1
    assert lo - 2 <= res.report["iterations"] <= hi + 2, (res.report["iterations"], lo, hi)
    nu = s.layout.n_u
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


@pytest.mark.parametrize("name", ["C2s", "C4s", "C5s"])
def test_split_block_pcg_path(monkeypatch, name):
    """The split block-PCG kernels (k_pcg_spmv_p / k_pcg_alpha / k_pcg_vec_blk / k_pcg_beta /
    k_pcg_pupd, graph chunks): the form every k >= 1 system above 262,144 pressure unknowns
    runs (full C4, C5) when the inner preconditioner is the element-block Jacobi.  The reduced
    cases take the one-launch persistent kernel by default, so it is switched off here."""
    monkeypatch.setenv("VEM_PCG_PERSIST", "0")
    s = system(name)
    eps = configs.eps_for(s)
    sv = solver_for(s, inner_precond=0, restart=configs.CONFIGS[name].restart)
    P = O.Preconditioner(O.PRECOND_BLOCK_REG, s.M, s.B, eps=eps, block=s.layout.n_p_dof, inner_precond=0)
    v = RNG.normal(size=s.n)
    z, its = sv.precond_apply(pkg.PRECOND_BLOCK_REG, torch.from_numpy(v).cuda())
    zo = P.apply(v)
    nu = s.layout.n_u
    log_counts(test="split_block_pcg_apply", config=name, gpu_inner=its, oracle_inner=P.inner_iterations)
    assert abs(its - P.inner_iterations) <= 2
    assert rel_inf(z.cpu().numpy()[:nu], zo[:nu]) <= 1e-8
    if name != "C5s":   # kind 2 stagnates on the C5 type (R24)
        ref = O.solve(s.M, s.B, s.rhs, 2, 1e-10, configs.CONFIGS[name].restart, eps=eps, block=s.layout.n_p_dof,
                      inner_precond=0)
        res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 2)
        log_counts(test="split_block_pcg_solve", config=name, gpu=res.report["iterations"], oracle=ref.iterations)
        assert res.report["converged"] == 1
        assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


def test_amg_sell_coarse_levels(monkeypatch):
    """VEM_AMG_WARP_ROWS=0: every coarse level of the C3m hierarchy runs the SELL-32
    one-thread-per-row kernels, the form full C3's 206,540-row level 1 takes (levels with at
    least 100,000 rows); by default every C3m coarse level takes the CSR group kernels."""
    from oracle.amg import AMG
    monkeypatch.setenv("VEM_AMG_WARP_ROWS", "0")
    if "C3m" not in _CACHE:
        _CACHE["C3m"] = C3M.build()
    s = _CACHE["C3m"]
    h = AMG(O.schur_diag(s.M, s.B))
    sv = solver_for(s, restart=50)
    assert sv.amg_levels() == [(lev.A.shape[0], lev.A.nnz) for lev in h.levels]
    nu = s.layout.n_u
    v = RNG.normal(size=s.n)
    z, _ = sv.precond_apply(pkg.PRECOND_BLOCK_SCHUR_AMG, torch.from_numpy(v).cuda())
    assert rel_inf(z.cpu().numpy()[nu:], -h.vcycle(v[nu:])) <= 1e-10
    ref = O.solve(s.M, s.B, s.rhs, 3, 1e-10, 50)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 3)
    log_counts(test="amg_sell_coarse_levels", config="C3m", gpu=res.report["iterations"], oracle=ref.iterations)
    assert res.report["converged"] == 1 and abs(res.report["iterations"] - ref.iterations) <= 2
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


def test_fixed_grid_cgs_fallback(monkeypatch):
    """ADVICE (round 1): the fixed-grid k_mdot / k_update launch forms (VEM_MDOT_WAVE=0,
    VEM_UPDATE_WAVE=0) stay tested: same count, same solution as the oracle on C3s."""
    monkeypatch.setenv("VEM_MDOT_WAVE", "0")
    monkeypatch.setenv("VEM_UPDATE_WAVE", "0")
    s = system("C3s")
    ref = O.solve(s.M, s.B, s.rhs, 3, 1e-10, 50)
    sv = solver_for(s, restart=50)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 3)
    nu = s.layout.n_u
    assert res.report["converged"] == 1 and abs(res.report["iterations"] - ref.iterations) <= 2
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


@pytest.mark.parametrize("name,kind", [("C1", 1), ("C3s", 1), ("C3s", 3), ("C2s", 1), ("C3s", 2)])
def test_compressed_basis_parity(name, kind):
    """opts.basis_f32 (traffic-reduced Krylov): the basis vectors are the
    float32 roundings of the Arnoldi vectors, the CGS kernels stream the float copy.  Same
    definition in the oracle (gmres(basis32=True)): count +-2, u and p to 1e-8 of the oracle's
    compressed-basis solve AND of its full-precision solve (the restart recovers the accuracy)."""
    s = system(name)
    cfg = configs.CONFIGS[name]
    eps = configs.eps_for(s)
    nb = s.layout.n_p_dof
    ref = O.solve(s.M, s.B, s.rhs, kind, 1e-10, cfg.restart, eps=eps, block=nb, basis32=True)
    full = O.solve(s.M, s.B, s.rhs, kind, 1e-10, cfg.restart, eps=eps, block=nb)
    assert ref.converged
    sv = solver_for(s, restart=cfg.restart, basis_f32=1)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, kind)
    r = res.report
    log_counts(test="compressed_basis", config=name, precond=kind, gpu=r["iterations"], oracle=ref.iterations,
               oracle_fp64_basis=full.iterations)
    assert r["converged"] == 1 and abs(r["iterations"] - ref.iterations) <= 2, (r["iterations"], ref.iterations)
    nu = s.layout.n_u
    for x in (ref.x, full.x):
        assert rel_inf(res.u.cpu().numpy(), x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), x[nu:]) <= 1e-8
    # switching back restores the full-precision basis
    sv.set_options(basis_f32=0)
    res2 = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, kind)
    assert abs(res2.report["iterations"] - full.iterations) <= 2
    sv.close()


def test_solve_host_matches_device_and_is_deterministic():
    s = system("C3s")
    sv = solver_for(s, restart=50)
    a = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 1)
    b = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 1)
    h = sv.solve_host(s.rhs, 1e-10, 10000, 1)
    assert np.array_equal(a.u.cpu().numpy(), b.u.cpu().numpy())
    assert np.array_equal(a.u.cpu().numpy(), h.u) and np.array_equal(a.p.cpu().numpy(), h.p)
    assert a.report["iterations"] == b.report["iterations"] == h.report["iterations"]
    sv.close()


def test_graphs_and_timing_mode_agree():
    s = system("C3s")
    sv = solver_for(s, restart=50)
    a = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 1)
    sv.set_options(use_graphs=0, timing=1)
    b = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 1)
    assert np.array_equal(a.u.cpu().numpy(), b.u.cpu().numpy())
    st = sv.kernel_stats(reset=True)
    assert st["spmv"]["launches"] >= b.report["iterations"] and st["cheb"]["launches"] > 0
    sv.set_options(use_graphs=1, timing=2)      # sampled events inside the cycle graphs
    c = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 1)
    assert np.array_equal(a.u.cpu().numpy(), c.u.cpu().numpy())
    st = sv.kernel_stats(reset=True)
    assert st["cheb"]["launches"] == c.report["iterations"] and st["cheb"]["ms"] > 0
    sv.close()


def test_edge_cases():
    s = system("C1")
    sv = solver_for(s)
    z = torch.zeros(s.n, dtype=torch.float64, device="cuda")
    r = sv.solve(z, 1e-10, 100, 1)
    assert r.report["iterations"] == 0 and r.report["converged"] == 1
    assert float(r.u.abs().max()) == 0.0
    r = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 3, 1)
    assert r.report["status"] == 1 and r.report["iterations"] == 3
    ref = O.solve(s.M, s.B, s.rhs, 1, 1e-10, 30, maxit=3, block=1)
    nu = s.layout.n_u
    assert rel_inf(r.u.cpu().numpy(), ref.x[:nu]) <= 1e-10
    with pytest.raises(pkg.VemError):
        sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 100, 7)
    sv.close()
    # no eps -> Block-Reg unsupported
    sv = solver_for(s, eps=0.0)
    with pytest.raises(pkg.VemError):
        sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 100, 2)
    sv.close()


def test_invalid_uploads():
    s = system("C1")
    bad = s.M.copy()
    bad.data[bad.indptr[5]:bad.indptr[6]] *= 0.0  # zero row incl. diagonal
    with pytest.raises(pkg.VemError, match="DIAG_M"):
        pkg.VemMixed(bad, s.B)
    Bz = s.B.tolil()
    Bz[3, :] = 0
    Bz = Bz.tocsr()
    Bz.eliminate_zeros()
    with pytest.raises(pkg.VemError, match="DIAG_S"):
        pkg.VemMixed(s.M, Bz)
    with pytest.raises(pkg.VemError, match="INVALID"):
        pkg.VemMixed(s.M, s.B[:, :-1])


@pytest.mark.parametrize("n,k", [(1, 0), (1, 1), (3, 2), (5, 0), (3, 1)])
def test_tiny_and_ragged_meshes(n, k):
    """Counts: strict at k = 0; at k >= 1 on these K = I cube grids the oracle's own count
    spreads under 1e-15 RHS perturbations (3^3 k = 2: 138..143, k = 1: 45..47; the C4s
    mechanism of DESIGN.md R20), so the band of 8 perturbed oracle runs applies."""
    s = build_system(mesh.cube_mesh(n), k)
    ref, lo, hi = oracle_iteration_band(s, 1, 30, 0.0, 8 if k >= 1 else 0)
    sv = solver_for(s)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 1)
    assert lo - 2 <= res.report["iterations"] <= hi + 2, (res.report["iterations"], lo, hi)
    x = np.concatenate([res.u.cpu().numpy(), res.p.cpu().numpy()])
    nu = s.layout.n_u
    assert rel_inf(x[:nu], ref.x[:nu]) <= 1e-8 and rel_inf(x[nu:], ref.x[nu:]) <= 1e-8
    sv.close()


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C2", "C4"])
def test_full_size_k1_k2_sampled_and_properties(name):
    """C2 (k=1 tets) and C4 (k=2 cubes) at full size: sampled SpMV rows and S_D
    rows against the oracle definitions; both preconditioners converge to the
    true residual with element-wise conservation."""
    s = system(name)
    cfg = configs.CONFIGS[name]
    sv = solver_for(s, restart=cfg.restart)
    x = RNG.normal(size=s.n)
    y = sv.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    A = sp.bmat([[s.M, s.B.T], [s.B, None]]).tocsr()
    rows = RNG.choice(s.n, 20000, replace=False)
    yo = A[rows] @ x
    assert np.abs(y[rows] - yo).max() <= 1e-12 * np.abs(yo).max()
    xp = RNG.normal(size=s.layout.n_p)
    ys = sv.schur_spmv(torch.from_numpy(xp).cuda()).cpu().numpy()
    prow = RNG.choice(s.layout.n_p, 5000, replace=False)
    So = (s.B[prow] @ sp.diags(1 / s.M.diagonal()) @ s.B.T).tocsr()
    yso = So @ xp
    assert np.abs(ys[prow] - yso).max() <= 1e-12 * np.abs(yso).max()
    for kind in cfg.precs:
        res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 20000, kind)
        assert res.report["converged"] == 1, res.report
        u, p = res.u.cpu().numpy(), res.p.cpu().numpy()
        r = s.rhs - A @ np.concatenate([u, p])
        assert np.linalg.norm(r) <= 1.0001e-10 * np.linalg.norm(s.rhs)
        assert np.abs(s.B @ u - s.f).max() <= 1e-7 * np.abs(s.f).max()
    sv.close()


@pytest.mark.slow
def test_full_c5_sampled():
    """C5 at full size (14.0M DOFs, pairs, SELL-C-sigma reordered): sampled rows of the
    saddle SpMV and of S_D against the oracle definitions in the caller's numbering
    and the converging kind-5 solve."""
    s = system("C5")
    sv = solver_for(s, restart=50)
    assert sv.info()["reordered"] == 1
    x = RNG.normal(size=s.n)
    y = sv.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    A = sp.bmat([[s.M, s.B.T], [s.B, None]]).tocsr()
    rows = RNG.choice(s.n, 20000, replace=False)
    yo = A[rows] @ x
    assert np.abs(y[rows] - yo).max() <= 1e-12 * np.abs(yo).max()
    xp = RNG.normal(size=s.layout.n_p)
    ys = sv.schur_spmv(torch.from_numpy(xp).cuda()).cpu().numpy()
    prow = RNG.choice(s.layout.n_p, 5000, replace=False)
    So = (s.B[prow] @ sp.diags(1 / s.M.diagonal()) @ s.B.T).tocsr()
    yso = So @ xp
    assert np.abs(ys[prow] - yso).max() <= 1e-12 * np.abs(yso).max()
    # the headline solve at its stated size, in the configuration bench.py times (kind 5, FGMRES(50),
    # default options): the oracle cannot run at this size (one outer iteration takes ~20 min), so
    # what holds at any size is checked: convergence flag, the true residual and the element-wise
    # conservation recomputed on the host, the outer count in the h-independent range the oracle and
    # the GPU agree on from 6^3 to 64^3 (42..64), and the level sizes of the inner
    # hierarchy against the oracle's own construction (integer work, bit-exact)
    from oracle.amg import AMG
    eps = configs.eps_for(s)
    nb = s.layout.n_p_dof
    Se = (O.schur_diag(s.M, s.B) + eps * sp.identity(s.layout.n_p)).tocsr()
    h = AMG(Se[0::nb, 0::nb].tocsr())
    assert sv.inner_amg_levels() == [(lv.A.shape[0], lv.A.nnz) for lv in h.levels]
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 3000, pkg.PRECOND_BLOCK_REG_M)
    r = res.report
    log_counts(test="full_c5_kind5", gpu=r["iterations"], k=r["k_iterations"], inner=r["inner_iterations"],
               solve_ms=r["solve_ms"], rel_residual_true=r["rel_residual_true"])
    assert r["status"] == 0 and r["converged"] == 1, r
    assert 40 <= r["iterations"] <= 66, r
    u, p = res.u.cpu().numpy(), res.p.cpu().numpy()
    rr = s.rhs - A @ np.concatenate([u, p])
    assert np.linalg.norm(rr) <= 1.0001e-10 * np.linalg.norm(s.rhs)
    assert np.abs(s.B @ u - s.f).max() <= 1e-9 * np.abs(s.f).max()
    sv.close()


@pytest.mark.slow
def test_full_c3_sampled_and_properties():
    """C3 at full size (8.4M DOFs) in the bench's configuration: sampled SpMV
    rows against the oracle definition, then the solve's true residual and
    element-wise conservation recomputed on the host."""
    s = system("C3")
    sv = solver_for(s, restart=50)
    x = RNG.normal(size=s.n)
    y = sv.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    A = sp.bmat([[s.M, s.B.T], [s.B, None]]).tocsr()
    rows = RNG.choice(s.n, 20000, replace=False)
    yo = A[rows] @ x
    assert np.abs(y[rows] - yo).max() <= 1e-12 * np.abs(yo).max()
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 20000, 1)
    assert res.report["converged"] == 1
    u, p = res.u.cpu().numpy(), res.p.cpu().numpy()
    r = s.rhs - A @ np.concatenate([u, p])
    assert np.linalg.norm(r) <= 1.0001e-10 * np.linalg.norm(s.rhs)
    assert np.abs(s.B @ u - s.f).max() <= 1e-8 * np.abs(s.f).max()
    sv.close()


def test_full_c3_block_schur_amg_vs_oracle():
    """The round-1 headline path at its stated size: C3 (8.4M DOFs), kind 3, against the
    oracle's own full solve (about two minutes of numpy): level-by-level hierarchy rows,
    iteration count +-2, u and p to 1e-8."""
    from oracle.amg import AMG
    s = system("C3")
    SD = O.schur_diag(s.M, s.B)
    h = AMG(SD)
    sv = solver_for(s, restart=50)
    got = sv.amg_levels()
    want = [(lev.A.shape[0], lev.A.nnz) for lev in h.levels]
    log_counts(test="full_c3_hierarchy", gpu=got, oracle=want)
    # integer work, bit-exact: rows and nonzeros of every level (one exact-zero rule on both
    # sides: an entry exists iff a term of its sum exists, oracle/amg.py with_structure)
    assert got == want
    ref = O.solve(s.M, s.B, s.rhs, 3, 1e-10, 50)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 20000, 3)
    log_counts(test="full_c3_kind3", gpu=res.report["iterations"], oracle=ref.iterations)
    assert res.report["converged"] == 1 and abs(res.report["iterations"] - ref.iterations) <= 2
    nu = s.layout.n_u
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()


def test_full_c2_block_schur_vs_oracle():
    """C2 at its stated size (397,824 DOFs, Kuhn tets, k = 1), Block-Schur: the oracle's own full
    solve (about 20 s) against the GPU's: same iteration count +-2, u and p to 1e-8.  (Block-Reg at
    this size, C4 and the other stated-size comparisons take minutes of oracle time and are run
    once by tools/full_parity.py: profiles/R2_18_full_parity_c2.jsonl, R2_19_full_parity_c4.jsonl.)"""
    s = system("C2")
    cfg = configs.CONFIGS["C2"]
    ref = O.solve(s.M, s.B, s.rhs, 1, 1e-10, cfg.restart, block=s.layout.n_p_dof)
    sv = solver_for(s, restart=cfg.restart)
    res = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 20000, 1)
    log_counts(test="full_c2_kind1", gpu=res.report["iterations"], oracle=ref.iterations)
    assert res.report["converged"] == 1 and abs(res.report["iterations"] - ref.iterations) <= 2
    nu = s.layout.n_u
    assert rel_inf(res.u.cpu().numpy(), ref.x[:nu]) <= 1e-8 and rel_inf(res.p.cpu().numpy(), ref.x[nu:]) <= 1e-8
    sv.close()
