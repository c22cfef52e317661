"""Element-parallel device assembly (vem_mixed_assemble) against
the host generator (vemgen.assemble.build_system), which defines the system.

Pattern (integers) must be identical; values are the same rounded products summed
in (class, cell, entry) order on both sides, so they agree to a few ulps (the host's
duplicate-summation order inside scipy's COO->CSR conversion is not specified);
f to 1e-14.  A solve from the device-assembled system matches the host-uploaded one.
"""
import time

import numpy as np
import pytest

from vemgen import configs
from vemgen.assemble import class_templates

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_02330_b200 as pkg  # noqa: E402


def _compare(s, M, B, f):
    assert np.array_equal(M.indptr, s.M.indptr) and np.array_equal(M.indices, s.M.indices)
    assert np.array_equal(B.indptr, s.B.indptr) and np.array_equal(B.indices, s.B.indices)
    dm = np.abs(M.data - s.M.data)
    assert dm.max() <= 4e-16 * np.abs(s.M.data).max() + 0.0, dm.max()
    assert np.all(dm <= 4 * np.spacing(np.abs(s.M.data)))
    assert np.array_equal(B.data, s.B.data)          # B entries are never summed (one cell per pressure row)
    assert np.abs(f - s.f).max() <= 1e-14 * np.abs(s.f).max()
    return float(np.mean(dm == 0.0))


@pytest.mark.parametrize("name", ["C1", "C3s", "C4s", "C5s"])
def test_device_assembly_matches_host(name):
    cfg = configs.CONFIGS[name]
    s = cfg.build()
    a = pkg.Assembled(class_templates(cfg.make_mesh(), cfg.k), s.layout.n_u, s.layout.n_p)
    assert a.nnz() == (s.M.nnz, s.B.nnz)
    M, B, f = a.to_host()
    exact = _compare(s, M, B, f)
    print(f"{name}: {exact:.4%} of M values bit-identical")
    a.close()


def test_solve_from_device_assembly():
    cfg = configs.CONFIGS["C3s"]
    s = cfg.build()
    a = pkg.Assembled(class_templates(cfg.make_mesh(), cfg.k), s.layout.n_u, s.layout.n_p)
    _, _, f = a.to_host()
    opts = pkg.default_options(restart=cfg.restart)
    sa = pkg.VemMixed.from_assembled(a, eps=configs.eps_for(s), layout=s.layout, opts=opts)
    a.close()                                          # the solver owns its own copy
    sh = pkg.VemMixed(s.M, s.B, eps=configs.eps_for(s), layout=s.layout, opts=opts)
    rhs = torch.from_numpy(np.concatenate([np.zeros(s.layout.n_u), f])).cuda()
    for kind in (1, 2, 3):
        ra = sa.solve(rhs, 1e-10, 10000, kind)
        rh = sh.solve(rhs, 1e-10, 10000, kind)
        assert ra.report["converged"] == 1
        assert abs(ra.report["iterations"] - rh.report["iterations"]) <= 2
        for x, y in ((ra.u, rh.u), (ra.p, rh.p)):
            x, y = x.cpu().numpy(), y.cpu().numpy()
            assert np.abs(x - y).max() <= 1e-9 * np.abs(y).max()
    sa.close()
    sh.close()


def test_assembly_rejects_bad_input():
    cfg = configs.CONFIGS["C1"]
    s = cfg.build()
    t = class_templates(cfg.make_mesh(), cfg.k)
    t[0] = dict(t[0])
    L = t[0]["L"].copy()
    L[3, 2] = s.layout.n_u + 5
    t[0]["L"] = L
    with pytest.raises(pkg.VemError, match="INVALID"):
        pkg.Assembled(t, s.layout.n_u, s.layout.n_p)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C5"])
def test_full_size_device_assembly(name):
    cfg = configs.CONFIGS[name]
    mesh = cfg.make_mesh()
    t0 = time.perf_counter()
    tm = class_templates(mesh, cfg.k)
    t1 = time.perf_counter()
    s = cfg.build()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    a = pkg.Assembled(tm, s.layout.n_u, s.layout.n_p)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    M, B, f = a.to_host()
    exact = _compare(s, M, B, f)
    print(f"{name}: shape cache {t1 - t0:.2f} s, host assembly {t2 - t1:.2f} s, device assembly "
          f"{t4 - t3:.3f} s (incl. H2D of the maps), {exact:.4%} of M values bit-identical")
    a.close()


@pytest.mark.parametrize("name", ["C2s"])
def test_device_local_operators_tets_match_host(name):
    """Kuhn tetrahedra (non-congruent, C2): the local operators (face polynomials,
    divergence, Pi^0_k, consistency, stabilisation) are computed on the device, one
    thread per cell, and assembled there.  Against the host generator: the same
    pattern, values to rounding (different order of the small dense solves), f to
    rounding; and a solve from the device-assembled system matches."""
    from vemgen.assemble import tet_class_input
    cfg = configs.CONFIGS[name]
    s = cfg.build()
    mesh = cfg.make_mesh()
    tin = [tet_class_input(mesh, c, cfg.k) for c in mesh.classes]
    a = pkg.Assembled(None, s.layout.n_u, s.layout.n_p, tets=tin)
    M, B, f = a.to_host()
    assert np.array_equal(M.indptr, s.M.indptr) and np.array_equal(M.indices, s.M.indices)
    assert np.array_equal(B.indptr, s.B.indptr) and np.array_equal(B.indices, s.B.indices)
    assert np.abs(M.data - s.M.data).max() <= 1e-12 * np.abs(s.M.data).max()
    assert np.abs(B.data - s.B.data).max() <= 1e-12 * np.abs(s.B.data).max()
    assert np.abs(f - s.f).max() <= 1e-12 * np.abs(s.f).max()
    opts = pkg.default_options(restart=cfg.restart)
    sa = pkg.VemMixed.from_assembled(a, eps=configs.eps_for(s), layout=s.layout, opts=opts)
    sh = pkg.VemMixed(s.M, s.B, eps=configs.eps_for(s), layout=s.layout, opts=opts)
    rhs = torch.from_numpy(s.rhs).cuda()
    ra, rh = sa.solve(rhs, 1e-10, 10000, 1), sh.solve(rhs, 1e-10, 10000, 1)
    assert ra.report["converged"] == 1 and abs(ra.report["iterations"] - rh.report["iterations"]) <= 2
    assert np.abs(ra.p.cpu().numpy() - rh.p.cpu().numpy()).max() <= 1e-8 * np.abs(rh.p.cpu().numpy()).max()
    sa.close()
    sh.close()
    a.close()


@pytest.mark.slow
def test_full_size_device_local_operators_c2():
    from vemgen.assemble import tet_class_input
    cfg = configs.CONFIGS["C2"]
    mesh = cfg.make_mesh()
    t0 = time.perf_counter()
    tin = [tet_class_input(mesh, c, cfg.k) for c in mesh.classes]
    t1 = time.perf_counter()
    s = cfg.build()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    a = pkg.Assembled(None, s.layout.n_u, s.layout.n_p, tets=tin)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    M, B, f = a.to_host()
    assert np.array_equal(M.indices, s.M.indices) and np.array_equal(B.indices, s.B.indices)
    assert np.abs(M.data - s.M.data).max() <= 1e-12 * np.abs(s.M.data).max()
    assert np.abs(f - s.f).max() <= 1e-12 * np.abs(s.f).max()
    print(f"C2: host inputs {t1 - t0:.2f} s, host assembly {t2 - t1:.2f} s, device local operators + "
          f"assembly {t4 - t3:.3f} s")
    a.close()
