"""The C-ABI library loads on a CPU-only host and exports every function that
include/vem_mixed.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vem_mixed.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vem_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("vem_mixed_upload", "vem_mixed_solve", "vem_mixed_solve_host", "vem_mixed_spmv",
                 "vem_mixed_precond_apply", "vem_mixed_destroy", "vem_status_string"):
        assert must in names


def test_library_exports_all_declared_symbols():
    from paper_1901_02330_b200 import build as b
    b.build()
    lib = ctypes.CDLL(b.LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    import paper_1901_02330_b200 as pkg
    assert set(pkg.EXPORTS) <= set(declared_functions())


def test_status_strings_without_gpu():
    import paper_1901_02330_b200 as pkg
    lib = pkg.load_library()
    assert lib.vem_status_string(0) == b"OK"
    assert lib.vem_status_string(-6) == b"ERR_INNER"


def test_binding_refuses_without_cuda():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import scipy.sparse as sp
    import paper_1901_02330_b200 as pkg
    M = sp.identity(3, format="csr")
    B = sp.csr_matrix(np.ones((1, 3)))
    with pytest.raises(pkg.VemError):
        pkg.VemMixed(M, B)
