"""Thin ctypes binding of include/vem_mixed.h (argument marshalling only).

Every step of the solve runs in libvem_mixed.so (sm_100a CUDA kernels).  There
is no CPU fallback: if the library or a CUDA device is missing, the calls raise.
PyTorch is used only for device memory and the current CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvem_mixed.so")

PRECOND_NONE = 0
PRECOND_BLOCK_SCHUR = 1
PRECOND_BLOCK_REG = 2
PRECOND_BLOCK_SCHUR_AMG = 3
PRECOND_BLOCK_SCHUR_AMG_F32 = 4
PRECOND_BLOCK_REG_M = 5

STATUS = {0: "OK", 1: "NOT_CONVERGED", 2: "BREAKDOWN", -1: "ERR_INVALID", -2: "ERR_DIAG_M",
          -3: "ERR_DIAG_S", -4: "ERR_CUDA", -5: "ERR_PRECOND", -6: "ERR_INNER"}

KCLASSES = ["spmv", "cheb", "pcg_spmv", "pcg_vec", "dot", "update", "precond_vec", "cycle", "mg_fine"]


class vem_csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("indptr", C.POINTER(C.c_int64)), ("indices", C.POINTER(C.c_int32)),
                ("values", C.POINTER(C.c_double))]


class vem_layout(C.Structure):
    _fields_ = [("k", C.c_int32), ("n_face_dof", C.c_int32), ("n_int_dof", C.c_int32),
                ("n_p_dof", C.c_int32), ("n_faces", C.c_int64), ("n_elems", C.c_int64)]


class vem_opts(C.Structure):
    _fields_ = [("restart", C.c_int32), ("cheb_degree", C.c_int32), ("cheb_ratio", C.c_double),
                ("inner_rtol", C.c_double), ("inner_maxit", C.c_int32), ("use_graphs", C.c_int32),
                ("timing", C.c_int32), ("pcg_chunk", C.c_int32), ("reorth", C.c_int32),
                ("l2_persist", C.c_int32), ("reorder", C.c_int32), ("inner_precond", C.c_int32),
                ("k_maxit", C.c_int32), ("k_rtol", C.c_double), ("k_inner_rtol", C.c_double),
                ("mg_chunk", C.c_int32), ("basis_f32", C.c_int32)]


class vem_solve_report(C.Structure):
    _fields_ = [("status", C.c_int32), ("iterations", C.c_int32), ("restarts", C.c_int32),
                ("converged", C.c_int32), ("breakdown", C.c_int32), ("cycles", C.c_int32),
                ("inner_iterations", C.c_int64), ("k_iterations", C.c_int64),
                ("rel_residual_true", C.c_double),
                ("rel_residual_est", C.c_double), ("setup_ms", C.c_double), ("solve_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class vem_info(C.Structure):
    _fields_ = [("n_u", C.c_int64), ("n_p", C.c_int64), ("nnz_M", C.c_int64), ("nnz_B", C.c_int64),
                ("nnz_A", C.c_int64), ("nnz_S", C.c_int64), ("lambda_max", C.c_double),
                ("eps", C.c_double), ("spmv_group", C.c_int32), ("schur_group", C.c_int32),
                ("sm_count", C.c_int32), ("device_bytes", C.c_int64), ("l2_window_bytes", C.c_int64),
                ("amg_levels", C.c_int32), ("amg_coarsest", C.c_int64), ("reordered", C.c_int32),
                ("amg_coarse_cluster", C.c_int32), ("nnz_A_stored", C.c_int64), ("nnz_S_stored", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_PI = C.POINTER(C.c_int32)
_PD = C.POINTER(C.c_double)


class vem_cell_class(C.Structure):
    _fields_ = [("n_cells", C.c_int64), ("n_loc", C.c_int32), ("n_p", C.c_int32), ("dof", _PI), ("pdof", _PI),
                ("n_t", C.c_int32), ("ti", _PI), ("tj", _PI), ("tA", _PD), ("tS", _PD), ("coef", _PD),
                ("n_b", C.c_int32), ("bi", _PI), ("bj", _PI), ("tB", _PD), ("Hinv", _PD), ("F", _PD),
                ("vol", _PD)]


class vem_tet_class(C.Structure):
    _fields_ = [("k", C.c_int32), ("n_cells", C.c_int64), ("cell", _PD), ("faces", _PD), ("signs", _PD),
                ("coef", _PD), ("dof", _PI), ("pdof", _PI), ("F", _PD), ("n_qv", C.c_int32), ("vref", _PD),
                ("n_qf", C.c_int32), ("fref", _PD), ("alphas1", _PD), ("betas", _PD), ("rgrad", _PD),
                ("rcross", _PD), ("dgrad", _PD), ("gens", _PD)]


class vem_kernel_stats(C.Structure):
    _fields_ = [("launches", C.c_int64 * 9), ("ms", C.c_double * 9), ("bytes", C.c_double * 9)]

    def as_dict(self):
        return {k: {"launches": int(self.launches[i]), "ms": float(self.ms[i]), "bytes": float(self.bytes[i])}
                for i, k in enumerate(KCLASSES)}


EXPORTS = ["vem_mixed_default_options", "vem_mixed_upload", "vem_mixed_solve", "vem_mixed_solve_host",
           "vem_mixed_assemble", "vem_mixed_assemble_tets", "vem_mixed_assembled_info", "vem_mixed_assembled_copy",
           "vem_mixed_upload_assembled", "vem_mixed_assembled_free",
           "vem_mixed_spmv", "vem_mixed_schur_spmv", "vem_mixed_precond_apply", "vem_mixed_set_options",
           "vem_mixed_get_options", "vem_mixed_get_info", "vem_mixed_get_schur", "vem_mixed_kernel_stats",
           "vem_mixed_amg_level", "vem_mixed_inner_amg_level", "vem_mixed_last_cycle_history",
           "vem_mixed_destroy", "vem_status_string", "vem_last_error"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libvem_mixed.so and declare the C signatures; raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    P = C.c_void_p
    D = C.POINTER(C.c_double)
    lib.vem_mixed_default_options.argtypes = [C.POINTER(vem_opts)]
    lib.vem_mixed_default_options.restype = None
    lib.vem_mixed_upload.argtypes = [C.POINTER(P), C.POINTER(vem_csr), C.POINTER(vem_csr), C.POINTER(vem_csr),
                                     C.c_double, C.POINTER(vem_layout), C.POINTER(vem_opts), P]
    lib.vem_mixed_solve.argtypes = [P, P, C.c_double, C.c_int32, C.c_int32, P, P, C.POINTER(vem_solve_report)]
    lib.vem_mixed_solve_host.argtypes = [P, D, C.c_double, C.c_int32, C.c_int32, D, D,
                                         C.POINTER(vem_solve_report)]
    lib.vem_mixed_spmv.argtypes = [P, P, P]
    lib.vem_mixed_schur_spmv.argtypes = [P, P, P]
    lib.vem_mixed_precond_apply.argtypes = [P, C.c_int32, P, P, C.POINTER(C.c_int64)]
    lib.vem_mixed_set_options.argtypes = [P, C.POINTER(vem_opts)]
    lib.vem_mixed_get_options.argtypes = [P, C.POINTER(vem_opts)]
    lib.vem_mixed_get_info.argtypes = [P, C.POINTER(vem_info)]
    lib.vem_mixed_get_schur.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int32), D]
    lib.vem_mixed_kernel_stats.argtypes = [P, C.POINTER(vem_kernel_stats), C.c_int32]
    lib.vem_mixed_amg_level.argtypes = [P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.vem_mixed_inner_amg_level.argtypes = [P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.vem_mixed_last_cycle_history.argtypes = [P, D, C.c_int32, C.POINTER(C.c_int32)]
    lib.vem_mixed_assemble.argtypes = [C.POINTER(P), C.POINTER(vem_cell_class), C.c_int32, C.c_int64, C.c_int64, P]
    lib.vem_mixed_assemble_tets.argtypes = [C.POINTER(P), C.POINTER(vem_tet_class), C.c_int32, C.c_int64,
                                            C.c_int64, P]
    lib.vem_mixed_assembled_info.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.vem_mixed_assembled_copy.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int32), D,
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int32), D, D]
    lib.vem_mixed_upload_assembled.argtypes = [C.POINTER(P), P, C.POINTER(vem_csr), C.c_double,
                                               C.POINTER(vem_layout), C.POINTER(vem_opts), P]
    lib.vem_mixed_assembled_free.argtypes = [P]
    lib.vem_mixed_assembled_free.restype = None
    lib.vem_mixed_destroy.argtypes = [P]
    lib.vem_mixed_destroy.restype = None
    lib.vem_status_string.argtypes = [C.c_int]
    lib.vem_status_string.restype = C.c_char_p
    lib.vem_last_error.argtypes = [P]
    lib.vem_last_error.restype = C.c_char_p
    for name in EXPORTS:
        if name not in ("vem_mixed_default_options", "vem_mixed_destroy", "vem_status_string",
                        "vem_last_error"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def default_options(**kw) -> vem_opts:
    o = vem_opts()
    load_library().vem_mixed_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _csr_struct(A):
    """scipy CSR -> (vem_csr, keepalive arrays); int64 indptr, int32 indices, fp64 values."""
    indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(A.indices, dtype=np.int32)
    values = np.ascontiguousarray(A.data, dtype=np.float64)
    s = vem_csr(A.shape[0], A.shape[1], int(values.size),
                indptr.ctypes.data_as(C.POINTER(C.c_int64)),
                indices.ctypes.data_as(C.POINTER(C.c_int32)),
                values.ctypes.data_as(C.POINTER(C.c_double)))
    return s, (indptr, indices, values)


def _dptr(t):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("expected a contiguous float64 CUDA tensor")
    return C.c_void_p(t.data_ptr())


class VemError(RuntimeError):
    pass


@dataclass
class SolveResult:
    u: object
    p: object
    report: dict


class VemMixed:
    """vem_mixed_upload / vem_mixed_solve on one CUDA device and stream."""

    def __init__(self, M, B, W=None, eps: float = 0.0, layout=None, opts: vem_opts | None = None,
                 stream=None):
        import torch
        self._lib = load_library()
        if not torch.cuda.is_available():
            raise VemError("no CUDA device: the VEM solver has no CPU path")
        self._stream = stream if stream is not None else torch.cuda.current_stream()
        ms, keep_m = _csr_struct(M)
        bs, keep_b = _csr_struct(B)
        ws, keep_w = (None, None)
        if W is not None:
            ws, keep_w = _csr_struct(W)
        lay = None
        if layout is not None:
            lay = vem_layout(layout.k, layout.n_face_dof, layout.n_int_dof, layout.n_p_dof,
                             layout.n_faces, layout.n_elems)
        self._h = C.c_void_p()
        rc = self._lib.vem_mixed_upload(C.byref(self._h), C.byref(ms), C.byref(bs),
                                        C.byref(ws) if ws is not None else None, float(eps),
                                        C.byref(lay) if lay is not None else None,
                                        C.byref(opts) if opts is not None else None,
                                        C.c_void_p(self._stream.cuda_stream))
        if rc != 0:
            raise VemError(f"vem_mixed_upload: {STATUS.get(rc, rc)}: "
                           f"{self._lib.vem_last_error(None).decode()}")
        self.n_u, self.n_p = M.shape[0], B.shape[0]
        self.n = self.n_u + self.n_p

    @classmethod
    def from_assembled(cls, asm, W=None, eps: float = 0.0, layout=None, opts: vem_opts | None = None,
                       stream=None):
        """vem_mixed_upload_assembled: the solver from a device-assembled system."""
        import torch
        self = cls.__new__(cls)
        self._lib = load_library()
        self._stream = stream if stream is not None else torch.cuda.current_stream()
        ws, keep_w = (None, None)
        if W is not None:
            ws, keep_w = _csr_struct(W)
        lay = None
        if layout is not None:
            lay = vem_layout(layout.k, layout.n_face_dof, layout.n_int_dof, layout.n_p_dof,
                             layout.n_faces, layout.n_elems)
        self._h = C.c_void_p()
        rc = self._lib.vem_mixed_upload_assembled(C.byref(self._h), asm._h,
                                                  C.byref(ws) if ws is not None else None, float(eps),
                                                  C.byref(lay) if lay is not None else None,
                                                  C.byref(opts) if opts is not None else None,
                                                  C.c_void_p(self._stream.cuda_stream))
        if rc != 0:
            self._h = None
            raise VemError(f"vem_mixed_upload_assembled: {STATUS.get(rc, rc)}: "
                           f"{self._lib.vem_last_error(None).decode()}")
        self.n_u, self.n_p = asm.n_u, asm.n_p
        self.n = self.n_u + self.n_p
        return self

    # -- helpers ---------------------------------------------------------
    def _check(self, rc, what, allow=(0,)):
        if rc not in allow:
            raise VemError(f"{what}: {STATUS.get(rc, rc)}: {self._lib.vem_last_error(self._h).decode()}")
        return rc

    def close(self):
        if getattr(self, "_h", None):
            self._lib.vem_mixed_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- API -------------------------------------------------------------
    def info(self) -> dict:
        i = vem_info()
        self._check(self._lib.vem_mixed_get_info(self._h, C.byref(i)), "get_info")
        return i.as_dict()

    def options(self) -> vem_opts:
        o = vem_opts()
        self._check(self._lib.vem_mixed_get_options(self._h, C.byref(o)), "get_options")
        return o

    def set_options(self, **kw):
        o = self.options()
        for k, v in kw.items():
            setattr(o, k, v)
        self._check(self._lib.vem_mixed_set_options(self._h, C.byref(o)), "set_options")

    def solve(self, rhs, tol=1e-10, maxit=10000, precond=PRECOND_BLOCK_SCHUR, out_u=None, out_p=None):
        """rhs: float64 CUDA tensor (n_u + n_p).  Returns SolveResult(u, p, report)."""
        import torch
        if out_u is None:
            out_u = torch.empty(self.n_u, dtype=torch.float64, device=rhs.device)
        if out_p is None:
            out_p = torch.empty(self.n_p, dtype=torch.float64, device=rhs.device)
        if rhs.numel() != self.n:
            raise ValueError("rhs has the wrong length")
        if out_u.numel() != self.n_u or out_p.numel() != self.n_p:
            raise ValueError("out_u / out_p must hold exactly n_u / n_p values")
        rep = vem_solve_report()
        rc = self._lib.vem_mixed_solve(self._h, _dptr(rhs), float(tol), int(maxit), int(precond),
                                       _dptr(out_u), _dptr(out_p), C.byref(rep))
        self._check(rc, "solve", allow=(0, 1, 2))
        d = rep.as_dict()
        d["status_name"] = STATUS.get(rc, str(rc))
        return SolveResult(out_u, out_p, d)

    def solve_host(self, rhs: np.ndarray, tol=1e-10, maxit=10000, precond=PRECOND_BLOCK_SCHUR,
                   u=None, p=None):
        """Host (numpy) buffers: the H2D/D2H copies happen inside the C call."""
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        if rhs.size != self.n:
            raise ValueError("rhs has the wrong length")
        u = np.empty(self.n_u) if u is None else u
        p = np.empty(self.n_p) if p is None else p
        for name, a, size in (("u", u, self.n_u), ("p", p, self.n_p)):
            # the C call writes 8 * size bytes through the raw pointer
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
                    and a.flags.writeable and a.size == size):
                raise ValueError(f"{name} must be a writeable C-contiguous float64 array of {size} values")
        rep = vem_solve_report()
        D = C.POINTER(C.c_double)
        rc = self._lib.vem_mixed_solve_host(self._h, rhs.ctypes.data_as(D), float(tol), int(maxit),
                                            int(precond), u.ctypes.data_as(D), p.ctypes.data_as(D),
                                            C.byref(rep))
        self._check(rc, "solve_host", allow=(0, 1, 2))
        d = rep.as_dict()
        d["status_name"] = STATUS.get(rc, str(rc))
        return SolveResult(u, p, d)

    def spmv(self, x, y=None):
        import torch
        y = torch.empty_like(x) if y is None else y
        self._check(self._lib.vem_mixed_spmv(self._h, _dptr(x), _dptr(y)), "spmv")
        return y

    def schur_spmv(self, x, y=None):
        import torch
        y = torch.empty_like(x) if y is None else y
        self._check(self._lib.vem_mixed_schur_spmv(self._h, _dptr(x), _dptr(y)), "schur_spmv")
        return y

    def precond_apply(self, kind, v, z=None):
        import torch
        z = torch.empty_like(v) if z is None else z
        its = C.c_int64(0)
        self._check(self._lib.vem_mixed_precond_apply(self._h, int(kind), _dptr(v), _dptr(z), C.byref(its)),
                    "precond_apply")
        return z, int(its.value)

    def get_schur(self):
        import scipy.sparse as sp
        i = self.info()
        indptr = np.empty(i["n_p"] + 1, dtype=np.int64)
        indices = np.empty(i["nnz_S"], dtype=np.int32)
        values = np.empty(i["nnz_S"], dtype=np.float64)
        self._check(self._lib.vem_mixed_get_schur(
            self._h, indptr.ctypes.data_as(C.POINTER(C.c_int64)), indices.ctypes.data_as(C.POINTER(C.c_int32)),
            values.ctypes.data_as(C.POINTER(C.c_double))), "get_schur")
        return sp.csr_matrix((values, indices, indptr), shape=(i["n_p"], i["n_p"]))

    def amg_levels(self):
        """[(rows, nnz)] of the S_D aggregation hierarchy (precond kind 3)."""
        out = []
        n, z = C.c_int64(), C.c_int64()
        for lev in range(self.info()["amg_levels"]):
            self._check(self._lib.vem_mixed_amg_level(self._h, lev, C.byref(n), C.byref(z)), "amg_level")
            out.append((n.value, z.value))
        return out

    def last_cycle_history(self) -> np.ndarray:
        """Givens residual estimates |g_{j+1}| / ||rhs|| of the last GMRES cycle of the last solve."""
        buf = np.zeros(128)
        cnt = C.c_int32(0)
        self._check(self._lib.vem_mixed_last_cycle_history(self._h, buf.ctypes.data_as(C.POINTER(C.c_double)), 128,
                                                           C.byref(cnt)), "last_cycle_history")
        return buf[:min(cnt.value, 128)].copy()

    def inner_amg_levels(self):
        """(rows, nnz) per level of the S_D + eps W hierarchy of the inner MG-PCG (R23)."""
        out = []
        n, z = C.c_int64(), C.c_int64()
        lev = 0
        while self._lib.vem_mixed_inner_amg_level(self._h, lev, C.byref(n), C.byref(z)) == 0:
            out.append((n.value, z.value))
            lev += 1
        return out

    def kernel_stats(self, reset=False) -> dict:
        s = vem_kernel_stats()
        self._check(self._lib.vem_mixed_kernel_stats(self._h, C.byref(s), 1 if reset else 0), "kernel_stats")
        return s.as_dict()


class Assembled:
    """vem_mixed_assemble: element-parallel device assembly of M, B and f from the
    per-class shape caches (vemgen.assemble.class_templates); marshalling only."""

    def __init__(self, templates, n_u: int, n_p: int, stream=None, tets=None):
        """templates: congruent-class shape caches (vemgen.assemble.class_templates);
        tets: inputs of single-tetrahedron classes (vemgen.assemble.tet_class_input),
        whose local operators are computed on the device."""
        import torch
        self._lib = load_library()
        if not torch.cuda.is_available():
            raise VemError("no CUDA device: the VEM assembly has no CPU path")
        stream = stream if stream is not None else torch.cuda.current_stream()
        self._keep = []
        if tets is not None:
            self._init_tets(tets, n_u, n_p, stream)
            return
        arr = (vem_cell_class * len(templates))()

        def i32(a):
            a = np.ascontiguousarray(a, dtype=np.int32)
            self._keep.append(a)
            return a.ctypes.data_as(_PI)

        def f64(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            self._keep.append(a)
            return a.ctypes.data_as(_PD)

        for q, t in enumerate(templates):
            E, nloc = t["L"].shape
            nk = t["P"].shape[1]
            arr[q] = vem_cell_class(E, nloc, nk, i32(t["L"]), i32(t["P"]), len(t["ii"]), i32(t["ii"]),
                                    i32(t["jj"]), f64(t["A"]), f64(t["S"]), f64(t["coef"]), len(t["bi"]),
                                    i32(t["bi"]), i32(t["bj"]), f64(t["B"]), f64(t["Hinv"]), f64(t["F"]),
                                    f64(t["vol"]))
        self._h = C.c_void_p()
        rc = self._lib.vem_mixed_assemble(C.byref(self._h), arr, len(templates), int(n_u), int(n_p),
                                          C.c_void_p(stream.cuda_stream))
        self._keep = []
        if rc != 0:
            self._h = None
            raise VemError(f"vem_mixed_assemble: {STATUS.get(rc, rc)}: {self._lib.vem_last_error(None).decode()}")
        self.n_u, self.n_p = int(n_u), int(n_p)

    def _init_tets(self, tets, n_u, n_p, stream):
        def i32(a):
            a = np.ascontiguousarray(a, dtype=np.int32)
            self._keep.append(a)
            return a.ctypes.data_as(_PI)

        def f64(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            self._keep.append(a)
            return a.ctypes.data_as(_PD)

        arr = (vem_tet_class * len(tets))()
        for q, t in enumerate(tets):
            arr[q] = vem_tet_class(t["k"], t["L"].shape[0], f64(t["cell"]), f64(t["faces"]), f64(t["signs"]),
                                   f64(t["coef"]), i32(t["L"]), i32(t["P"]), f64(t["F"]), t["vref"].shape[0],
                                   f64(t["vref"]), t["fref"].shape[0], f64(t["fref"]), f64(t["alphas1"]),
                                   f64(t["betas"]), f64(t["rgrad"]), f64(t["rcross"]), f64(t["dgrad"]),
                                   f64(t["gens"]) if t["gens"].size else None)
        self._h = C.c_void_p()
        rc = self._lib.vem_mixed_assemble_tets(C.byref(self._h), arr, len(tets), int(n_u), int(n_p),
                                               C.c_void_p(stream.cuda_stream))
        self._keep = []
        if rc != 0:
            self._h = None
            raise VemError(f"vem_mixed_assemble_tets: {STATUS.get(rc, rc)}: "
                           f"{self._lib.vem_last_error(None).decode()}")
        self.n_u, self.n_p = int(n_u), int(n_p)

    def nnz(self):
        m, b = C.c_int64(), C.c_int64()
        self._lib.vem_mixed_assembled_info(self._h, C.byref(m), C.byref(b))
        return m.value, b.value

    def to_host(self):
        """(M, B, f) as scipy CSR / numpy, copied back from the device."""
        import scipy.sparse as sp
        nm, nb = self.nnz()
        mrp, mci, mva = np.empty(self.n_u + 1, np.int64), np.empty(nm, np.int32), np.empty(nm)
        brp, bci, bva = np.empty(self.n_p + 1, np.int64), np.empty(nb, np.int32), np.empty(nb)
        f = np.empty(self.n_p)
        rc = self._lib.vem_mixed_assembled_copy(
            self._h, mrp.ctypes.data_as(C.POINTER(C.c_int64)), mci.ctypes.data_as(_PI), mva.ctypes.data_as(_PD),
            brp.ctypes.data_as(C.POINTER(C.c_int64)), bci.ctypes.data_as(_PI), bva.ctypes.data_as(_PD),
            f.ctypes.data_as(_PD))
        if rc != 0:
            raise VemError(f"vem_mixed_assembled_copy: {STATUS.get(rc, rc)}")
        M = sp.csr_matrix((mva, mci, mrp), shape=(self.n_u, self.n_u))
        B = sp.csr_matrix((bva, bci, brp), shape=(self.n_p, self.n_u))
        return M, B, f

    def close(self):
        if getattr(self, "_h", None):
            self._lib.vem_mixed_assembled_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
