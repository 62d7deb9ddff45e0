"""Thin ctypes binding of libhdiv (include/hdiv.h).  Argument marshalling only: every step
of the hot path runs in the CUDA kernels of libhdiv.so.  PyTorch provides device memory and
streams.  There is NO CPU fallback: if the library is missing this module raises."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhdiv.so")

GRAD_DIV, DARCY = 0, 1
STATUS = {0: "ok", 1: "invalid order", 2: "invalid mesh", 3: "coefficient error",
          4: "shape error", 5: "CUDA error", 6: "NCCL error", 7: "MINRES breakdown",
          8: "unsupported", 9: "null argument"}


class HdivError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"hdiv status {code} ({STATUS.get(code, '?')}): {msg}")
        self.code = code


class MeshDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("ez_begin", C.c_int64), ("ez_end", C.c_int64),
                ("vertices", C.POINTER(C.c_double))]


class Coeffs(C.Structure):
    _fields_ = [("alpha", C.POINTER(C.c_double)), ("beta", C.POINTER(C.c_double)),
                ("gamma", C.POINTER(C.c_double)), ("eps", C.POINTER(C.c_double)),
                ("alpha0", C.c_double), ("beta0", C.c_double), ("gamma0", C.c_double),
                ("eps0", C.c_double), ("gamma_vertex", C.POINTER(C.c_double))]


class Options(C.Structure):
    _fields_ = [("tau", C.c_double), ("cheb_degree", C.c_int), ("cheb_ratio", C.c_double),
                ("kernel", C.c_int), ("schur_solver", C.c_int), ("amg_sweeps", C.c_int),
                ("amg_max_coarse", C.c_int), ("essential_sides", C.c_int),
                ("project_mean", C.c_int), ("tri_geometry", C.c_int),
                ("amg_cheb_degree", C.c_int), ("amg_cheb_ratio", C.c_double),
                ("amg_global_coarse", C.c_int)]


SCHUR_SOLVERS = {"chebyshev": 0, "amg": 1, "auto": 2}


class Report(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("rel_resid", C.c_double),
                ("t_solve_ms", C.c_double)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libhdiv.so; raises if absent (the product has no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libhdiv.so not built at {path}: run __graft_entry__.build()")
    lib = C.CDLL(path)
    vp, dp, i64p = C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)
    sig = {
        "hdiv_setup": (C.c_int, [C.POINTER(MeshDesc), C.c_int, C.POINTER(Coeffs), C.c_int,
                                 C.POINTER(Options), vp, C.c_int, C.c_int, vp, C.POINTER(vp)]),
        "hdiv_destroy": (None, [vp]),
        "hdiv_status_string": (C.c_char_p, [C.c_int]),
        "hdiv_last_error": (C.c_char_p, []),
        "hdiv_version": (C.c_int, []),
        "hdiv_sizes": (C.c_int, [vp, i64p, i64p, i64p, i64p]),
        "hdiv_apply_mass": (C.c_int, [vp, dp, dp, vp]),
        "hdiv_apply_div": (C.c_int, [vp, dp, dp, vp]),
        "hdiv_apply_divT": (C.c_int, [vp, dp, dp, vp]),
        "hdiv_apply_block": (C.c_int, [vp, dp, dp, vp]),
        "hdiv_apply_block_host": (C.c_int, [vp, dp, dp, vp]),
        "hdiv_apply_launches": (C.c_int, [vp, C.POINTER(C.c_int)]),
        "hdiv_assemble_mass_diag": (C.c_int, [vp, dp, vp]),
        "hdiv_assemble_schur_diag_term": (C.c_int, [vp, dp, vp]),
        "hdiv_schur_nnz": (C.c_int, [vp, i64p]),
        "hdiv_assemble_schur_csr": (C.c_int, [vp, dp, dp, dp, vp]),
        "hdiv_apply_schur": (C.c_int, [vp, dp, dp, vp]),
        "hdiv_export_div_csr": (C.c_int, [vp, dp, dp, dp, vp]),
        "hdiv_apply_precond": (C.c_int, [vp, dp, dp, vp]),
        "hdiv_minres_solve": (C.c_int, [vp, dp, dp, C.c_double, C.c_int, C.POINTER(Report), vp]),
        "hdiv_debug_tables": (C.c_int, [C.c_int, C.c_int] + [dp] * 7),
        "hdiv_debug_gl_tables": (C.c_int, [C.c_int, C.c_int, dp, dp]),
        "hdiv_amg_levels": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
        "hdiv_apply_z": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "hdiv_apply_precond_tri": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "hdiv_gmres_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                       C.c_int, C.POINTER(Report), C.c_void_p]),
        "hdiv_amg_level": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_void_p,
                                     C.c_void_p]),
        "hdiv_nccl_unique_id": (C.c_int, [vp, C.c_int64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(code: int):
    if code != 0:
        msg = _lib.hdiv_last_error().decode()
        raise HdivError(code, msg)


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from the library (rank 0 creates it and broadcasts the bytes)."""
    lib = load_library()
    buf = C.create_string_buffer(128)
    _check(lib.hdiv_nccl_unique_id(C.cast(buf, C.c_void_p), 128))
    return buf.raw


def loopback_id(key: int) -> bytes:
    """Communicator id of a LOOPBACK slab group (single-GPU tests of the multi-rank path): the P
    ranks live in one process, one host thread each, and exchange by device-to-device copies
    (libhdiv comm.cu); `key` names the group."""
    return b"HDIVLOOP" + int(key).to_bytes(8, "little") + bytes(112)


def debug_tables(p: int, Q: int = 0) -> dict:
    """Host-only: the library's 1D tables (no GPU needed)."""
    lib = load_library()
    Q = Q or p + 2
    out = {"xq": np.zeros(Q), "wq": np.zeros(Q), "Bl": np.zeros((Q, p + 1)),
           "Bh": np.zeros((Q, p)), "Ml": np.zeros((p + 1, p + 1)), "Mh": np.zeros((p, p)),
           "Mhinv": np.zeros((p, p))}
    _check(lib.hdiv_debug_tables(p, Q, *[C.c_void_p(out[k].ctypes.data) for k in
                                         ("xq", "wq", "Bl", "Bh", "Ml", "Mh", "Mhinv")]))
    return out


def debug_gl_tables(p: int, Q: int = 0) -> dict:
    """Host-only: the Gauss-Legendre nodal tables of the W^-1 local CG (no GPU needed)."""
    lib = load_library()
    Q = Q or p + 2
    out = {"BG": np.zeros((Q, p)), "HG": np.zeros((p, p))}
    _check(lib.hdiv_debug_gl_tables(p, Q, C.c_void_p(out["BG"].ctypes.data),
                                    C.c_void_p(out["HG"].ctypes.data)))
    return out


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class Sizes:
    n_rt: int
    n_l2: int
    n_rt_global: int
    n_l2_global: int

    @property
    def n(self):
        return self.n_rt + self.n_l2


class HdivOperator:
    """Handle on one discretised problem (one rank's slab).  Vectors are torch CUDA fp64
    tensors in the canonical numbering."""

    def __init__(self, dim, N, p, kind, vertices=None, alpha=None, beta=None, gamma=None,
                 eps=None, gamma_vertex=None, tau=1.0, cheb_degree=4, cheb_ratio=30.0, kernel=0,
                 schur="auto", amg_sweeps=2, amg_max_coarse=512, essential=0,
                 project_mean=False, tri_geometry=0, amg_cheb_degree=0, amg_cheb_ratio=20.0,
                 amg_global_coarse=0,
                 slab=None, nccl_id: Optional[bytes] = None, rank=0, nranks=1, stream=None):
        import torch
        self.lib = load_library()
        self._torch = torch
        N = tuple(int(n) for n in N) + (1,) * (3 - len(N))
        last = dim - 1
        z0, z1 = slab if slab is not None else (0, N[last])
        self._keep = []

        def arr(a):
            if a is None:
                return None
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
            self._keep.append(a)
            return a

        V = arr(vertices)
        md = MeshDesc(dim, N[0], N[1], N[2] if dim == 3 else 1, z0, z1, _dptr(V))
        a_, b_, g_, e_ = arr(alpha), arr(beta), arr(gamma), arr(eps)
        gv_ = arr(gamma_vertex)
        co = Coeffs(_dptr(a_), _dptr(b_), _dptr(g_), _dptr(e_), 1.0, 1.0, 0.0, 1.0, _dptr(gv_))
        op = Options(tau, cheb_degree, cheb_ratio, kernel, SCHUR_SOLVERS[schur], amg_sweeps,
                     amg_max_coarse, int(essential), int(bool(project_mean)), int(tri_geometry),
                     int(amg_cheb_degree), float(amg_cheb_ratio), int(amg_global_coarse))
        h = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), len(nccl_id))
        s = self._stream_handle(stream)
        kind_i = GRAD_DIV if kind in ("grad_div", GRAD_DIV) else DARCY
        _check(self.lib.hdiv_setup(C.byref(md), int(p), C.byref(co), kind_i, C.byref(op),
                                   C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                                   rank, nranks, s, C.byref(h)))
        self.h = h
        self._keep = []
        self.dim, self.N, self.p, self.kind = dim, N, p, kind
        a = [C.c_int64() for _ in range(4)]
        _check(self.lib.hdiv_sizes(h, *[C.byref(x) for x in a]))
        self.sizes = Sizes(*[x.value for x in a])

    # -- helpers --------------------------------------------------------------------
    def _stream_handle(self, stream):
        torch = self._torch
        if stream is None:
            if not torch.cuda.is_available():
                return None
            stream = torch.cuda.current_stream()
        return C.c_void_p(stream.cuda_stream)

    def _ptr(self, t, n=None):
        torch = self._torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                and t.is_contiguous()):
            raise TypeError("expected a contiguous CUDA float64 tensor")
        if n is not None and t.numel() != n:
            raise ValueError(f"expected {n} entries, got {t.numel()}")
        return C.c_void_p(t.data_ptr())

    def empty(self, n):
        return self._torch.empty(n, dtype=self._torch.float64, device="cuda")

    # -- applies --------------------------------------------------------------------
    def apply_mass(self, u, y=None, stream=None):
        s = self.sizes
        y = self.empty(s.n_rt) if y is None else y
        _check(self.lib.hdiv_apply_mass(self.h, self._ptr(u, s.n_rt), self._ptr(y, s.n_rt),
                                        self._stream_handle(stream)))
        return y

    def apply_div(self, u, y=None, stream=None):
        s = self.sizes
        y = self.empty(s.n_l2) if y is None else y
        _check(self.lib.hdiv_apply_div(self.h, self._ptr(u, s.n_rt), self._ptr(y, s.n_l2),
                                       self._stream_handle(stream)))
        return y

    def apply_divT(self, q, y=None, stream=None):
        s = self.sizes
        y = self.empty(s.n_rt) if y is None else y
        _check(self.lib.hdiv_apply_divT(self.h, self._ptr(q, s.n_l2), self._ptr(y, s.n_rt),
                                        self._stream_handle(stream)))
        return y

    def apply_z(self, q, y=None, stream=None):
        """y = Z q, the (2,2) block alone (3D; element-local CG for W^-1)."""
        s = self.sizes
        y = self.empty(s.n_l2) if y is None else y
        _check(self.lib.hdiv_apply_z(self.h, self._ptr(q, s.n_l2), self._ptr(y, s.n_l2),
                                     self._stream_handle(stream)))
        return y

    def apply_block(self, x, y=None, stream=None):
        s = self.sizes
        y = self.empty(s.n) if y is None else y
        _check(self.lib.hdiv_apply_block(self.h, self._ptr(x, s.n), self._ptr(y, s.n),
                                         self._stream_handle(stream)))
        return y

    def apply_block_host(self, x_host: "np.ndarray | object", y_host, stream=None):
        """x_host/y_host: host arrays (numpy or pinned torch CPU tensors) of length n.
        The library copies n doubles out of / into them, so both must be fp64, C-contiguous,
        CPU-resident and exactly n long (checked here; anything else raises)."""
        n = self.sizes.n

        def hp(a, name):
            if hasattr(a, "data_ptr"):   # torch tensor
                import torch
                if a.device.type != "cpu" or a.dtype != torch.float64 or not a.is_contiguous() \
                        or a.numel() != n:
                    raise ValueError(f"{name}: need a contiguous CPU float64 tensor of {n} "
                                     f"elements, got {a.dtype} {tuple(a.shape)} on {a.device}")
                return C.c_void_p(a.data_ptr())
            if not isinstance(a, np.ndarray) or a.dtype != np.float64 or \
                    not a.flags["C_CONTIGUOUS"] or a.size != n:
                raise ValueError(f"{name}: need a C-contiguous float64 numpy array of {n} "
                                 f"elements")
            if name == "y_host" and not a.flags["WRITEABLE"]:
                raise ValueError("y_host is read-only")
            return C.c_void_p(a.ctypes.data)
        px, py = hp(x_host, "x_host"), hp(y_host, "y_host")
        _check(self.lib.hdiv_apply_block_host(self.h, px, py, self._stream_handle(stream)))
        return y_host

    def apply_launches(self) -> int:
        n = C.c_int()
        _check(self.lib.hdiv_apply_launches(self.h, C.byref(n)))
        return n.value

    def mass_diag(self, stream=None):
        y = self.empty(self.sizes.n_rt)
        _check(self.lib.hdiv_assemble_mass_diag(self.h, self._ptr(y), self._stream_handle(stream)))
        return y

    def schur_diag_term(self, stream=None):
        y = self.empty(self.sizes.n_l2)
        _check(self.lib.hdiv_assemble_schur_diag_term(self.h, self._ptr(y),
                                                      self._stream_handle(stream)))
        return y

    def schur_csr(self, stream=None):
        torch = self._torch
        nnz = C.c_int64()
        _check(self.lib.hdiv_schur_nnz(self.h, C.byref(nnz)))
        n = self.sizes.n_l2
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(nnz.value, dtype=torch.int64, device="cuda")
        val = torch.empty(nnz.value, dtype=torch.float64, device="cuda")
        _check(self.lib.hdiv_assemble_schur_csr(self.h, C.c_void_p(rp.data_ptr()),
                                                C.c_void_p(col.data_ptr()),
                                                C.c_void_p(val.data_ptr()),
                                                self._stream_handle(stream)))
        return rp, col, val

    def apply_schur(self, x, y=None, stream=None):
        n = self.sizes.n_l2
        y = self.empty(n) if y is None else y
        _check(self.lib.hdiv_apply_schur(self.h, self._ptr(x, n), self._ptr(y, n),
                                         self._stream_handle(stream)))
        return y

    def div_csr(self, stream=None):
        torch = self._torch
        n = self.sizes.n_l2
        nd = 2 * self.dim
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(nd * n, dtype=torch.int64, device="cuda")
        val = torch.empty(nd * n, dtype=torch.float64, device="cuda")
        _check(self.lib.hdiv_export_div_csr(self.h, C.c_void_p(rp.data_ptr()),
                                            C.c_void_p(col.data_ptr()),
                                            C.c_void_p(val.data_ptr()),
                                            self._stream_handle(stream)))
        return rp, col, val

    def apply_precond(self, v, z=None, stream=None):
        n = self.sizes.n
        z = self.empty(n) if z is None else z
        _check(self.lib.hdiv_apply_precond(self.h, self._ptr(v, n), self._ptr(z, n),
                                           self._stream_handle(stream)))
        return z

    def minres(self, b, x=None, rtol=1e-12, maxit=1000, stream=None):
        n = self.sizes.n
        x = self.empty(n) if x is None else x
        rep = Report()
        _check(self.lib.hdiv_minres_solve(self.h, self._ptr(b, n), self._ptr(x, n), rtol, maxit,
                                          C.byref(rep), self._stream_handle(stream)))
        return x, rep

    def apply_precond_tri(self, v, z=None, stream=None):
        """z = B^-1 v, B = [tau M~, D^T; 0, -S^] (NEXT-4)."""
        n = self.sizes.n
        z = self.empty(n) if z is None else z
        _check(self.lib.hdiv_apply_precond_tri(self.h, self._ptr(v, n), self._ptr(z, n),
                                               self._stream_handle(stream)))
        return z

    def gmres(self, b, x=None, rtol=1e-12, maxit=1000, restart=30, stream=None):
        """Right-preconditioned GMRES(restart) with the block-triangular preconditioner."""
        n = self.sizes.n
        x = self.empty(n) if x is None else x
        rep = Report()
        _check(self.lib.hdiv_gmres_solve(self.h, self._ptr(b, n), self._ptr(x, n), rtol, maxit,
                                         restart, C.byref(rep), self._stream_handle(stream)))
        return x, rep

    def amg_levels(self) -> int:
        n = C.c_int()
        _check(self.lib.hdiv_amg_levels(self.h, C.byref(n)))
        return n.value

    def amg_level(self, level: int):
        """(dims, omega, stencil) of AMG level `level`; stencil [3^d][n] (None for level 0)."""
        torch = self._torch
        dims = (C.c_int64 * 3)()
        n, om = C.c_int64(), C.c_double()
        _check(self.lib.hdiv_amg_level(self.h, level, dims, C.byref(n), C.byref(om), None, None))
        st = None
        if level > 0:
            ns = 27 if self.dim == 3 else 9
            st = torch.empty((ns, n.value), dtype=torch.float64, device="cuda")
            _check(self.lib.hdiv_amg_level(self.h, level, dims, C.byref(n), C.byref(om),
                                           C.c_void_p(st.data_ptr()),
                                           self._stream_handle(None)))
        return tuple(dims), om.value, st

    def close(self):
        if getattr(self, "h", None):
            self.lib.hdiv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def from_problem(prob, **kw) -> HdivOperator:
    """Build an operator from a synth.Problem (inputs only)."""
    kw.setdefault("essential", getattr(prob, "essential", 0))
    kw.setdefault("gamma_vertex", getattr(prob, "gamma_vertex", None))
    kw.setdefault("project_mean", getattr(prob, "project_mean", False))
    return HdivOperator(prob.dim, prob.N, prob.p, prob.kind, vertices=prob.vertices,
                        alpha=prob.alpha, beta=prob.beta, gamma=prob.gamma, eps=prob.eps, **kw)
