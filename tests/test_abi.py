"""CPU tests of the C-ABI library: it loads without a GPU, exports every symbol declared in
include/hdiv.h, validates inputs before any device work, and its host-built 1D tables agree
with the oracle's independently constructed ones."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2304_12387_b200", "libhdiv.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2304_12387_b200 import build
        build.build()
    from paper_2304_12387_b200 import binding
    return binding.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hdiv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hdiv_[a-z_0-9]+)\s*\(", src)))


def test_all_declared_symbols_exported(lib):
    syms = declared_symbols()
    assert "hdiv_setup" in syms and "hdiv_minres_solve" in syms and len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"


def test_status_strings(lib):
    assert lib.hdiv_status_string(0) == b"ok"
    assert b"breakdown" in lib.hdiv_status_string(7).lower()
    assert lib.hdiv_version() >= 1


def _setup(lib, dim=3, N=(2, 2, 2), p=2, kind=0, alpha=None, beta=None, eps=None, gamma=None,
           slab=None, nranks=1, rank=0, verts=None, gvert=None, essential=0, kernel=0):
    from paper_2304_12387_b200 import binding as b
    z0, z1 = slab or (0, N[min(dim, 3) - 1])
    md = b.MeshDesc(dim, N[0], N[1], N[2] if dim == 3 else 1, z0, z1,
                    None if verts is None else verts.ctypes.data_as(C.POINTER(C.c_double)))
    keep = []

    def ptr(a):
        if a is None:
            return None
        a = np.ascontiguousarray(a, float)
        keep.append(a)
        return a.ctypes.data_as(C.POINTER(C.c_double))
    co = b.Coeffs(ptr(alpha), ptr(beta), ptr(gamma), ptr(eps), 1.0, 1.0, 0.0, 1.0, ptr(gvert))
    op = b.Options(1.0, 4, 30.0, kernel, 0, 0, 0, essential, 0)
    h = C.c_void_p()
    st = lib.hdiv_setup(C.byref(md), p, C.byref(co), kind, C.byref(op), None, rank, nranks, None,
                        C.byref(h))
    return st, h


def test_setup_validation_before_device_work(lib):
    # these all fail in host validation (no CUDA call is made, so they run without a GPU)
    assert _setup(lib, p=0)[0] == 1                                 # INVALID_ORDER
    assert _setup(lib, p=7)[0] == 1
    assert _setup(lib, dim=4)[0] == 4                               # SHAPE
    assert _setup(lib, N=(0, 2, 2))[0] == 2                         # INVALID_MESH
    assert _setup(lib, slab=(1, 2))[0] == 2                         # single rank must own all
    assert _setup(lib, alpha=-np.ones(8))[0] == 3                   # COEFFICIENT
    assert _setup(lib, kind=1, eps=np.ones(8), gamma=-np.ones(8))[0] == 3
    assert _setup(lib, nranks=2)[0] == 9                            # NULL nccl id
    # inverted box element
    from synth import cartesian_vertices
    V = cartesian_vertices(3, (2, 2, 2))[:, :, ::-1, :].copy()
    assert _setup(lib, verts=V)[0] == 2
    # unsupported combinations, rejected before device work: the general (vertex-field) gamma
    # in 2D (NEXT-3, 3D only), the affine tile kernel forced on a non-box mesh
    from synth import cartesian_vertices as cv
    V2 = cv(2, (2, 2)).copy()
    V2[1, 1] += [0.1, 0.05]
    assert _setup(lib, dim=2, N=(2, 2, 1), kind=1, eps=np.ones(4), gvert=np.ones(9))[0] == 8
    assert _setup(lib, dim=2, N=(2, 2, 1), verts=V2, alpha=np.ones(4), beta=np.ones(4),
                  kernel=2)[0] == 8
    # essential_sides beyond the 2 dim side bits -> SHAPE
    assert _setup(lib, dim=2, N=(2, 2, 1), essential=16)[0] == 4
    assert _setup(lib, essential=64)[0] == 4


@pytest.mark.parametrize("p", range(1, 7))
def test_library_tables_match_oracle(lib, p):
    """Independent constructions (library: GLL as roots of P_{p+1}-P_{p-1}, Newton GL,
    barycentric l, h = -cumsum l'; oracle: Newton on P_p', leggauss, product-form l,
    histopolation DOF solve) agree to round-off."""
    from paper_2304_12387_b200.binding import debug_tables
    from oracle import basis1d
    t = debug_tables(p)
    xq, wq = basis1d.gl_rule(p + 2)
    assert np.allclose(t["xq"], xq, atol=1e-15) and np.allclose(t["wq"], wq, atol=1e-15)
    Bl = basis1d.lagrange(basis1d.gll_nodes(p), xq)
    Bh = basis1d.histopolation(p, xq)
    assert np.abs(t["Bl"] - Bl).max() < 1e-13
    assert np.abs(t["Bh"] - Bh).max() < 1e-11 * max(1, np.abs(Bh).max())
    Ml, Mh = basis1d.mass_1d(p)
    assert np.abs(t["Ml"] - Ml).max() < 1e-14
    assert np.abs(t["Mh"] - Mh).max() < 1e-12 * np.abs(Mh).max()
    assert np.abs(t["Mhinv"] @ Mh - np.eye(p)).max() < 1e-12


@pytest.mark.parametrize("p", range(1, 7))
def test_library_gl_tables(lib, p):
    """Tables of the W^-1 local CG (NEXT-2): the GL-nodal basis spans the same Q_{p-1} as the
    histopolation basis, so B_G = B_h HG; and with the exact Q-point rule the GL-nodal mass is
    diagonal (the GL weights), so HG W_g^-1 HG^T equals the oracle's M_h^-1."""
    from paper_2304_12387_b200.binding import debug_gl_tables
    from oracle import basis1d
    g = debug_gl_tables(p)
    xq, wq = basis1d.gl_rule(p + 2)
    Bh = basis1d.histopolation(p, xq)
    assert np.abs(g["BG"] - Bh @ g["HG"]).max() < 1e-12
    Wg = g["BG"].T @ np.diag(wq) @ g["BG"]
    assert np.abs(Wg - np.diag(np.diag(Wg))).max() < 1e-13
    Mh = Bh.T @ np.diag(wq) @ Bh
    assert np.abs(g["HG"] @ np.linalg.inv(Wg) @ g["HG"].T - np.linalg.inv(Mh)).max() < 1e-9
