"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle, element by element, on the
same seeded inputs (north_star bars: D / CSR structure bit-exact; applies and diagonals 1e-12
relative per block; S~ values 1e-10; MINRES iteration counts +-1)."""
import numpy as np
import pytest

from synth import make_config, random_vector, Problem, cartesian_vertices, graded_two_material

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _rel(a, b):
    d = np.abs(np.asarray(a) - np.asarray(b)).max()
    s = np.abs(np.asarray(b)).max()
    return d / s if s > 0 else d


def _gpu(prob, **kw):
    from paper_2304_12387_b200 import from_problem
    kw.setdefault("amg_cheb_degree", 1)   # the oracle's BlockDiagPrecond default (plain V-cycle)
    return from_problem(prob, **kw)


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


# small cases spanning several tiles with ragged tails (tile sizes: p1 8^3, p2 8x8x4,
# p3 4^3, p4 4x4x2, p5 4x2x2, p6 2^3)
CASES = [
    ("c1", None, None, 0),                 # 2D 4x4 p=2 Darcy (config 1), general kernel
    ("c1", (5, 3), 3, 0),                  # 2D ragged
    ("c2", (3, 2, 2), 3, 0),               # 3D box, affine tile kernel
    ("c2", (5, 3, 6), 2, 0),
    ("c2", (9, 5, 3), 1, 0),
    ("c2", (5, 3, 3), 4, 0),
    ("c2", (5, 3, 3), 5, 0),
    ("c2", (3, 3, 3), 6, 0),
    ("c2", (5, 3, 3), 4, 1),               # same, forced general kernel
    ("c3", (3, 2, 3), 2, 0),               # trilinear Darcy gamma = 0, general kernel
    ("c3", (2, 3, 2), 4, 0),
    ("c3", (3, 2, 2), 3, 0),               # odd orders: padded layouts differ (U0 largest)
    ("c3", (3, 3, 2), 1, 0),
    ("c3", (2, 2, 2), 5, 0),
    ("c5", (5, 5, 3), 3, 0),               # graded two-material, box kernel
    ("c3gd", (3, 2, 2), 2, 0),             # trilinear grad-div: W_alpha^-1 by the local CG
    ("c3gd", (2, 2, 3), 4, 0),
    ("c3gd", (2, 2, 2), 6, 0),
    ("c3gd", (2, 3, 2), 1, 0),
    ("c3gd", (2, 2, 2), 5, 0),
    ("c3g", (3, 2, 2), 3, 0),              # trilinear Darcy gamma > 0 (config 3b)
    ("c3g", (2, 2, 2), 5, 0),
]


def _problem(name, N, p):
    if name in ("c3gd", "c3g"):   # config-3 meshes with a nonzero (2,2) block (NEXT-2)
        pr = make_config("c3", N=N, p=p)
        if name == "c3gd":
            pr.kind = "grad_div"
            pr.alpha = 10.0 ** random_vector(pr.E, 33)
            pr.beta = 10.0 ** random_vector(pr.E, 34)
        else:
            pr.gamma = 10.0 ** random_vector(pr.E, 35)
        return pr
    pr = make_config(name, N=N, p=p)
    if name == "c2":   # heterogeneous coefficients so per-element weights matter
        pr.alpha = 10.0 ** random_vector(pr.E, 31)
        pr.beta = 10.0 ** random_vector(pr.E, 32)
    return pr


# box kernel (one production tile per order): ragged tiles on every axis, single-element meshes,
# graded two-material meshes
VARIANTS = [("c2", (5, 3, 7), 4, {}), ("c2", (4, 6, 4), 3, {}), ("c2", (6, 4, 6), 5, {}),
            ("c2", (5, 4, 6), 2, {}), ("c2", (3, 3, 4), 6, {}), ("c2", (9, 5, 5), 1, {}),
            ("c2", (10, 10, 6), 1, {}), ("c2", (9, 9, 5), 2, {}), ("c5", (5, 5, 6), 3, {}),
            ("c5", (6, 6, 4), 5, {}), ("c5", (5, 5, 3), 6, {}), ("c2", (1, 1, 1), 4, {}),
            ("c2", (1, 2, 1), 5, {}), ("c2", (2, 1, 1), 6, {})]


@pytest.mark.parametrize("name,N,p,env", VARIANTS)
def test_box_kernel_variants(name, N, p, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from oracle import operators
    pr = _problem(name, N, p)
    A = operators.Assembled(pr, with_schur=False)
    op = _gpu(pr)
    s = op.sizes
    x = random_vector(s.n, 17)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL
    assert _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    u = x[:s.n_rt]
    assert _rel(_host(op.apply_mass(_dev(u))), A.M @ u) < TOL


@pytest.mark.parametrize("name,N,p,kernel", CASES)
def test_block_apply_parity(name, N, p, kernel):
    from oracle import operators
    pr = _problem(name, N, p)
    A = operators.Assembled(pr, with_schur=False)
    op = _gpu(pr, kernel=kernel)
    s = op.sizes
    assert (s.n_rt, s.n_l2) == (A.n_rt, A.n_l2)
    x = random_vector(s.n, 7)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL
    assert _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    # the Z q~ term alone (u = 0), measured separately
    x0 = x.copy()
    x0[:s.n_rt] = 0
    y0 = _host(op.apply_block(_dev(x0)))
    yo0 = A.apply_block(x0)
    assert _rel(y0[s.n_rt:], yo0[s.n_rt:]) < TOL
    # mass, D, D^T separately
    u = x[:s.n_rt]
    q = x[s.n_rt:]
    assert _rel(_host(op.apply_mass(_dev(u))), A.M @ u) < TOL
    assert np.array_equal(_host(op.apply_div(_dev(u))), A.D @ u) or \
        _rel(_host(op.apply_div(_dev(u))), A.D @ u) < 1e-15
    assert _rel(_host(op.apply_divT(_dev(q))), A.D.T @ q) < 1e-15
    # determinism: bitwise identical repeat
    y2 = _host(op.apply_block(_dev(x)))
    assert np.array_equal(y, y2)


@pytest.mark.parametrize("name,N,p,kernel", CASES[:8] + CASES[9:])
def test_setup_objects_parity(name, N, p, kernel):
    """diag(M) (1e-12), C~, D CSR (bit-exact), S~ CSR structure (bit-exact) and values (1e-10)."""
    from oracle import operators
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    op = _gpu(pr, kernel=kernel)
    assert _rel(_host(op.mass_diag()), A.Mdiag) < TOL
    assert _rel(_host(op.schur_diag_term()), A.Ctil) < TOL
    rp, col, val = [_host(t) for t in op.div_csr()]
    assert np.array_equal(rp, A.Dptr) and np.array_equal(col, A.Dcol)
    assert np.array_equal(val, A.Dval)
    rp, col, val = [_host(t) for t in op.schur_csr()]
    S = A.S.tocsr()
    S.sort_indices()
    assert np.array_equal(rp, S.indptr) and np.array_equal(col, S.indices)
    assert _rel(val, S.data) < 1e-10
    xq = random_vector(A.n_l2, 5)
    assert _rel(_host(op.apply_schur(_dev(xq))), S @ xq) < 1e-12


@pytest.mark.parametrize("name,N,p", [("c1", None, None), ("c2", (2, 2, 2), 2),
                                      ("c3", (2, 2, 2), 2), ("c2", (3, 2, 2), 3),
                                      ("c3gd", (2, 2, 2), 3), ("c3g", (2, 2, 2), 2)])
def test_preconditioner_and_minres_parity(name, N, p):
    from oracle import operators, solvers
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    op = _gpu(pr, tau=1.0, cheb_degree=4, cheb_ratio=30.0)
    n = A.n_rt + A.n_l2
    v = random_vector(n, 3)
    P = solvers.BlockDiagPrecond(A, tau=1.0, degree=4, ratio=30.0)
    z = _host(op.apply_precond(_dev(v)))
    zo = P.apply(v)
    assert _rel(z[:A.n_rt], zo[:A.n_rt]) < TOL
    assert _rel(z[A.n_rt:], zo[A.n_rt:]) < 1e-11
    xs = random_vector(n, 1)
    b = A.apply_block(xs)
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=2000)
    x, rep = op.minres(_dev(b), rtol=1e-12, maxit=2000)
    x = _host(x)
    assert conv_o and rep.converged
    assert abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    assert _rel(x, xo) < 1e-9


def test_config2_minres_full():
    """Config 2 (8^3, p=3, grad-div): MINRES to 1e-12, iteration count within +-1 of the oracle,
    solution against the known x*."""
    from oracle import operators, solvers
    pr = make_config("c2")
    A = operators.Assembled(pr)
    n = A.n_rt + A.n_l2
    xs = random_vector(n, 2)
    b = A.apply_block(xs)
    P = solvers.BlockDiagPrecond(A)
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=3000)
    op = _gpu(pr)
    x, rep = op.minres(_dev(b), rtol=1e-12, maxit=3000)
    assert rep.converged and conv_o
    assert abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    assert _rel(_host(x), xs) < 1e-7


# full BASELINE sizes + the bench's p sweep sizes (bench.py `sweep`: N = 160/128/128/96/80 for
# p = 2..6), each in the launch configuration bench.py times
FULL_CASES = [("c4", 4, None), ("c3", 4, None), ("c3gv", 4, None),
              ("c4", 2, 160), ("c4", 3, 128), ("c4", 5, 96), ("c4", 6, 80),
              # config 5b's size (128^3, p = 6): 1.81e9 DOFs, S~ with 3.2e9 nonzeros (> 2^31: the
              # int64 row pointers of the setup's scan and every 64-bit index of the apply)
              ("c4", 6, 128)]


@pytest.mark.parametrize("name,p,Nn", FULL_CASES)
def test_full_size_sampled_parity(name, p, Nn):
    """BASELINE full sizes (config 4: 128^3 p=4 grad-div; config 3: 64^3 p=4 perturbed Darcy;
    config 3b with a general vertex-field gamma, NEXT-3) and the bench's p = 2, 3, 5, 6 sweep
    meshes, in the launch configuration bench.py times; sampled outputs computed one by one by
    the oracle from the element matrices of the touching elements, at the north_star bar
    (1e-12 relative per block)."""
    from oracle import sample
    base = "c3" if name == "c3gv" else name
    pr = make_config(base, N=(Nn,) * 3 if Nn else None, p=p)
    if name == "c3gv":
        pr.gamma_vertex = (10.0 ** random_vector(pr.vertices[..., 0].size, 42)).reshape(
            pr.vertices.shape[:-1])
    if name == "c4":
        pr.alpha = 10.0 ** random_vector(pr.E, 41)   # heterogeneous, exercises per-element c_e
        pr.beta = 10.0 ** random_vector(pr.E, 42)
    op = _gpu(pr)
    s = op.sizes
    x = random_vector(s.n, 9)
    y = _host(op.apply_block(_dev(x)))
    op.close()
    rng = np.random.default_rng(0)
    n_rt, n_l2 = s.n_rt, s.n_l2
    # first/last rows, the three RT component blocks' first and last rows, random rows
    offs = [0, n_rt - 1]
    nf = [int(v) for v in (op_offsets(pr))]
    k = 240 if p <= 4 else 100          # the oracle's dense p = 5, 6 element matrices are slow
    rt_rows = np.unique(np.concatenate([offs, nf, rng.integers(0, n_rt, k)]))
    l2_rows = np.unique(np.concatenate([[0, n_l2 - 1], rng.integers(0, n_l2, k // 2)]))
    yu, yq = sample.block_apply_rows(pr, x, rt_rows, l2_rows)
    eu = np.abs(y[rt_rows] - yu).max() / np.abs(yu).max()
    eq = np.abs(y[n_rt + l2_rows] - yq).max() / np.abs(yq).max()
    assert eu < TOL and eq < TOL, (eu, eq)


def op_offsets(pr):
    """First and last rows of the y- and z-face blocks (canonical numbering)."""
    n = [pr.N[a] * pr.p for a in range(3)]
    nx_f = (n[0] + 1) * n[1] * n[2]
    ny_f = n[0] * (n[1] + 1) * n[2]
    return [nx_f - 1, nx_f, nx_f + ny_f - 1, nx_f + ny_f]


@pytest.mark.parametrize("name,N,p,deg", [("c1", None, None, 4), ("c2", (3, 2, 2), 3, 4),
                                          ("c5", (5, 5, 3), 2, 4), ("c2", (5, 3, 4), 4, 1),
                                          ("c2", (5, 3, 4), 6, 2), ("c3", (3, 4, 2), 5, 7),
                                          ("c1", (5, 4), 3, 3)])
def test_preconditioner_chebyshev_paths(name, N, p, deg):
    """S^-1 = the Chebyshev polynomial (reading A10) as a three-term recurrence on the iterate,
    S~ by the matrix-free cell stencil (3D) or the SELL-32 copy (2D): matches the oracle's r/d
    form of the same polynomial (every degree, ragged element grids)."""
    from oracle import operators, solvers
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    P = solvers.BlockDiagPrecond(A, tau=1.0, degree=deg, ratio=30.0)
    v = random_vector(A.n_rt + A.n_l2, 13)
    zo = P.apply(v)
    op = _gpu(pr, tau=1.0, cheb_degree=deg, cheb_ratio=30.0)
    z = _host(op.apply_precond(_dev(v)))
    eu, eq = _rel(z[:A.n_rt], zo[:A.n_rt]), _rel(z[A.n_rt:], zo[A.n_rt:])
    op.close()
    assert eu < TOL and eq < 1e-11, (eu, eq)


# ---- NEXT-1: AMG V-cycle for S^-1 (reading A9b) ----
AMG_CASES = [("c2", (5, 4, 3), 3, 16), ("c1", (6, 5), 2, 8), ("c3", (4, 3, 3), 2, 20),
             ("c5", (5, 5, 3), 2, 30)]


@pytest.mark.parametrize("name,N,p,mc", AMG_CASES)
def test_amg_hierarchy_parity(name, N, p, mc):
    """Level extents, prolongator weights and Galerkin coarse operators (27/9-point stencils,
    formed matrix-free per coarse row on the GPU) against the oracle's scipy P^T A P."""
    from oracle import operators, amg
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    P = amg.AMGSchur(A, nu=2, max_coarse=mc)
    op = _gpu(pr, schur="amg", amg_max_coarse=mc)
    assert op.amg_levels() == len(P.levels)
    for l, lv in enumerate(P.levels):
        dims, omega, st = op.amg_level(l)
        assert tuple(dims[:pr.dim]) == lv.dims
        if lv.omega is not None:
            assert abs(omega - lv.omega) < 1e-14 * lv.omega
        if l == 0:
            continue
        st = _host(st)
        n = st.shape[1]
        ref = lv.A.toarray()
        dense = np.zeros((n, n))
        d = lv.dims + (1,) * (3 - len(lv.dims))
        for i in range(n):
            X, Y, Z = i % d[0], (i // d[0]) % d[1], i // (d[0] * d[1])
            for k in range(st.shape[0]):
                dx, dy, dz = k % 3 - 1, (k // 3) % 3 - 1, (k // 9 - 1) if pr.dim == 3 else 0
                x, y, z = X + dx, Y + dy, Z + dz
                if 0 <= x < d[0] and 0 <= y < d[1] and 0 <= z < d[2]:
                    dense[i, x + d[0] * (y + d[1] * z)] = st[k, i]
                else:
                    assert st[k, i] == 0.0
        assert _rel(dense, ref) < 1e-11


@pytest.mark.parametrize("name,N,p,mc", AMG_CASES)
def test_amg_precond_and_minres_parity(name, N, p, mc):
    from oracle import operators, solvers
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    P = solvers.BlockDiagPrecond(A, schur="amg", amg_nu=2, amg_max_coarse=mc)
    op = _gpu(pr, schur="amg", amg_max_coarse=mc)
    n = A.n_rt + A.n_l2
    v = random_vector(n, 23)
    z = _host(op.apply_precond(_dev(v)))
    zo = P.apply(v)
    assert _rel(z[:A.n_rt], zo[:A.n_rt]) < TOL
    assert _rel(z[A.n_rt:], zo[A.n_rt:]) < 1e-11
    b = A.apply_block(random_vector(n, 1))
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=2000)
    x, rep = op.minres(_dev(b), rtol=1e-12, maxit=2000)
    assert conv_o and rep.converged
    assert abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    assert _rel(_host(x), xo) < 1e-9


@pytest.mark.parametrize("name,N,p,mc,k,ratio", [("c2", (5, 4, 3), 3, 16, 3, 20.0),
                                                 ("c1", (6, 5), 2, 8, 2, 20.0),
                                                 ("c3", (4, 3, 3), 2, 20, 3, 20.0),
                                                 ("c3", (3, 3, 4), 3, 20, 2, 10.0),
                                                 ("c3s", (3, 4, 3), 2, 20, 3, 20.0),
                                                 ("c5", (5, 5, 3), 2, 30, 4, 40.0)])
def test_amg_chebyshev_precond_and_minres_parity(name, N, p, mc, k, ratio):
    """Reading A9d: S^-1 = the degree-k Chebyshev polynomial in B S~ (B = one V-cycle) — the
    preconditioner output and the MINRES iteration count (+-1) against the oracle's r/d form."""
    from oracle import operators, solvers
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    P = solvers.BlockDiagPrecond(A, schur="amg", amg_nu=2, amg_max_coarse=mc, amg_cheb_degree=k,
                                 amg_cheb_ratio=ratio)
    op = _gpu(pr, schur="amg", amg_max_coarse=mc, amg_cheb_degree=k, amg_cheb_ratio=ratio)
    n = A.n_rt + A.n_l2
    v = random_vector(n, 23)
    z = _host(op.apply_precond(_dev(v)))
    zo = P.apply(v)
    assert _rel(z[:A.n_rt], zo[:A.n_rt]) < TOL
    assert _rel(z[A.n_rt:], zo[A.n_rt:]) < 1e-11
    b = A.apply_block(random_vector(n, 1))
    if getattr(pr, "project_mean", False):
        b[A.n_rt:] -= b[A.n_rt:].mean()
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=2000)
    x, rep = op.minres(_dev(b), rtol=1e-12, maxit=2000)
    assert conv_o and rep.converged
    assert abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    if not getattr(pr, "project_mean", False):
        assert _rel(_host(x), xo) < 1e-9


@pytest.mark.parametrize("name,N,p", [("c3gd", (3, 2, 2), 2), ("c3gd", (2, 2, 3), 5), ("c3g", (2, 3, 2), 4),
                                      ("c2", (3, 2, 2), 3), ("c5", (5, 5, 3), 1), ("c1", None, None),
                                      ("c1", (5, 3), 4)])
def test_apply_z_parity(name, N, p):
    """Z q alone (W^-1 through the local CG on any 3D geometry; 2D: the quadrature kernel's
    Kronecker / dense element solve) against the oracle's Cholesky."""
    from oracle import operators
    pr = _problem(name, N, p)
    A = operators.Assembled(pr, with_schur=False)
    op = _gpu(pr)
    q = random_vector(A.n_l2, 29)
    assert _rel(_host(op.apply_z(_dev(q))), A.apply_Z(q)) < TOL



# ---- NEXT-4: block-triangular preconditioner + GMRES ----
@pytest.mark.parametrize("name,N,p,schur,k", [("c1", None, None, "chebyshev", 1),
                                              ("c2", (3, 2, 2), 3, "chebyshev", 1),
                                              ("c3", (2, 2, 2), 2, "amg", 1), ("c5", (5, 5, 3), 1, "amg", 1),
                                              ("c3", (3, 2, 3), 2, "amg", 3)])
def test_gmres_triangular_parity(name, N, p, schur, k):
    from oracle import operators, solvers
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    mc = 16
    B = solvers.BlockTriPrecond(A, schur=schur, amg_max_coarse=mc, amg_cheb_degree=k)
    op = _gpu(pr, schur=schur, amg_max_coarse=mc, amg_cheb_degree=k)
    n = A.n_rt + A.n_l2
    v = random_vector(n, 41)
    z = _host(op.apply_precond_tri(_dev(v)))
    zo = B.apply(v)
    assert _rel(z[:A.n_rt], zo[:A.n_rt]) < 1e-11
    assert _rel(z[A.n_rt:], zo[A.n_rt:]) < 1e-11
    b = A.apply_block(random_vector(n, 43))
    xo, it_o, conv_o, _ = solvers.gmres(A.apply_block, B.apply, b, rtol=1e-10, restart=20,
                                        maxit=2000)
    x, rep = op.gmres(_dev(b), rtol=1e-10, maxit=2000, restart=20)
    assert conv_o and rep.converged
    assert abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    assert _rel(_host(x), xo) < 1e-7


# ---- end-to-end host apply: z-chunked H2D / apply / D2H pipeline (box meshes) ----
@pytest.mark.parametrize("name,N,p,ess", [("c2", (5, 3, 19), 4, 0), ("c2", (4, 3, 17), 3, 63),
                                          ("c5", (5, 5, 9), 2, 0), ("c2", (3, 2, 33), 6, 48),
                                          ("c3", (3, 2, 9), 2, 0)])
def test_host_apply_pipeline_matches_device_apply(name, N, p, ess, monkeypatch):
    """hdiv_apply_block_host (pinned host buffers) returns exactly the device apply's bytes,
    for chunk boundaries inside the mesh, every tile depth, eliminated sides, and (c3) the
    unpipelined quadrature path."""
    import torch
    pr = _problem(name, N, p)
    pr.essential = ess
    op = _gpu(pr)
    n = op.sizes.n
    x = random_vector(n, 23)
    y = _host(op.apply_block(_dev(x)))
    xh = torch.from_numpy(x).pin_memory()
    for pipe in ("1", "0"):
        monkeypatch.setenv("HDIV_HOST_PIPELINE", pipe)
        yh = torch.full((n,), np.nan, dtype=torch.float64).pin_memory()
        op.apply_block_host(xh, yh)
        assert np.array_equal(yh.numpy(), y), pipe
    op.close()


# ---- 2D non-affine quadrilaterals with a nonzero (2,2) block: Z = s_e W^-1 by a dense element
#      solve (Cholesky of the quadrature-assembled W) ----
@pytest.mark.parametrize("N,p,kind", [((4, 3), 2, "grad_div"), ((3, 3), 3, "darcy"),
                                      ((2, 3), 5, "grad_div"), ((3, 2), 1, "darcy")])
def test_2d_quadrilateral_block_and_minres(N, p, kind):
    from oracle import operators, solvers
    from synth import Problem
    from synth.gen import counter_uniform
    V = cartesian_vertices(2, N)
    jit = (2.0 * counter_uniform(11, V.size).reshape(V.shape) - 1.0) * 0.2 / max(N)
    inner = np.zeros(V.shape[:2], bool)
    inner[1:-1, 1:-1] = True
    V = V + jit * inner[..., None]
    E = N[0] * N[1]
    pr = Problem("q2d", 2, tuple(N) + (1,), p, kind, V, alpha=10.0 ** random_vector(E, 1),
                 beta=10.0 ** random_vector(E, 2), eps=10.0 ** random_vector(E, 3),
                 gamma=10.0 ** random_vector(E, 4), affine=False)
    A = operators.Assembled(pr)
    op = _gpu(pr)
    s = op.sizes
    x = random_vector(s.n, 17)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL
    assert _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    q = random_vector(s.n_l2, 29)
    assert _rel(_host(op.apply_z(_dev(q))), A.apply_Z(q)) < TOL     # the (2,2) block alone
    b = A.apply_block(random_vector(s.n, 1))
    P = solvers.BlockDiagPrecond(A)
    _, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=3000)
    xg, rep = op.minres(_dev(b), rtol=1e-12, maxit=3000)
    assert conv_o and rep.converged and abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    op.close()


# ---- degenerate sizes: single elements and one-element-thick meshes, every order ----
@pytest.mark.parametrize("N,p", [((1, 1, 1), 1), ((1, 1, 1), 4), ((1, 1, 1), 6), ((1, 2, 1), 3),
                                 ((2, 1, 1), 5), ((1, 1, 3), 2), ((7, 1, 1), 4)])
def test_tiny_meshes(N, p):
    from oracle import operators, solvers
    pr = _problem("c2", N, p)
    A = operators.Assembled(pr)
    op = _gpu(pr)
    s = op.sizes
    x = random_vector(s.n, 5)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL and _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    rp, col, val = [_host(t) for t in op.schur_csr()]
    assert np.array_equal(rp, A.S.indptr) and np.array_equal(col, A.S.indices)
    b = A.apply_block(random_vector(s.n, 6))
    P = solvers.BlockDiagPrecond(A)
    _, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=2000)
    _, rep = op.minres(_dev(b), rtol=1e-12, maxit=2000)
    assert conv_o and rep.converged and abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    op.close()


# ---- trilinear mass / gamma = 0 applies with several elements per CTA (tri_multi_kernel):
#      element counts not divisible by EPC, eliminated sides, both the 1-element and batched kernels
@pytest.mark.parametrize("epc", ["0", "1", "2", "3", "4", "8"])
@pytest.mark.parametrize("N,p,ess", [((3, 3, 1), 3, 0), ((5, 3, 1), 2, 2 | 16), ((3, 2, 1), 6, 4),
                                     ((7, 1, 1), 1, 1 | 2), ((5, 2, 1), 4, 1 | 32), ((3, 1, 3), 5, 0),
                                     ((7, 1, 1), 4, 63), ((1, 1, 1), 3, 0)])
def test_trilinear_multi_element_ctas(monkeypatch, epc, N, p, ess):
    from oracle import operators
    monkeypatch.setenv("HDIV_TRI_EPC", epc)
    pr = _problem("c3", N, p)
    pr.essential = ess
    A = operators.Assembled(pr, with_schur=False)
    op = _gpu(pr, tri_geometry=1)   # Jacobian from the vertices in every apply
    s = op.sizes
    x = random_vector(s.n, 41)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL and _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    u = x[:s.n_rt]
    assert _rel(_host(op.apply_mass(_dev(u))), A.M @ u) < TOL
    op.close()


# ---- W^-1 on trilinear hexes: precomputed explicit element inverses (default at p <= 4,
#      P:796-798) and the local CG (HDIV_WINV=cg) — block apply, Z alone and MINRES ----
@pytest.mark.parametrize("winv", ["explicit", "explicit-separate", "cg"])
@pytest.mark.parametrize("name,N,p", [("c3gd", (3, 2, 2), 1), ("c3gd", (3, 2, 2), 2), ("c3g", (2, 3, 2), 3),
                                      ("c3gd", (2, 2, 3), 4), ("c3g", (3, 1, 2), 4)])
def test_trilinear_winv_modes(monkeypatch, winv, name, N, p):
    """explicit: the inverses fused into the batched kernel's epilogue; explicit-separate: the
    one-element kernel (HDIV_TRI_EPC=0) + the separate streaming apply; cg: the local CG."""
    from oracle import operators, solvers
    if winv == "cg":
        monkeypatch.setenv("HDIV_WINV", "cg")
    else:
        monkeypatch.delenv("HDIV_WINV", raising=False)
    if winv == "explicit-separate":
        monkeypatch.setenv("HDIV_TRI_EPC", "0")
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    op = _gpu(pr)
    s = op.sizes
    x = random_vector(s.n, 43)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL and _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    q = x[s.n_rt:]
    assert _rel(_host(op.apply_z(_dev(q))), A.apply_Z(q)) < TOL
    b = A.apply_block(random_vector(s.n, 1))
    P = solvers.BlockDiagPrecond(A)
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=3000)
    xg, rep = op.minres(_dev(b), rtol=1e-12, maxit=3000)
    assert conv_o and rep.converged and abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    assert _rel(_host(xg), xo) < 1e-9
    op.close()


# ---- stored quadrature-point factors (partial assembly): tri_geometry=2 stores
#      G_q = w_q mw / det J_q J_q^T J_q at setup; mass, gamma = 0 and explicit-W^-1 block applies
@pytest.mark.parametrize("name,N,p,ess", [("c3", (3, 3, 1), 3, 0), ("c3", (5, 3, 1), 2, 2 | 16),
                                          ("c3", (3, 2, 1), 6, 4), ("c3", (7, 1, 1), 1, 1 | 2),
                                          ("c3", (5, 2, 1), 4, 1 | 32), ("c3", (3, 1, 3), 5, 0),
                                          ("c3", (7, 1, 1), 4, 63), ("c3", (1, 1, 1), 3, 0),
                                          ("c3", (3, 2, 3), 4, 0), ("c3gd", (3, 2, 2), 4, 0),
                                          ("c3gd", (2, 3, 2), 3, 0), ("c3gd", (3, 2, 2), 2, 0)])
def test_trilinear_stored_geometry(name, N, p, ess):
    from oracle import operators
    pr = _problem(name, N, p)
    pr.essential = ess
    A = operators.Assembled(pr, with_schur=False)
    op = _gpu(pr, tri_geometry=2)
    s = op.sizes
    x = random_vector(s.n, 47)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL and _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    u = x[:s.n_rt]
    assert _rel(_host(op.apply_mass(_dev(u))), A.M @ u) < TOL
    y2 = _host(op.apply_block(_dev(x)))
    assert np.array_equal(y, y2)
    op.close()


def test_schur_auto_choice():
    """HDIV_SCHUR_AUTO (the binding's default): Chebyshev below 10^6 global L2 rows, the AMG
    V-cycle from there on (the polynomial is not h-robust); explicit choices are kept."""
    def levels(op):
        try:
            return op.amg_levels()
        except Exception:   # HDIV_ERR_UNSUPPORTED: the handle has no AMG hierarchy
            return 0
    small = make_config("c2", N=(4, 4, 4), p=3)            # 1728 L2 rows
    big = make_config("c2", N=(40, 40, 40), p=3)           # 1.73e6 L2 rows
    for pr, kw, amg in [(small, {}, False), (big, {}, True), (big, {"schur": "chebyshev"}, False),
                        (small, {"schur": "amg"}, True)]:
        op = _gpu(pr, **kw)
        assert (levels(op) >= 1) == amg, (pr.N, kw)
        op.close()


@pytest.mark.gpu
def test_amg_auto_polynomial_degree():
    """options.amg_cheb_degree = 0 (the binding default): the degree-3 polynomial (reading A9d)
    when the element mass weights span more than 10^2 (config 3's eps = 10^U(-2,2)), the plain
    V-cycle on constant coefficients — checked through the preconditioner output against the
    oracle at both degrees."""
    from oracle import operators, solvers
    from paper_2304_12387_b200 import from_problem
    for name, N, p, k in [("c3", (4, 3, 3), 2, 3), ("c4", (4, 3, 3), 2, 1)]:
        pr = make_config(name, N=N, p=p)
        A = operators.Assembled(pr)
        op = from_problem(pr, schur="amg", amg_max_coarse=20)
        v = random_vector(A.n_rt + A.n_l2, 23)
        z = _host(op.apply_precond(_dev(v)))[A.n_rt:]
        for kk in (1, 3):
            P = solvers.BlockDiagPrecond(A, schur="amg", amg_max_coarse=20, amg_cheb_degree=kk)
            err = _rel(z, P.apply(v)[A.n_rt:])
            assert (err < 1e-11) == (kk == k), (name, kk, err)
        op.close()
