"""GPU parity of NEXT-3 (reading A21): essential-flux sides eliminated by identity
rows/columns in every apply kernel (box tiles, trilinear, 2D quadrature), S~ without the
eliminated faces, and the pure-Neumann projection after S^-1 inside MINRES — CUDA path
through the C-ABI vs the CPU oracle on the same seeded inputs."""
import numpy as np
import pytest

from synth import make_config, random_vector

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _rel(a, b):
    d = np.abs(np.asarray(a) - np.asarray(b)).max()
    s = np.abs(np.asarray(b)).max()
    return d / s if s > 0 else d


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _problem(name, N, p, ess, project=False):
    pr = make_config("c3" if name == "c3gd" else name, N=N, p=p)
    if name == "c3gd":
        pr.kind = "grad_div"
        pr.alpha = 10.0 ** random_vector(pr.E, 33)
        pr.beta = 10.0 ** random_vector(pr.E, 34)
    if name == "c2":
        pr.alpha = 10.0 ** random_vector(pr.E, 31)
        pr.beta = 10.0 ** random_vector(pr.E, 32)
    pr.essential, pr.project_mean = ess, project
    return pr


# (config, N, p, essential sides): box tiles (every order, ragged, one-tile and multi-tile
# sides), trilinear hexes, 2D quadrilaterals
CASES = [("c2", (5, 3, 3), 4, 63), ("c2", (5, 3, 6), 2, 1 | 8 | 32), ("c2", (9, 5, 3), 1, 2 | 4),
         ("c2", (3, 3, 3), 6, 63), ("c2", (5, 3, 3), 5, 16 | 32), ("c2", (3, 2, 2), 3, 63),
         ("c5", (5, 5, 3), 3, 63), ("c3", (3, 2, 3), 2, 63), ("c3gd", (2, 3, 2), 4, 1 | 32),
         ("c3", (3, 3, 2), 3, 2 | 4), ("c1", None, None, 15), ("c1", (5, 3), 3, 1 | 8)]


@pytest.mark.parametrize("name,N,p,ess", CASES)
def test_masked_applies(name, N, p, ess):
    from oracle import operators
    from paper_2304_12387_b200 import from_problem
    pr = _problem(name, N, p, ess)
    A = operators.Assembled(pr)
    op = from_problem(pr)
    s = op.sizes
    x = random_vector(s.n, 17)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL
    assert _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    assert np.array_equal(y[:s.n_rt][A.ess], x[:s.n_rt][A.ess])     # identity rows, bitwise
    u, q = x[:s.n_rt], x[s.n_rt:]
    assert _rel(_host(op.apply_mass(_dev(u))), A.M @ u) < TOL
    assert _rel(_host(op.apply_div(_dev(u))), A.D @ u) < TOL
    assert _rel(_host(op.apply_divT(_dev(q))), A.D.T @ q) < TOL
    md = _host(op.mass_diag())
    assert _rel(md, A.Mdiag) < TOL and np.all(md[A.ess] == 1.0)
    rp, col, val = [_host(t) for t in op.schur_csr()]
    assert np.array_equal(rp, A.S.indptr) and np.array_equal(col, A.S.indices)
    assert _rel(val, A.S.data) < 1e-10
    op.close()


@pytest.mark.parametrize("schur", ["chebyshev", "amg", "amg3"])
@pytest.mark.parametrize("name,N,p", [("c3", (3, 3, 2), 2), ("c2", (4, 3, 3), 3), ("c1", (5, 4), 2)])
def test_pure_neumann_minres_parity(name, N, p, schur):
    """All sides essential, Darcy gamma = 0 (the SPE10 shape): singular S~,
    projection after every S^-1; iteration counts +-1 vs the oracle, u unique, p~ up to a
    constant (A16)."""
    from oracle import operators, solvers
    from paper_2304_12387_b200 import from_problem
    pr = _problem(name, N, p, (1 << 2 * (2 if name == "c1" else 3)) - 1, project=True)
    if name != "c1":
        pr.kind, pr.eps, pr.gamma = "darcy", 10.0 ** random_vector(pr.E, 5), np.zeros(pr.E)
    else:
        pr.gamma = np.zeros(pr.E)
    A = operators.Assembled(pr)
    n = A.n_rt + A.n_l2
    xs = random_vector(n, 4)
    b = A.apply_block(xs)
    k = 3 if schur == "amg3" else 1   # amg3: the A9d polynomial over the pinned V-cycle
    schur = "amg" if k == 3 else schur
    P = solvers.BlockDiagPrecond(A, schur=schur, amg_max_coarse=16, amg_cheb_degree=k)
    op = from_problem(pr, schur=schur, amg_max_coarse=16, amg_cheb_degree=k)
    v = random_vector(n, 8)
    v[A.n_rt:] -= v[A.n_rt:].mean()
    z, zo = _host(op.apply_precond(_dev(v))), P.apply(v)
    assert _rel(z[:A.n_rt], zo[:A.n_rt]) < TOL and _rel(z[A.n_rt:], zo[A.n_rt:]) < 1e-11
    assert abs(z[A.n_rt:].mean()) < 1e-13 * np.abs(z[A.n_rt:]).max()
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=3000)
    x, rep = op.minres(_dev(b), rtol=1e-12, maxit=3000)
    x = _host(x)
    assert conv_o and rep.converged and abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    assert _rel(x[:A.n_rt], xo[:A.n_rt]) < 1e-9
    dq = x[A.n_rt:] - xs[A.n_rt:]
    assert np.ptp(dq) < 1e-8 * np.abs(xs[A.n_rt:]).max()
    op.close()


def test_uniform_flow_on_the_gpu():
    """SPE10's boundary condition u.n = (1,0,0).n with constant eps on a graded box mesh: the
    GPU MINRES reproduces u = (1,0,0) exactly (its RT interpolant; oracle pin
    test_uniform_flow_is_reproduced_exactly)."""
    from oracle import operators
    from paper_2304_12387_b200 import from_problem
    pr = make_config("c5", N=(6, 5, 3), p=3)
    pr.kind, pr.eps, pr.gamma = "darcy", np.full(pr.E, 2.5), np.zeros(pr.E)
    pr.essential, pr.project_mean = 63, True
    A = operators.Assembled(pr)
    pr0 = make_config("c5", N=(6, 5, 3), p=3)
    pr0.kind, pr0.eps, pr0.gamma = "darcy", np.full(pr.E, 2.5), np.zeros(pr.E)
    A0 = operators.Assembled(pr0, with_schur=False)
    # x-face DOFs of u = (1, 0, 0): the subcell-face areas (y widths x z widths)
    from oracle import basis1d
    V = pr.vertices
    xi = basis1d.gll_nodes(pr.p)
    ax = [V[0, 0, :, 0], V[0, :, 0, 1], V[:, 0, 0, 2]]
    w = [np.diff(np.append((a[:-1, None] + np.diff(a)[:, None] * xi[None, :-1]).ravel(), a[-1]))
         for a in ax]
    n = [pr.N[a] * pr.p for a in range(3)]
    ustar = np.zeros(A.n_rt)
    ustar[:(n[0] + 1) * n[1] * n[2]] = np.repeat(np.outer(w[2], w[1]).ravel(), n[0] + 1)
    ub = np.where(A.ess, ustar, 0.0)
    b = -A0.apply_block(np.concatenate([ub, np.zeros(A.n_l2)]))
    b[:A.n_rt][A.ess] = ub[A.ess]
    op = from_problem(pr)
    x, rep = op.minres(_dev(b), rtol=1e-13, maxit=5000)
    x = _host(x)
    assert rep.converged
    assert np.abs(x[:A.n_rt] - ustar).max() < 1e-9 * ustar.max()
    op.close()


@pytest.mark.parametrize("ess", [1 | 2 | 16, 63, 4 | 32])
def test_masked_chebyshev_cell_stencil(ess):
    """The matrix-free cell stencil inside S^-1 (3D) drops the eliminated faces too (their
    weights are 0 in the cell-major arrays and they are not in diag(S~))."""
    from oracle import operators, solvers
    from paper_2304_12387_b200 import from_problem
    pr = _problem("c2", (4, 3, 3), 3, ess)
    A = operators.Assembled(pr)
    P = solvers.BlockDiagPrecond(A)
    v = random_vector(A.n_rt + A.n_l2, 13)
    zo = P.apply(v)
    op = from_problem(pr)
    z = _host(op.apply_precond(_dev(v)))
    op.close()
    assert _rel(z[:A.n_rt], zo[:A.n_rt]) < TOL and _rel(z[A.n_rt:], zo[A.n_rt:]) < 1e-11
