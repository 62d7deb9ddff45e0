"""Pins of the oracle's assembled operators, S~, preconditioner and MINRES."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import basis1d, operators, solvers, space, mms
from synth import make_config, random_vector, Problem, cartesian_vertices, perturbed_vertices


@pytest.fixture(scope="module")
def c1():
    return operators.Assembled(make_config("c1"))


def test_config1_traces(c1):
    # closed forms (SURVEY §8(c) pins; sympy): trace(M) = 1792/15, trace(W) = 50176/9
    assert abs(c1.M.diagonal().sum() - 1792 / 15) < 1e-12
    assert abs(c1.Wdiag.sum() - 50176 / 9) < 1e-9
    # Darcy eps=gamma=1 natural BC: interior face terms cancel in row sums
    assert abs(c1.S.sum() - 103.591836734694) < 1e-10
    assert abs(c1.S.diagonal().sum() - 360.734693877551) < 1e-10


def test_trace_closed_form_uniform():
    """trace(M) = E d h^{2-d} tr(M_l) tr(M_h)^{d-1}; trace(W) = E h^-d tr(M_h)^d
    (uniform Cartesian, coefficients 1)."""
    for (dim, n, p) in [(2, 3, 3), (3, 2, 2), (3, 2, 3)]:
        N = (n,) * dim + ((1,) if dim == 2 else ())
        E = n ** dim
        h = 1.0 / n
        pr = Problem("t", dim, N, p, "grad_div", cartesian_vertices(dim, N),
                     alpha=np.ones(E), beta=np.ones(E))
        A = operators.Assembled(pr, with_schur=False)
        Ml, Mh = basis1d.mass_1d(p)
        trM = E * dim * h ** (2 - dim) * np.trace(Ml) * np.trace(Mh) ** (dim - 1)
        trW = E * h ** (-dim) * np.trace(Mh) ** dim
        assert abs(A.M.diagonal().sum() - trM) < 1e-12 * trM
        assert abs(A.Wdiag.sum() - trW) < 1e-12 * trW


def test_schur_two_paths_and_m_matrix(c1):
    S2 = operators.schur_triple_product(c1.D, c1.Mdiag, c1.Ctil)
    assert abs(c1.S - S2).max() < 1e-13 * abs(S2).max()
    assert np.array_equal(c1.S.indptr, S2.indptr) and np.array_equal(c1.S.indices, S2.indices)
    S = c1.S.toarray()
    off = S - np.diag(np.diag(S))
    assert np.all(np.diag(S) > 0) and np.all(off <= 0)
    assert np.all(S.sum(1) >= c1.Ctil - 1e-12)
    assert np.array_equal(S, S.T)                                       # bitwise symmetric


def test_schur_single_element_closed_forms():
    for dim, want in [(2, 13.0), (3, 19.0)]:
        N = (1,) * dim + ((1,) if dim == 2 else ())
        pr = Problem("t", dim, N, 1, "grad_div", cartesian_vertices(dim, N),
                     alpha=np.ones(1), beta=np.ones(1))
        A = operators.Assembled(pr)
        assert abs(A.S.toarray()[0, 0] - want) < 1e-12
    pr = Problem("t", 2, (1, 1, 1), 2, "grad_div", cartesian_vertices(2, (1, 1)),
                 alpha=np.ones(1), beta=np.ones(1))
    S = operators.Assembled(pr).S.toarray()
    assert np.allclose(np.diag(S), 1611 / 196, atol=1e-12)
    off = S[np.abs(S) > 0]
    assert np.allclose(np.sort(off)[:8], -45 / 56, atol=1e-12)


def test_block_symmetry_and_Z(c1):
    x = random_vector(c1.n_rt + c1.n_l2, 11)
    y = random_vector(c1.n_rt + c1.n_l2, 12)
    a = c1.apply_block(x) @ y
    b = x @ c1.apply_block(y)
    assert abs(a - b) < 1e-12 * abs(a)


def test_darcy_piecewise_constant_identity():
    """W^-1 W_gamma W^-1 = W_{1/gamma}^-1 for piecewise-constant gamma."""
    pr = make_config("c3", N=(2, 2, 1), p=2)
    pr.gamma = 10.0 ** random_vector(pr.E, 5)
    A = operators.Assembled(pr, with_schur=False)
    from oracle import fem
    ref = fem.ref_tables(3, 2, 4)
    for e in range(pr.E):
        X = fem.element_vertices(pr.vertices, 3, space.element_index(3, pr.N, e))
        W1g = fem.element_l2_mass(X, 1.0 / pr.gamma[e], ref)
        assert np.allclose(A.Z[e] @ W1g, np.eye(8), atol=1e-11)


def test_grad_div_Z_times_W():
    pr = make_config("c2", N=(2, 2, 2), p=2)
    pr.alpha = 10.0 ** random_vector(pr.E, 3)
    A = operators.Assembled(pr, with_schur=False)
    from oracle import fem
    ref = fem.ref_tables(3, 2, 4)
    for e in range(pr.E):
        X = fem.element_vertices(pr.vertices, 3, space.element_index(3, pr.N, e))
        W = fem.element_l2_mass(X, pr.alpha[e], ref)
        assert np.allclose(A.Z[e] @ W, np.eye(8), atol=1e-12)


@pytest.mark.parametrize("tau,interval", [(1.0, (-1, (1 - 5 ** 0.5) / 2, 1, (1 + 5 ** 0.5) / 2)),
                                          (2.0, (-1, -0.5, 0.5, 1))])
def test_prop21_22_spectra(tau, interval):
    """Props 2.1/2.2: exact blocks give the printed eigenvalue intervals."""
    pr = make_config("c1", N=(2, 2), p=2)
    pr.eps = 10.0 ** random_vector(pr.E, 1)
    pr.gamma = 10.0 ** random_vector(pr.E, 2)
    A = operators.Assembled(pr)
    Ad = A.dense_block()
    P = solvers.BlockDiagPrecond(A, tau=tau, exact_blocks=True)
    n = A.n_rt
    Bd = sla.block_diag(tau * P.Mfull, P.Sfull)
    lam = sla.eigh(Ad, Bd, eigvals_only=True)
    lo1, hi1, lo2, hi2 = interval
    neg, pos = lam[lam < 0], lam[lam > 0]
    tol = 1e-9
    assert np.all(neg >= lo1 - tol) and np.all(neg <= hi1 + tol)
    assert np.all(pos >= lo2 - tol) and np.all(pos <= hi2 + tol)
    assert len(neg) == A.n_l2 and len(pos) == n


def test_chebyshev_polynomial_closed_form():
    """Residual polynomial of the Chebyshev semi-iteration (reading A10) on a unit-diagonal
    M-matrix S = tridiag(-c, 1, -c) (Jacobi scaling D = I): for an eigenpair (lam, v),
    S^-1_hat v = p(lam) v with 1 - lam p(lam) = T_k((theta - lam)/delta) / T_k(theta/delta)."""
    import scipy.sparse as sp
    from numpy.polynomial import chebyshev as C
    n, c = 40, 0.49
    S = sp.diags([-c * np.ones(n - 1), np.ones(n), -c * np.ones(n - 1)], [-1, 0, 1]).tocsr()
    lam, V = np.linalg.eigh(S.toarray())
    a, b = 2.0 / 30, 2.0
    th, de = (a + b) / 2, (b - a) / 2
    for k in [1, 2, 4, 7]:
        Tk = C.Chebyshev.basis(k)
        for t in range(0, n, 5):
            y = solvers.chebyshev_jacobi(S, V[:, t], k, 30.0)
            pl = (1 - Tk((th - lam[t]) / de) / Tk(th / de)) / lam[t]
            assert np.allclose(y, pl * V[:, t], atol=1e-12)
            assert pl > 0


def test_minres_matches_dense_solve_c1(c1):
    n = c1.n_rt + c1.n_l2
    xs = random_vector(n, 1)
    b = c1.apply_block(xs)
    P = solvers.BlockDiagPrecond(c1, tau=1.0, degree=4, ratio=30.0)
    x, it, conv, hist = solvers.minres(c1.apply_block, P.apply, b, rtol=1e-12, maxit=500)
    assert conv
    xd = np.linalg.solve(c1.dense_block(), b)
    assert np.abs(x - xd).max() <= 1e-9 * np.abs(xd).max()
    assert np.all(np.diff(hist) <= 1e-15)   # preconditioned residual monotone


def test_minres_indefinite_two_by_two():
    A = np.diag([1.0, -1.0])
    x, it, conv, _ = solvers.minres(lambda v: A @ v, lambda v: v, np.array([1.0, 2.0]))
    assert conv and it <= 2 and np.allclose(x, [1.0, -2.0])


def test_minres_3d_perturbed_darcy_dense():
    pr = make_config("c3", N=(2, 2, 2), p=2)
    A = operators.Assembled(pr)
    n = A.n_rt + A.n_l2
    b = A.apply_block(random_vector(n, 9))
    P = solvers.BlockDiagPrecond(A, tau=1.0, degree=4, ratio=30.0)
    x, it, conv, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=2000)
    xd = np.linalg.solve(A.dense_block(), b)
    assert conv
    assert np.abs(x - xd).max() <= 1e-8 * np.abs(xd).max()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_mms_convergence_rate_2d(p):
    """MMS (reading A13): ||u - u_h||_L2 = O(h^p) for RT degree p."""
    errs = []
    for n in (2, 4, 8):
        pr = Problem("mms", 2, (n, n, 1), p, "grad_div", cartesian_vertices(2, (n, n)),
                     alpha=np.ones(n * n), beta=np.ones(n * n))
        A = operators.Assembled(pr)
        b = np.concatenate([mms.load_vector(pr), np.zeros(A.n_l2)])
        x = np.linalg.solve(A.dense_block(), b) if A.n_rt + A.n_l2 < 4000 else None
        errs.append(mms.l2_error(pr, x[:A.n_rt]))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates >= p - 0.25), rates


# ---- NEXT-4: block-triangular preconditioner + GMRES ----
@pytest.mark.parametrize("cfg,N,p", [("c1", (2, 2), 2), ("c2", (2, 2, 2), 2), ("c3", (2, 2, 2), 2)])
def test_gmres_exact_triangular_converges_in_two(cfg, N, p):
    """with the exact blocks B = [M, D^T; 0, -S], GMRES converges in at most two
    iterations (sigma(B^-1 A) = {1}, minimal polynomial of degree 2)."""
    from synth import make_config, random_vector
    from oracle import operators, solvers
    A = operators.Assembled(make_config(cfg, N=N, p=p))
    B = solvers.BlockTriPrecond(A, exact_blocks=True)
    n = A.n_rt + A.n_l2
    xs = random_vector(n, 4)
    b = A.apply_block(xs)
    x, it, conv, _ = solvers.gmres(A.apply_block, B.apply, b, rtol=1e-12, restart=30)
    assert conv and it <= 2, it
    assert np.abs(x - xs).max() < 1e-9 * np.abs(xs).max()


def test_gmres_matches_dense_solve_and_restarts():
    """Unpreconditioned GMRES on a small nonsymmetric system: full GMRES reaches the dense solve
    within n iterations; restarted GMRES(5) reaches the same solution."""
    from oracle import solvers
    rng = np.random.default_rng(3)
    n = 40
    M = np.eye(n) * 4 + rng.standard_normal((n, n)) * 0.3
    b = rng.standard_normal(n)
    xd = np.linalg.solve(M, b)
    x, it, conv, _ = solvers.gmres(lambda v: M @ v, lambda v: v, b, rtol=1e-13, restart=n)
    assert conv and it <= n and np.abs(x - xd).max() < 1e-10
    x5, it5, conv5, _ = solvers.gmres(lambda v: M @ v, lambda v: v, b, rtol=1e-12, restart=5,
                                      maxit=2000)
    assert conv5 and it5 > it and np.abs(x5 - xd).max() < 1e-9


def test_gmres_triangular_vs_minres_diagonal():
    """Inexact blocks: GMRES + block-triangular needs fewer iterations than MINRES +
    block-diagonal on the same problem (recorded empirically)."""
    from synth import make_config, random_vector
    from oracle import operators, solvers
    A = operators.Assembled(make_config("c2", N=(4, 4, 4), p=2))
    n = A.n_rt + A.n_l2
    b = A.apply_block(random_vector(n, 6))
    Pd = solvers.BlockDiagPrecond(A)
    _, it_m, conv_m, _ = solvers.minres(A.apply_block, Pd.apply, b, rtol=1e-10, maxit=2000)
    Pt = solvers.BlockTriPrecond(A)
    _, it_g, conv_g, _ = solvers.gmres(A.apply_block, Pt.apply, b, rtol=1e-10, restart=50,
                                       maxit=2000)
    assert conv_m and conv_g
    assert it_g < it_m, (it_g, it_m)
