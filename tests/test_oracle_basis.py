"""Pins of the oracle's 1D tables and element matrices against closed forms and
mathematical identities that the oracle does NOT use in its construction."""
import numpy as np
import pytest

from oracle import basis1d, fem, space


def test_gll_closed_forms():
    # P:178 Gauss-Lobatto points; closed forms on [0,1]
    assert np.allclose(basis1d.gll_nodes(1), [0, 1], atol=0, rtol=0)
    assert np.allclose(basis1d.gll_nodes(2), [0, 0.5, 1], atol=1e-16)
    s = np.sqrt(5) / 10
    assert np.allclose(basis1d.gll_nodes(3), [0, 0.5 - s, 0.5 + s, 1], atol=1e-15)
    # p=4: interior 1/2, 1/2 +- sqrt(21)/14
    r = np.sqrt(21) / 14
    assert np.allclose(basis1d.gll_nodes(4), [0, 0.5 - r, 0.5, 0.5 + r, 1], atol=1e-15)


@pytest.mark.parametrize("p", range(1, 9))
def test_gll_quadrature_exactness(p):
    # GLL weights from the Lagrange basis integrals must integrate degree 2p-1 exactly
    xi = basis1d.gll_nodes(p)
    xq, wq = basis1d.gl_rule(p + 2)
    w = wq @ basis1d.lagrange(xi, xq)
    for k in range(2 * p):
        assert abs(w @ xi ** k - 1.0 / (k + 1)) < 1e-14


@pytest.mark.parametrize("Q", range(1, 10))
def test_gl_exactness(Q):
    x, w = basis1d.gl_rule(Q)
    for k in range(2 * Q):
        assert abs(w @ x ** k - 1.0 / (k + 1)) < 1e-14
    if Q == 1:
        assert np.allclose(x, [0.5]) and np.allclose(w, [1.0])
    if Q == 2:
        assert np.allclose(x, [0.5 - 0.5 / np.sqrt(3), 0.5 + 0.5 / np.sqrt(3)], atol=1e-16)


def test_histopolation_p2_closed_form():
    x = np.linspace(0, 1, 11)
    H = basis1d.histopolation(2, x)
    assert np.allclose(H[:, 0], 3 - 4 * x, atol=1e-14)
    assert np.allclose(H[:, 1], 4 * x - 1, atol=1e-14)


@pytest.mark.parametrize("p", range(1, 11))
def test_histopolation_identities(p):
    """l_i' = h_{i-1} - h_i (h_{-1} = h_p = 0): integral of l_i' over subinterval m is
    delta_{i,m+1} - delta_{i,m}; a property of the GLL Lagrange basis, not used by the
    oracle's construction (which solves the histopolation DOF system)."""
    xi = basis1d.gll_nodes(p)
    x = np.random.default_rng(p).random(17)
    dL = basis1d.lagrange_deriv(xi, x)
    H = basis1d.histopolation(p, x)
    Hp = np.concatenate([np.zeros((len(x), 1)), H, np.zeros((len(x), 1))], axis=1)
    for i in range(p + 1):
        assert np.allclose(dL[:, i], Hp[:, i] - Hp[:, i + 1], atol=1e-11 * max(1, p ** 3))
    # partition-of-unity in the histopolation sense: sum_j |I_j| h_j == 1
    assert np.allclose(H @ np.diff(xi), 1.0, atol=1e-13)
    # defining DOFs checked with an independent fine quadrature on each subinterval
    t, w = np.polynomial.legendre.leggauss(p + 3)
    for m in range(p):
        a, b = xi[m], xi[m + 1]
        pts = a + (b - a) * 0.5 * (t + 1)
        integ = (0.5 * (b - a) * w) @ basis1d.histopolation(p, pts)
        assert np.allclose(integ, np.eye(p)[m], atol=1e-13)


def test_1d_masses_closed_form():
    Ml, Mh = basis1d.mass_1d(1)
    assert np.allclose(Ml, np.array([[2, 1], [1, 2]]) / 6, atol=1e-16)
    assert np.allclose(Mh, [[1.0]])
    Ml, Mh = basis1d.mass_1d(2)
    assert np.allclose(Ml, np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]) / 30, atol=1e-15)
    assert np.allclose(Mh, np.array([[7, -1], [-1, 7]]) / 3, atol=1e-14)
    assert np.allclose(np.linalg.inv(Mh), np.array([[7, 1], [1, 7]]) / 16, atol=1e-15)
    # p=3 M_h entries (sympy)
    Ml, Mh = basis1d.mass_1d(3)
    s5 = np.sqrt(5)
    assert abs(Mh[0, 0] - 13 / 3) < 1e-13 and abs(Mh[0, 2] - 1 / 6) < 1e-13
    assert abs(Mh[0, 1] - (9 / 4 - 5 * s5 / 4)) < 1e-13
    assert abs(Mh[1, 1] - (17 / 2 - 5 * s5 / 2)) < 1e-13
    assert abs(np.trace(Mh) - (103 / 6 - 5 * s5 / 2)) < 1e-13


def _unit_X(dim, h=None):
    h = np.ones(dim) if h is None else np.asarray(h, float)
    if dim == 2:
        X = np.zeros((2, 2, 2))
        for b in range(2):
            for a in range(2):
                X[b, a] = [a * h[0], b * h[1]]
        return X
    X = np.zeros((2, 2, 2, 3))
    for c in range(2):
        for b in range(2):
            for a in range(2):
                X[c, b, a] = [a * h[0], b * h[1], c * h[2]]
    return X


def test_rt0_unit_square():
    ref = fem.ref_tables(2, 1, 3)
    M = fem.element_rt_mass(_unit_X(2), 1.0, ref)
    assert np.allclose(M[:2, :2], np.array([[2, 1], [1, 2]]) / 6, atol=1e-15)
    assert np.allclose(M[:2, 2:], 0, atol=1e-15)
    W = fem.element_l2_mass(_unit_X(2), 1.0, ref)
    assert np.allclose(W, [[1.0]])


def test_unit_square_p2_diag():
    ref = fem.ref_tables(2, 2, 4)
    M = fem.element_rt_mass(_unit_X(2), 1.0, ref)
    want = np.array([14, 56, 14, 14, 56, 14, 14, 14, 56, 56, 14, 14], float)
    assert np.allclose(45 * np.diag(M), want, atol=1e-12)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_affine_mass_is_kronecker(p):
    """On an axis-aligned box M^e = blockdiag(c_x Mh(x)Mh(x)Ml, ...): exact polynomial
    integration (independent closed form: Kronecker of 1D masses)."""
    h = np.array([0.3, 0.7, 1.9])
    ref = fem.ref_tables(3, p, p + 2)
    M = fem.element_rt_mass(_unit_X(3, h), 2.5, ref)
    Ml, Mh = basis1d.mass_1d(p, p + 3)
    det = np.prod(h)
    nc = (p + 1) * p * p
    Kx = 2.5 * h[0] ** 2 / det * np.kron(Mh, np.kron(Mh, Ml))
    Ky = 2.5 * h[1] ** 2 / det * np.kron(Mh, np.kron(Ml, Mh))
    Kz = 2.5 * h[2] ** 2 / det * np.kron(Ml, np.kron(Mh, Mh))
    assert np.allclose(M[:nc, :nc], Kx, rtol=1e-13, atol=1e-13 * abs(Kx).max())
    assert np.allclose(M[nc:2 * nc, nc:2 * nc], Ky, atol=1e-13 * abs(Ky).max())
    assert np.allclose(M[2 * nc:, 2 * nc:], Kz, atol=1e-13 * abs(Kz).max())
    assert np.allclose(M[:nc, nc:], 0, atol=1e-13 * abs(M).max())
    W = fem.element_l2_mass(_unit_X(3, h), 0.5, ref)
    assert np.allclose(W, 0.5 / det * np.kron(Mh, np.kron(Mh, Mh)), atol=1e-13 * abs(W).max())


@pytest.mark.parametrize("p", [2, 4])
def test_affine_mass_quadrature_invariant(p):
    ref1 = fem.ref_tables(3, p, p + 1)
    ref2 = fem.ref_tables(3, p, p + 5)
    X = _unit_X(3, [0.5, 1.0, 2.0])
    M1 = fem.element_rt_mass(X, 1.0, ref1)
    M2 = fem.element_rt_mass(X, 1.0, ref2)
    assert np.allclose(M1, M2, atol=1e-14 * abs(M1).max())


def _jittered_X(seed):
    X = _unit_X(3)
    rng = np.random.default_rng(seed)
    return X + rng.uniform(-0.2, 0.2, X.shape)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("seed", [0, 1])
def test_B_equals_W_D(p, seed):
    """D = W^-1 B, i.e. B = W D with D the topological incidence."""
    X = _jittered_X(seed)
    ref = fem.ref_tables(3, p, p + 2)
    W = fem.element_l2_mass(X, 1.0, ref)
    B = fem.element_div_form(X, ref)
    v2f, sig = space.volume_to_face(3, p)
    nl = p ** 3
    D = np.zeros((nl, ref.n_rt))
    D[np.arange(nl)[None, :].repeat(6, 0), v2f] = sig
    assert np.abs(B - W @ D).max() <= 1e-13 * np.abs(B).max()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_mass_spd_on_distorted(p):
    X = _jittered_X(7)
    ref = fem.ref_tables(3, p, p + 2)
    M = fem.element_rt_mass(X, 1.0, ref)
    assert np.allclose(M, M.T, atol=1e-14 * abs(M).max())
    np.linalg.cholesky(M)
    W = fem.element_l2_mass(X, 1.0, ref)
    np.linalg.cholesky(W)


def test_inverted_element_rejected():
    X = _unit_X(3)
    X[1, 1, 1] = [-0.5, -0.5, -0.5]
    with pytest.raises(ValueError):
        fem.element_rt_mass(X, 1.0, fem.ref_tables(3, 2, 4))
