"""Pins of the oracle's Piola-mapped element matrices on NON-axis-aligned elements.

P:84  (§2, H(div) Piola map): V_h(kappa) = det(J)^-1 J V_h(kappa_hat), so the physical RT basis
      function is phi = J phi_hat / det J and
      M^e_mn = int_kappa beta phi_m . phi_n = int_hat beta phi_hat_m^T (J^T J / det J) phi_hat_n.
P:117 L2 basis psi = psi_hat / det J;  P:135 eq.(matrices).

These are pinned against things the oracle does not compute itself:
  * the parallelepiped closed form: a constant J gives M^e_{(c,m),(c',n)} =
    (beta / det J) (J^T J)_{c c'} * prod_axes (exact 1D integral of the two factors) — the 1D
    functions here are built independently (numpy Legendre series: GLL nodes as the roots of
    P_p', Lagrange products, h_j = -sum_{i<=j} l_i', integrals by exact antiderivatives);
  * rotation invariance of M^e and W^e on general trilinear elements (J -> R J leaves J^T J
    and det J unchanged; J J^T would rotate);
  * the scaling law M^e(s X) = s^{2-d} M^e(X);
  * manufactured-solution convergence on smoothly distorted (genuinely trilinear) 2D/3D meshes.
A J <-> J^T swap anywhere in fem.jacobian / fem.element_rt_mass fails the first three.
"""
import numpy as np
from numpy.polynomial import Legendre as Leg
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import fem, mms, operators
from synth import Problem, cartesian_vertices

# --------------------------------------------------------------------------------------------
# independent 1D functions (power basis on [0,1])


def _gll01(p):
    """GLL nodes on [0,1]: endpoints and the roots of P_p'(2x-1) (numpy Legendre class)."""
    if p == 1:
        return np.array([0.0, 1.0])
    r = np.polynomial.legendre.Legendre.basis(p).deriv().roots()
    return np.sort(np.concatenate([[0.0, 1.0], 0.5 * (np.real(r) + 1.0)]))


def _lagrange_polys(p):
    """l_i as numpy Legendre series on the domain [0,1] (well conditioned at high p)."""
    xi = _gll01(p)
    out = []
    for i in range(p + 1):
        c = Leg.fromroots(np.delete(xi, i), domain=[0, 1])
        out.append(c / c(xi[i]))
    return out


def _histo_polys(p):
    """h_j = -sum_{i<=j} l_i'   (from int_{xi_m}^{xi_{m+1}} l_i' = delta_{i,m+1} - delta_{i,m})."""
    L = _lagrange_polys(p)
    out, acc = [], Leg([0.0], domain=[0, 1])
    for j in range(p):
        acc = acc - L[j].deriv()
        out.append(acc)
    return out


def _int01(a, b):
    c = (a * b).integ()
    return c(1.0) - c(0.0)


def _mix(fa, fb):
    return np.array([[_int01(a, b) for b in fb] for a in fa])


def test_independent_histopolation_dofs():
    """The test's own h_j satisfy the histopolation DOF definition."""
    for p in range(1, 6):
        xi = _gll01(p)
        H = _histo_polys(p)
        for j, h in enumerate(H):
            c = h.integ()
            I = c(xi[1:]) - c(xi[:-1])
            assert np.abs(I - np.eye(p)[j]).max() < 1e-12


def _closed_form_mass(dim, p, J, beta):
    """(beta/det J) (J^T J)_{cc'} (x) exact 1D integrals, in the oracle's local order
    (x-block i + (p+1)(j + p k), y-block i + p(j + (p+1)k), z-block i + p(j + p k))."""
    L, H = _lagrange_polys(p), _histo_polys(p)
    # factor along axis a of component c: l if a == c else h
    fac = lambda c, a: L if a == c else H
    G = beta * (J.T @ J) / np.linalg.det(J)
    blocks = [[None] * dim for _ in range(dim)]
    for c in range(dim):
        for d in range(dim):
            K = np.ones((1, 1))
            for a in range(dim):          # kron order: last axis outermost, x fastest
                K = np.kron(_mix(fac(c, a), fac(d, a)), K)
            blocks[c][d] = G[c, d] * K
    return np.block(blocks)


def _parallelepiped(J, x0):
    dim = J.shape[0]
    if dim == 2:
        X = np.zeros((2, 2, 2))
        for b in range(2):
            for a in range(2):
                X[b, a] = x0 + J @ np.array([a, b], float)
        return X
    X = np.zeros((2, 2, 2, 3))
    for c in range(2):
        for b in range(2):
            for a in range(2):
                X[c, b, a] = x0 + J @ np.array([a, b, c], float)
    return X


_J3 = np.array([[1.10, 0.35, -0.20],
                [0.05, 0.80, 0.30],
                [0.15, -0.25, 1.30]])
_J2 = np.array([[0.9, 0.4],
                [-0.1, 1.2]])


@pytest.mark.parametrize("dim,p", [(2, 1), (2, 2), (2, 4), (3, 1), (3, 2), (3, 3)])
def test_parallelepiped_mass_closed_form(dim, p):
    """M^e on a constant-J (sheared, non-symmetric J) element = the closed form."""
    J = _J3 if dim == 3 else _J2
    assert np.abs(J - J.T).max() > 0.1       # J^T J != J J^T here
    assert np.abs(J.T @ J - J @ J.T).max() > 0.1
    X = _parallelepiped(J, np.full(dim, 0.3))
    beta = 2.5
    ref = fem.ref_tables(dim, p, p + 2)
    Me = fem.element_rt_mass(X, beta, ref)
    Mc = _closed_form_mass(dim, p, J, beta)
    assert np.abs(Me - Mc).max() <= 1e-13 * np.abs(Mc).max()


@pytest.mark.parametrize("dim,p", [(2, 2), (3, 2), (3, 3)])
def test_parallelepiped_l2_mass_closed_form(dim, p):
    """W^e = (c / det J) M_h^{(x)d} on a constant-J element."""
    J = _J3 if dim == 3 else _J2
    X = _parallelepiped(J, np.zeros(dim))
    ref = fem.ref_tables(dim, p, p + 2)
    We = fem.element_l2_mass(X, 3.0, ref)
    Mh = _mix(_histo_polys(p), _histo_polys(p))
    K = np.ones((1, 1))
    for _ in range(dim):
        K = np.kron(Mh, K)
    Wc = 3.0 / np.linalg.det(J) * K
    assert np.abs(We - Wc).max() <= 1e-13 * np.abs(Wc).max()


def _rotation(dim, seed):
    rng = np.random.default_rng(seed)
    Q, R = np.linalg.qr(rng.standard_normal((dim, dim)))
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def _trilinear_element(dim, seed):
    """A general (non-parallelepiped) element: unit cube corners jittered by up to 0.2."""
    rng = np.random.default_rng(seed)
    X = _parallelepiped(np.eye(dim), np.zeros(dim))
    return X + rng.uniform(-0.2, 0.2, X.shape)


@pytest.mark.parametrize("dim,p", [(2, 2), (2, 3), (3, 1), (3, 2)])
def test_rotation_invariance_trilinear(dim, p):
    """M^e, W^e, B^e are invariant under a rigid rotation of a general trilinear element:
    J -> R J leaves J^T J and det J unchanged."""
    ref = fem.ref_tables(dim, p, p + 2)
    for seed in range(3):
        X = _trilinear_element(dim, seed)
        R = _rotation(dim, 10 + seed)
        Xr = np.einsum("de,...e->...d", R, X) + 0.7
        M0, M1 = fem.element_rt_mass(X, 1.3, ref), fem.element_rt_mass(Xr, 1.3, ref)
        assert np.abs(M0 - M1).max() <= 1e-13 * np.abs(M0).max()
        W0, W1 = fem.element_l2_mass(X, 0.7, ref), fem.element_l2_mass(Xr, 0.7, ref)
        assert np.abs(W0 - W1).max() <= 1e-13 * np.abs(W0).max()
        B0, B1 = fem.element_div_form(X, ref), fem.element_div_form(Xr, ref)
        assert np.abs(B0 - B1).max() <= 1e-13 * np.abs(B0).max()
        # and the element is genuinely non-affine: J varies over the quadrature points
        J, _ = fem.jacobian(X, ref.pts)
        assert np.abs(J - J[0]).max() > 1e-2


@pytest.mark.parametrize("dim", [2, 3])
def test_scaling_law(dim):
    """x -> s x: J -> s J, so J^T J / det J -> s^{2-d} J^T J / det J."""
    p = 2
    ref = fem.ref_tables(dim, p, p + 2)
    X = _trilinear_element(dim, 5)
    s = 0.37
    M0, M1 = fem.element_rt_mass(X, 1.0, ref), fem.element_rt_mass(s * X, 1.0, ref)
    assert np.abs(M1 - s ** (2 - dim) * M0).max() <= 1e-13 * np.abs(M1).max()


def test_mass_not_symmetric_in_J_orientation():
    """Sanity of the pin itself: the J J^T variant of the closed form differs from the
    J^T J one for the test's J (so a transposed Jacobian cannot pass the closed-form test)."""
    for J in (_J2, _J3):
        A, B = J.T @ J, J @ J.T
        assert np.abs(A - B).max() > 0.1


# --------------------------------------------------------------------------------------------
# manufactured solutions on smoothly distorted meshes (every element a general trilinear hex)


def _distorted_vertices(dim, n, amp=0.08):
    """x + amp * sin(pi x) sin(2 pi y) [sin(pi z)] ... (vanishes on the boundary: the domain is
    still the unit box), different per component so J is non-symmetric."""
    V = cartesian_vertices(dim, (n,) * dim).copy()
    s = np.sin
    pi = np.pi
    if dim == 2:
        x, y = V[..., 0].copy(), V[..., 1].copy()
        V[..., 0] += amp * s(pi * x) * s(2 * pi * y)
        V[..., 1] += amp * s(2 * pi * x) * s(pi * y)
        return V
    x, y, z = V[..., 0].copy(), V[..., 1].copy(), V[..., 2].copy()
    V[..., 0] += amp * s(pi * x) * s(2 * pi * y) * s(pi * z)
    V[..., 1] += amp * s(pi * x) * s(pi * y) * s(2 * pi * z)
    V[..., 2] += amp * s(2 * pi * x) * s(pi * y) * s(pi * z)
    return V


def _mms_errors(dim, p, ns):
    errs = []
    for n in ns:
        N = (n,) * dim + ((1,) if dim == 2 else ())
        E = n ** dim
        pr = Problem("mms", dim, N, p, "grad_div", _distorted_vertices(dim, n),
                     alpha=np.ones(E), beta=np.ones(E), affine=False)
        A = operators.Assembled(pr, with_schur=False)
        K = sp.bmat([[A.M, A.D.T], [A.D, -sp.block_diag(A.Z)]], format="csc")
        b = np.concatenate([mms.load_vector(pr), np.zeros(A.n_l2)])
        x = spla.spsolve(K, b)
        errs.append(mms.l2_error(pr, x[:A.n_rt]))
    return np.array(errs)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_mms_rate_2d_distorted(p):
    """||u - u_h||_L2 = O(h^p) (reading A13) on smoothly distorted quadrilaterals."""
    e = _mms_errors(2, p, (4, 8, 16))
    rates = np.log2(e[:-1] / e[1:])
    assert np.all(rates >= p - 0.25), (e, rates)


@pytest.mark.parametrize("p,ns", [(1, (2, 4, 8)), (2, (2, 4, 8))])
def test_mms_rate_3d_distorted(p, ns):
    """||u - u_h||_L2 = O(h^p) (reading A13) on smoothly distorted hexahedra."""
    e = _mms_errors(3, p, ns)
    rates = np.log2(e[:-1] / e[1:])
    assert rates[-1] >= p - 0.25, (e, rates)
