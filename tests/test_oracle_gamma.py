"""Pins of the general-gamma Darcy (2,2) block W^-1 W_gamma W^-1 (NEXT-3: "in the general
case ... the full form of the (2,2)-block is used", "twice every iteration"; reading A22:
gamma = trilinear field of per-vertex values)."""
import numpy as np
import pytest
from numpy.polynomial import polynomial as Pl

from oracle import basis1d, operators
from synth import Problem, cartesian_vertices, perturbed_vertices, random_vector


def _darcy(N, p, V, gv, gamma_e=None):
    E = int(np.prod(N))
    return Problem("t", 3, tuple(N), p, "darcy", V, eps=np.ones(E),
                   gamma=np.zeros(E) if gamma_e is None else gamma_e, gamma_vertex=gv)


def test_constant_vertex_field_reduces_to_piecewise_constant():
    """gamma_v = c everywhere: W_gamma = c W, so W^-1 W_gamma W^-1 = c W^-1 = W_{1/c}^-1
    — the same operator as the per-element constant gamma = c."""
    N, p = (2, 2, 2), 3
    V = perturbed_vertices(N, 0.2, 7)
    A1 = operators.Assembled(_darcy(N, p, V, np.full(V.shape[:-1], 2.5)), with_schur=False)
    A2 = operators.Assembled(_darcy(N, p, V, None, np.full(8, 2.5)), with_schur=False)
    for Z1, Z2 in zip(A1.Z, A2.Z):
        assert np.abs(Z1 - Z2).max() < 1e-12 * np.abs(Z2).max()
    assert np.abs(A1.Ctil - A2.Ctil).max() < 1e-13 * np.abs(A2.Ctil).max()


def test_linear_gamma_on_unit_box_is_a_weighted_kronecker_product():
    """One unit element, gamma(x) = x (vertex values 0 / 1 along x): det J = 1, psi = h_a h_b h_c,
    so W_gamma = Mh ⊗ Mh ⊗ Mh^(x) with Mh^(x)_ab = int_0^1 x h_a h_b dx, integrated exactly
    here from the closed forms h_0 = 3 - 4x, h_1 = 4x - 1 (p = 2, SURVEY pins)."""
    p = 2
    V = cartesian_vertices(3, (1, 1, 1))
    gv = V[..., 0].copy()                                 # gamma = x at the vertices
    A = operators.Assembled(_darcy((1, 1, 1), p, V, gv), with_schur=False)
    h = [np.array([3.0, -4.0]), np.array([-1.0, 4.0])]    # coefficients in x (ascending)
    def integ(c):
        ci = Pl.polyint(c)
        return Pl.polyval(1.0, ci) - Pl.polyval(0.0, ci)
    Mh = np.array([[integ(Pl.polymul(h[a], h[b])) for b in range(2)] for a in range(2)])
    Mx = np.array([[integ(Pl.polymul([0.0, 1.0], Pl.polymul(h[a], h[b]))) for b in range(2)]
                   for a in range(2)])
    Wg = np.kron(Mh, np.kron(Mh, Mx))                     # a (x) fastest
    W = np.kron(Mh, np.kron(Mh, Mh))
    Z = np.linalg.solve(W, np.linalg.solve(W, Wg).T).T    # W^-1 Wg W^-1 (W symmetric)
    assert np.abs(A.Z[0] - Z).max() < 1e-13 * np.abs(Z).max()
    assert np.abs(A.Wgdiag - np.diag(Wg)).max() < 1e-14 * np.abs(Wg).max()


def test_p1_box_closed_form():
    """p = 1 on a box: one L2 DOF per element, psi = 1/det J, so
    Z_e = int gamma / |K|^-2 ... = (mean of the 8 vertex values) |K| (the trilinear mean is exact
    under the Q = 3 rule)."""
    ax = [np.array([0.0, 0.4, 1.0]), np.array([0.0, 0.7, 1.0]), np.array([0.0, 0.25, 1.0])]
    from synth.gen import tensor_vertices
    V = tensor_vertices(ax)
    gv = 10.0 ** random_vector(V[..., 0].size, 3).reshape(V.shape[:-1])
    A = operators.Assembled(_darcy((2, 2, 2), 1, V, gv), with_schur=False)
    for e in range(8):
        ex, ey, ez = e % 2, (e // 2) % 2, e // 4
        vol = np.diff(ax[0])[ex] * np.diff(ax[1])[ey] * np.diff(ax[2])[ez]
        mean = gv[ez:ez + 2, ey:ey + 2, ex:ex + 2].mean()
        assert abs(A.Z[e][0, 0] - mean * vol) < 1e-13 * mean * vol


def test_general_gamma_block_symmetric_and_definite():
    N, p = (2, 1, 2), 2
    V = perturbed_vertices(N, 0.2, 5)
    gv = 10.0 ** random_vector(V[..., 0].size, 9).reshape(V.shape[:-1])
    A = operators.Assembled(_darcy(N, p, V, gv))
    for Ze in A.Z:
        assert np.abs(Ze - Ze.T).max() < 1e-14 * np.abs(Ze).max()
        assert np.linalg.eigvalsh(Ze).min() > 0
    Ad = A.dense_block()
    assert np.abs(Ad - Ad.T).max() < 1e-13 * np.abs(Ad).max()
