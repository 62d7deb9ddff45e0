"""Pins of the oracle's essential-flux elimination and the pure-Neumann projection (NEXT-3).

P:1035: SPE10 prescribes u.n = (1,0,0).n on the whole boundary; the Schur
complement is then singular with the constants as nullspace, so every application of S^-1
is followed by an orthogonalization step.  Reading A21: elimination by identity
rows/columns, masked faces dropped from F(i), projection = subtract the plain mean.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import operators, solvers, space
from synth import Problem, cartesian_vertices, make_config, random_vector, perturbed_vertices

ALL3, ALL2 = 63, 15


def _darcy(dim, N, p, ess, eps=None, gamma=0.0, V=None, project=None):
    N = tuple(N) + ((1,) if dim == 2 else ())
    E = int(np.prod(N[:dim]))
    V = cartesian_vertices(dim, N[:dim]) if V is None else V
    eps = np.ones(E) if eps is None else eps
    pr = Problem("t", dim, N, p, "darcy", V, eps=eps, gamma=np.full(E, gamma),
                 essential=ess, project_mean=(ess == (1 << 2 * dim) - 1 and gamma == 0.0)
                 if project is None else project)
    return pr


@pytest.mark.parametrize("dim,N,p", [(2, (3, 2), 2), (3, (2, 3, 2), 2), (3, (1, 2, 1), 3)])
def test_mask_is_the_boundary_of_the_incidence(dim, N, p):
    """All sides essential <=> exactly the faces with one incident cell in D, and the
    count is the closed form sum_a prod_{b != a} n_b times 2."""
    m = space.essential_rt_mask(dim, N, p, (1 << 2 * dim) - 1)
    I, J, A = space.divergence_csr(dim, N, p)
    cnt = np.bincount(J, minlength=len(m))
    assert np.array_equal(m, cnt == 1)
    n = [N[a] * p for a in range(dim)]
    want = 2 * sum(int(np.prod([n[b] for b in range(dim) if b != a])) for a in range(dim))
    assert m.sum() == want
    # single sides: the x_a = min side has the faces whose only cell is on their + side
    for a in range(dim):
        lo = space.essential_rt_mask(dim, N, p, 1 << (2 * a))
        Dm = sp.csr_matrix((A, J, I))
        plus_only = np.asarray((Dm == -1).sum(axis=0)).ravel() == 1
        assert np.array_equal(lo, (cnt == 1) & plus_only & _component_mask(dim, N, p, a))


def _component_mask(dim, N, p, a):
    s = space.sizes(dim, N, p)
    m = np.zeros(s["n_rt"], bool)
    end = s["offs"][a + 1] if a + 1 < dim else s["n_rt"]
    m[s["offs"][a]:end] = True
    return m


@pytest.mark.parametrize("ess", [1, 2, 12, ALL3])
def test_eliminated_rows_are_identity_and_block_symmetric(ess):
    A = operators.Assembled(_darcy(3, (2, 2, 2), 2, ess, gamma=0.5))
    Ad = A.dense_block()
    assert np.abs(Ad - Ad.T).max() < 1e-14 * np.abs(Ad).max()
    b = np.flatnonzero(A.ess)
    assert len(b) > 0
    assert np.array_equal(Ad[b][:, b], np.eye(len(b)))
    assert not Ad[b].any(axis=0)[np.setdiff1d(np.arange(len(Ad)), b)].any()
    assert np.all(A.Mdiag[b] == 1.0)
    # unmasked rows of M are those of the natural-BC operator with the masked columns dropped
    A0 = operators.Assembled(_darcy(3, (2, 2, 2), 2, 0, gamma=0.5))
    f = np.flatnonzero(~A.ess)
    assert abs(A.M[f][:, f] - A0.M[f][:, f]).max() == 0.0


def test_pure_neumann_nullspace_and_singular_schur():
    """All sides essential, gamma = 0: the only null vector of A_hat is (u = 0, p~ = const)
    (reading A11), and S~ is a graph Laplacian: S~ 1 = 0, PSD with one zero eigenvalue."""
    A = operators.Assembled(_darcy(2, (4, 4), 2, ALL2))
    Ad = A.dense_block()
    w, V = np.linalg.eigh(Ad)
    k = np.abs(w) < 1e-10 * np.abs(w).max()
    assert k.sum() == 1
    v = V[:, k].ravel()
    assert np.abs(v[:A.n_rt]).max() < 1e-12
    q = v[A.n_rt:]
    assert np.ptp(q) < 1e-12 * np.abs(q).max()
    S = A.S.toarray()
    assert np.abs(S.sum(axis=1)).max() < 1e-12 * np.abs(S).max()
    ws = np.linalg.eigvalsh(S)
    assert (np.abs(ws) < 1e-10 * ws.max()).sum() == 1 and ws.min() > -1e-10 * ws.max()
    S2 = operators.schur_triple_product(A.D, A.Mdiag, A.Ctil)
    S2.eliminate_zeros()
    assert abs(A.S - S2).max() < 1e-13 * abs(S2).max()


def test_partial_sides_nonsingular_minres_matches_dense():
    pr = _darcy(2, (4, 3), 2, 1 | 4, gamma=0.0)     # x = 0 and y = 0 sides essential
    A = operators.Assembled(pr)
    n = A.n_rt + A.n_l2
    b = A.apply_block(random_vector(n, 3))
    x_ref = np.linalg.solve(A.dense_block(), b)
    P = solvers.BlockDiagPrecond(A, schur="chebyshev")
    x, it, conv, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-13, maxit=2000)
    assert conv and np.abs(x - x_ref).max() < 1e-9 * np.abs(x_ref).max()


@pytest.mark.parametrize("schur", ["chebyshev", "amg"])
def test_pure_neumann_minres_with_projection(schur):
    """with the projection after S^-1 MINRES converges on the singular system;
    the u part is unique and the p~ part is unique up to a constant (A16)."""
    pr = _darcy(3, (3, 3, 2), 2, ALL3, eps=10.0 ** random_vector(18, 5))
    A = operators.Assembled(pr)
    n = A.n_rt + A.n_l2
    xs = random_vector(n, 4)
    b = A.apply_block(xs)
    P = solvers.BlockDiagPrecond(A, schur=schur, amg_max_coarse=8)
    x, it, conv, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=3000)
    assert conv
    assert np.abs(x[:A.n_rt] - xs[:A.n_rt]).max() < 1e-8
    d = x[A.n_rt:] - xs[A.n_rt:]
    assert np.ptp(d) < 1e-8 * np.abs(xs[A.n_rt:]).max()


def test_uniform_flow_is_reproduced_exactly():
    """Darcy eps^-1 u + grad p = 0, div u = 0, u.n = (1,0,0).n on the boundary (SPE10's
    condition) with constant eps on a box mesh: u = (1,0,0) lies in RT_h and is the
    energy minimiser over the discretely divergence-free fields with that flux, so the mixed
    solution IS its interpolant — x-face DOFs = subcell-face areas (Piola; sum_j |I_j| h_j = 1),
    y/z-face DOFs = 0.  p = -x/eps + c, so the p~ = W p part is pinned up to W 1."""
    from oracle import basis1d
    N, p, eps = (2, 3, 2), 2, 2.5
    # non-uniform axis-aligned box mesh
    ax = [np.array([0.0, 0.3, 1.0]), np.array([0.0, 0.2, 0.7, 1.0]), np.array([0.0, 0.6, 1.0])]
    from synth.gen import tensor_vertices
    V = tensor_vertices(ax)
    E = 12
    pr = _darcy(3, N, p, ALL3, eps=np.full(E, eps), V=V)
    pr0 = _darcy(3, N, p, 0, eps=np.full(E, eps), V=V, project=False)
    A, A0 = operators.Assembled(pr), operators.Assembled(pr0)
    # subcell node coordinates along each axis (GLL nodes inside every element)
    xi = basis1d.gll_nodes(p)
    nodes = [np.append((a[:-1, None] + (a[1:] - a[:-1])[:, None] * xi[None, :-1]).ravel(), a[-1])
             for a in ax]
    widths = [np.diff(nd) for nd in nodes]
    s = space.sizes(3, N, p)
    n = s["n"]
    ustar = np.zeros(A.n_rt)
    area = np.outer(widths[2], widths[1])   # [K][J]
    for K in range(n[2]):
        for J in range(n[1]):
            for I in range(n[0] + 1):
                ustar[I + (n[0] + 1) * (J + n[1] * K)] = area[K, J]
    ub = np.where(A.ess, ustar, 0.0)
    # lifting with the natural-BC operator: b_I = -(A0 [u_b; 0])_I, b_b = u_b
    lift = A0.apply_block(np.concatenate([ub, np.zeros(A.n_l2)]))
    b = -lift
    b[:A.n_rt][A.ess] = ub[A.ess]
    P = solvers.BlockDiagPrecond(A)
    x, it, conv, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-13, maxit=4000)
    assert conv
    assert np.abs(x[:A.n_rt] - ustar).max() < 1e-9 * ustar.max()
    assert np.abs(A0.D @ x[:A.n_rt]).max() < 1e-9 * ustar.max()   # discretely div-free
