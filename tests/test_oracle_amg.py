"""Pins for the oracle's AMG V-cycle (NEXT-1, reading A9b): closed forms of the 1D smoothed-
aggregation prolongator and Galerkin operator, stencil-width and constant-preservation
invariants, SPD-ness, single-level exactness and h-robust contraction."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import amg


def _poisson(dims, neumann=False):
    """7/5/3-point Laplacian (unit weights) on a structured grid, x fastest; Dirichlet-like
    rows keep the full diagonal 2d unless neumann (zero row sums)."""
    d = len(dims)
    n = int(np.prod(dims))
    idx = np.arange(n).reshape(dims[::-1])
    rows, cols, vals = [], [], []
    diag = np.zeros(n)
    for a in range(d):
        ax = d - 1 - a
        lo = np.take(idx, range(0, dims[a] - 1), axis=ax).ravel()
        hi = np.take(idx, range(1, dims[a]), axis=ax).ravel()
        rows += [lo, hi]; cols += [hi, lo]; vals += [-np.ones(lo.size)] * 2
        if neumann:
            np.add.at(diag, lo, 1.0); np.add.at(diag, hi, 1.0)
    if not neumann:
        diag[:] = 2.0 * d
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)) + sp.diags(diag)
    coords = np.stack(np.meshgrid(*[np.arange(m) for m in dims], indexing="ij"), -1)
    coords = coords.transpose(list(range(d))[::-1] + [d]).reshape(n, d)
    return A.tocsr(), coords


def test_1d_prolongator_and_galerkin_closed_form():
    # tridiag(-1, 2, -1): D = 2, Gershgorin lam = 2 -> omega = 2/3; interior SA column is the
    # hat (1/3, 2/3, 1, 2/3, 1/3) and P^T A P = (1/3) tridiag(-1, 2, -1)
    A, c = _poisson((27,))
    lv = amg.build_hierarchy(A, c, (27,), max_coarse=2)
    assert abs(lv[0].omega - 2.0 / 3.0) < 1e-15
    col = lv[0].P[:, 4].toarray().ravel()          # aggregate {12, 13, 14}
    ref = np.zeros(27)
    ref[11:16] = [1 / 3, 2 / 3, 1, 2 / 3, 1 / 3]
    assert np.abs(col - ref).max() < 1e-15
    Ac = lv[1].A.toarray()
    for J in range(2, 7):
        row = np.zeros(9)
        row[J - 1:J + 2] = [-1 / 3, 2 / 3, -1 / 3]
        assert np.abs(Ac[J] - row).max() < 1e-14


@pytest.mark.parametrize("dims", [(10, 9, 8), (13, 7)])
def test_coarse_stencils_stay_compact_and_symmetric(dims):
    A, c = _poisson(dims)
    lv = amg.build_hierarchy(A, c, dims, max_coarse=8)
    assert len(lv) >= 2
    for k in range(1, len(lv)):
        Ak = lv[k].A.tocoo()
        assert abs(Ak - Ak.T).max() < 1e-13 * abs(Ak).max()
        ci, cj = lv[k].coords[Ak.row], lv[k].coords[Ak.col]
        assert np.abs(ci - cj).max() <= 1                    # 27-point (9-point) coarse stencil
        assert np.diff(lv[k].A.indptr).max() <= 3 ** len(dims)


def test_constants_preserved_on_neumann_laplacian():
    # zero row sums: P 1 = 1 - omega D^-1 A 1 = 1, so every Galerkin level keeps A_l 1 = 0
    dims = (12, 10, 9)
    A, c = _poisson(dims, neumann=True)
    assert np.abs(A @ np.ones(A.shape[0])).max() == 0
    lv = amg.build_hierarchy(A, c, dims, max_coarse=20, coarse_solve=False)
    for k in range(len(lv) - 1):
        nc = lv[k + 1].A.shape[0]
        assert np.abs(lv[k].P @ np.ones(nc) - 1.0).max() < 1e-13
        assert np.abs(lv[k + 1].A @ np.ones(nc)).max() < 1e-12 * abs(lv[k + 1].A).max()


def test_single_level_is_exact_and_vcycle_spd():
    from synth import make_config
    from oracle import operators
    asm = operators.Assembled(make_config("c2", N=(2, 2, 2), p=2))
    big = amg.AMGSchur(asm, max_coarse=10 ** 6)
    assert len(big.levels) == 1
    r = np.random.default_rng(0).standard_normal(asm.n_l2)
    assert np.abs(big(r) - np.linalg.solve(asm.S.toarray(), r)).max() < 1e-10 * np.abs(big(r)).max()
    ml = amg.AMGSchur(asm, max_coarse=4)
    assert len(ml.levels) >= 2
    B = np.stack([ml(e) for e in np.eye(asm.n_l2)], axis=1)
    assert np.abs(B - B.T).max() < 1e-12 * np.abs(B).max()
    assert np.linalg.eigvalsh(0.5 * (B + B.T)).min() > 0


def _contraction(dims, its=25, nu=2):
    A, c = _poisson(dims)
    lv = amg.build_hierarchy(A, c, dims, max_coarse=64)
    x = np.random.default_rng(1).standard_normal(A.shape[0])
    rate = 0.0
    for _ in range(its):   # power iteration on the error propagator I - B A
        y = x - amg.vcycle(lv, A @ x, nu)
        rate = np.linalg.norm(y) / np.linalg.norm(x)
        x = y / np.linalg.norm(y)
    return rate


def test_vcycle_contraction_is_h_robust():
    # 3D Poisson, 2 l1-Jacobi sweeps: ~0.71 at 18^3 and ~0.76 at 36^3 (3 and 4 levels); a
    # wrong omega, a missing smoothing step or a transposed P pushes it to >= 0.9
    r1 = _contraction((18, 18, 18))
    r2 = _contraction((36, 36, 36))
    assert r1 < 0.8 and r2 < 0.8, (r1, r2)
    assert r2 < r1 + 0.1, (r1, r2)
    assert _contraction((18, 18, 18), nu=1) > r1      # more smoothing contracts more


def test_minres_with_amg_beats_chebyshev_on_config2():
    from synth import make_config, random_vector
    from oracle import operators, solvers
    asm = operators.Assembled(make_config("c2"))
    n = asm.n_rt + asm.n_l2
    b = asm.apply_block(random_vector(n, 2))
    its = {}
    for schur in ("chebyshev", "amg"):
        P = solvers.BlockDiagPrecond(asm, schur=schur, amg_nu=2)
        x, it, conv, _ = solvers.minres(asm.apply_block, P.apply, b, rtol=1e-10, maxit=3000)
        assert conv
        its[schur] = it
    assert its["amg"] < its["chebyshev"], its


def test_block_jacobi_amg_of_slabs():
    """Reading A9c (multi-rank S^-1): the block-Jacobi of per-slab V-cycles.  With a one-level
    hierarchy per block (max_coarse >= block size) every block solve is exact, so it must equal
    the independent block-diagonal solve S~[slab, slab]^-1 v; with deeper hierarchies it stays
    symmetric positive definite."""
    import scipy.sparse.linalg as spla
    from oracle import amg as amgmod, operators
    from synth import make_config, random_vector
    pr = make_config("c2", N=(3, 3, 5), p=2)
    A = operators.Assembled(pr)
    slabs = [(0, 2), (2, 3), (3, 5)]
    per = 3 * 3 * 8
    v = random_vector(A.n_l2, 3)
    exact = amgmod.AMGSchur(A, max_coarse=10 ** 6, slabs=slabs)
    z = exact(v)
    S = A.S.tocsc()
    for z0, z1 in slabs:
        a, b = z0 * per, z1 * per
        zb = spla.spsolve(S[a:b, a:b], v[a:b])
        assert np.abs(z[a:b] - zb).max() < 1e-11 * np.abs(zb).max()
    deep = amgmod.AMGSchur(A, max_coarse=8, slabs=slabs)
    n = A.n_l2
    Bm = np.column_stack([deep(e) for e in np.eye(n)])
    assert np.abs(Bm - Bm.T).max() < 1e-12 * np.abs(Bm).max()
    assert np.linalg.eigvalsh(0.5 * (Bm + Bm.T)).min() > 0


@pytest.mark.parametrize("k,ratio", [(2, 20.0), (3, 20.0), (4, 30.0)])
def test_chebyshev_accelerated_vcycle(k, ratio):
    """Reading A9d: S^-1 = the degree-k Chebyshev polynomial in B S~ on [1.1 / ratio, 1.1].
    With a one-level hierarchy (B = S~^-1 exactly, B S~ = I) the r/d recurrence must reduce to
    the closed form (1 - T_k(s1) / T_k(s0)) S~^-1, s0 = (b + a) / (b - a), s1 = (b + a - 2) / (b - a)
    (the residual polynomial at the eigenvalue 1); with a deep hierarchy it is SPD and the
    preconditioned Schur operator is better conditioned than with one V-cycle."""
    import scipy.sparse.linalg as spla
    from numpy.polynomial import chebyshev as cheb
    from oracle import amg as amgmod, operators
    from synth import make_config, random_vector
    A = operators.Assembled(make_config("c2", N=(3, 3, 3), p=2))
    v = random_vector(A.n_l2, 5)
    exact = amgmod.AMGSchur(A, max_coarse=10 ** 6, cheb_degree=k, cheb_ratio=ratio)
    b, a = 1.1, 1.1 / ratio
    s0, s1 = (b + a) / (b - a), (b + a - 2.0) / (b - a)
    Tk = lambda t: cheb.chebval(t, [0] * k + [1])
    ref = (1.0 - Tk(s1) / Tk(s0)) * spla.spsolve(A.S.tocsc(), v)
    assert np.abs(exact(v) - ref).max() < 1e-11 * np.abs(ref).max()
    # heterogeneous coefficients (config 3's jittered mesh, contrast 10^4): one V-cycle leaves
    # cond(B S~) ~ 4 here, the polynomial brings it down
    A = operators.Assembled(make_config("c3", N=(4, 4, 4), p=2))
    deep = amgmod.AMGSchur(A, max_coarse=8, cheb_degree=k, cheb_ratio=ratio)
    one = amgmod.AMGSchur(A, max_coarse=8)
    n = A.n_l2
    Bm = np.column_stack([deep(e) for e in np.eye(n)])
    assert np.abs(Bm - Bm.T).max() < 1e-12 * np.abs(Bm).max()
    assert np.linalg.eigvalsh(0.5 * (Bm + Bm.T)).min() > 0
    S = A.S.toarray()
    B1 = np.column_stack([one(e) for e in np.eye(n)])
    def cond(Bx):   # spectrum of B S~ (similar to the SPD S^1/2 B S^1/2)
        lam = np.sort(np.linalg.eigvals(Bx @ S).real)
        assert lam[0] > 0
        return lam[-1] / lam[0]
    assert cond(Bm) < cond(B1), (cond(Bm), cond(B1))


def test_slab_block_jacobi_spectrum_bound():
    """Reading A9d with slabs (A9c): the block-Jacobi B over a chain of slabs has spectrum of
    B S~ in (0, 2] — checked with exact slab solves (one-level hierarchies, B = blockdiag
    S~[slab, slab]^-1) and with V-cycles on a 10^4-contrast mesh; it exceeds 1.1 (so the
    single-block interval would not cover it), which is why the slab polynomial takes b = 2.2."""
    from oracle import amg as amgmod, operators
    from synth import make_config
    A = operators.Assembled(make_config("c3", N=(3, 3, 6), p=2))
    S = A.S.toarray()
    n = A.n_l2
    for mc, bounds in [(10 ** 6, [(0, 2), (2, 4), (4, 6)]), (8, [(0, 3), (3, 6)]),
                       (8, [(0, 1), (1, 2), (2, 4), (4, 6)])]:
        B = amgmod.AMGSchur(A, max_coarse=mc, slabs=bounds)
        Bm = np.column_stack([B(e) for e in np.eye(n)])
        lam = np.sort(np.linalg.eigvals(Bm @ S).real)
        assert lam[0] > 0 and lam[-1] <= 2.0 + 1e-10, (mc, bounds, lam[0], lam[-1])
        if mc > n:
            assert lam[-1] > 1.1


def test_pinned_coarse_solve_spectrum():
    """Reading A21 (pure-Neumann S~, constants in its nullspace): the pinned coarsest solve fixes
    the last unknown at 0 and drops its equation, so with an exact one-level hierarchy
    B S~ x = x - x_last 1 — eigenvalues exactly {0, 1} — and with a deep hierarchy the spectrum
    of B S~ stays in [0, 1] (the interval the A9d polynomial assumes).  The identity-row pin
    alone (without dropping the equation) overshoots 1."""
    from oracle import amg as amgmod, operators
    from synth import make_config
    pr = make_config("c3", N=(3, 3, 4), p=2)
    pr.essential, pr.project_mean, pr.gamma = 63, True, np.zeros(pr.E)
    A = operators.Assembled(pr)
    S = A.S.toarray()
    n = A.n_l2
    assert np.abs(S @ np.ones(n)).max() < 1e-10 * np.abs(S).max()   # singular: constants
    for mc in (10 ** 6, 16):
        B = amgmod.AMGSchur(A, max_coarse=mc, pin=True)
        Bm = np.column_stack([B(e) for e in np.eye(n)])
        lam = np.sort(np.linalg.eigvals(Bm @ S).real)
        assert lam[0] > -1e-12 and lam[-1] < 1.0 + 1e-10, (mc, lam[0], lam[-1])
        if mc > n:
            x = np.arange(n, dtype=float) % 7
            assert np.abs(Bm @ (S @ x) - (x - x[-1])).max() < 1e-10 * np.abs(x).max()
    lv = amgmod.build_hierarchy(A.S.tocsr(), amgmod.l2_cell_coords(3, pr.N, 2), (6, 6, 8),
                                max_coarse=10 ** 6, coarse_solve=False)
    Ad = lv[-1].A.toarray()
    Ad[-1, :] = 0.0
    Ad[:, -1] = 0.0
    Ad[-1, -1] = 1.0
    lam = np.linalg.eigvals(np.linalg.inv(Ad) @ S).real
    assert lam.max() > 1.01


@pytest.mark.parametrize("name,N,p,bounds,pin", [
    ("c3", (3, 3, 6), 2, [(0, 2), (2, 4), (4, 6)], False),
    ("c2", (4, 3, 5), 2, [(0, 3), (3, 5)], False),
    ("c1", (6, 7), 2, [(0, 3), (3, 7)], False),
    ("c3", (3, 3, 4), 2, [(0, 2), (2, 4)], True)])
def test_global_coarse_balancing(name, N, p, bounds, pin):
    """Reading A9e: B = B0 + (I - B0 S~) B_bj (I - S~ B0), B0 = R^T A0^-1 R, A0 = R S~ R^T.
    Pins: (i) A0 equals the brute-force Galerkin sums sum_{i in I, j in J} S~_ij; (ii) B S~ is
    the identity on range(R^T) (a wrong A0 or R breaks it; with pin: modulo the constants);
    (iii) B is symmetric positive semidefinite (definite without pin) and the spectrum of B S~ lies
    in [0, 2] (the interval the A9d polynomial takes, b = 2.2)."""
    from oracle import amg as amgmod, operators
    from synth import make_config
    pr = make_config(name, N=N, p=p)
    if pin:
        pr.essential, pr.project_mean, pr.gamma = 63, True, np.zeros(pr.E)
    A = operators.Assembled(pr)
    S = A.S.toarray()
    n = A.n_l2
    B = amgmod.AMGSchur(A, max_coarse=8, slabs=bounds, global_coarse=True, pin=pin)
    R = B.R.toarray()
    agg = R.argmax(axis=0)
    A0 = np.zeros((R.shape[0], R.shape[0]))
    for i in range(n):
        for j in np.nonzero(S[i])[0]:
            A0[agg[i], agg[j]] += S[i, j]
    ref = (B.R @ A.S @ B.R.T).toarray()
    assert np.abs(A0 - ref).max() < 1e-12 * np.abs(ref).max()
    Bm = np.column_stack([B(e) for e in np.eye(n)])
    assert np.abs(Bm - Bm.T).max() < 1e-11 * np.abs(Bm).max()
    RT = R.T
    E = Bm @ S @ RT
    if pin:   # the constants are in the nullspace: compare after removing the mean
        E = E - E.mean(axis=0, keepdims=True)
        RT = RT - RT.mean(axis=0, keepdims=True)
    assert np.abs(E - RT).max() < 1e-10, np.abs(E - RT).max()
    lam = np.sort(np.linalg.eigvals(Bm @ S).real)
    assert lam[0] > -1e-10 and lam[-1] < 2.0 + 1e-9, (lam[0], lam[-1])
    if not pin:
        assert np.linalg.eigvalsh(0.5 * (Bm + Bm.T)).min() > 0
