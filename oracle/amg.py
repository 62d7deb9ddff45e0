"""AMG V-cycle approximation of S~^-1 (oracle; test infrastructure only — the product path never
imports this module).  NEXT-1 of SURVEY §8.

Paper: the Schur-complement block of the preconditioner is approximated by one AMG V-cycle
("one V-cycle of AMG"), hypre BoomerAMG on the GPU with l1-Jacobi smoothing
(P:900-901), Galerkin coarse operators.  The paper does not fix the coarsening,
interpolation, sweeps or coarse solve (reading A9).  Reading A9b (this build):

  * coarsening: deterministic aggregation of the structured subcell grid of the L2 space into
    3 x 3 (x 3) blocks (the last block of an axis may be shorter; an axis of extent 1 stays 1);
  * interpolation: smoothed aggregation, P = (I - omega D^-1 A) P_tent, P_tent the 0/1 aggregate
    indicator, omega = 4 / (3 lam), lam = max_i sum_j |a_ij| / a_ii (Gershgorin bound of D^-1 A);
  * coarse operators: Galerkin A_c = P^T A P;
  * smoother: l1-Jacobi, x <- x + D_l1^-1 (b - A x), D_l1 = diag(sum_j |a_ij|), nu sweeps before
    and nu after the coarse correction (symmetric, so the V-cycle is SPD);
  * coarsest level (<= max_coarse unknowns, or no axis left to coarsen): exact solve.

With 3-wide aggregates and a distance-1 smoother the coarse operators of a 7-point (5-point)
fine operator are 27-point (9-point) on the coarse grid, and stay so on every level.

Everything below is the plain algorithm with scipy sparse products: no fusion, no reordering.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def l2_cell_coords(dim, N, p):
    """Subcell coordinates (X, Y[, Z]) of every L2 row in the element-contiguous numbering
    e p^d + a + p b (+ p^2 c), e = ex + N_x (ey + N_y ez)."""
    nl = p ** dim
    E = int(np.prod(N[:dim]))
    i = np.arange(E * nl, dtype=np.int64)
    e, il = i // nl, i % nl
    ex = e % N[0]
    X = ex * p + il % p
    if dim == 2:
        ey = e // N[0]
        Y = ey * p + il // p
        return np.stack([X, Y], axis=1)
    ey = (e // N[0]) % N[1]
    ez = e // (N[0] * N[1])
    Y = ey * p + (il // p) % p
    Z = ez * p + il // (p * p)
    return np.stack([X, Y, Z], axis=1)


class Level:
    def __init__(self, A, dims, coords):
        self.A = A.tocsr()
        self.dims = tuple(int(d) for d in dims)
        self.coords = coords
        self.D = self.A.diagonal().copy()
        self.l1 = np.asarray(abs(self.A).sum(axis=1)).ravel()
        self.P = None
        self.omega = None


def _coarse_grid(dims, agg):
    return tuple((d + agg - 1) // agg for d in dims)


def build_hierarchy(S, coords, dims, agg=3, max_coarse=512, max_levels=25, coarse_solve=True,
                    pin=False):
    """Levels l = 0..L with A_0 = S; coords: the grid coordinates of the rows of S.
    coarse_solve=False skips the coarsest inverse (tests on singular operators).
    pin=True (singular S~ of the pure-Neumann problem, NEXT-3, reading A21): the coarsest
    solve fixes the last unknown at 0 and drops its equation (A_L without its last row and
    column inverted; the last entry of the correction is 0)."""
    levels = [Level(S, dims, coords)]
    while True:
        lv = levels[-1]
        n = lv.A.shape[0]
        cd = _coarse_grid(lv.dims, agg)
        if n <= max_coarse or cd == lv.dims or len(levels) >= max_levels:
            break
        # aggregate of each row and the lexicographic coarse numbering (x fastest)
        cc = lv.coords // agg
        J = cc[:, 0].copy()
        stride = 1
        for a in range(1, len(cd)):
            stride *= cd[a - 1]
            J += stride * cc[:, a]
        nc = int(np.prod(cd))
        Pt = sp.csr_matrix((np.ones(n), (np.arange(n), J)), shape=(n, nc))
        lam = float(np.max(lv.l1 / lv.D))
        lv.omega = 4.0 / (3.0 * lam)
        lv.P = (Pt - lv.omega * (sp.diags(1.0 / lv.D) @ (lv.A @ Pt))).tocsr()
        Ac = (lv.P.T @ lv.A @ lv.P).tocsr()
        # coarse coordinates in the coarse numbering
        ci = np.arange(nc, dtype=np.int64)
        ccoords = []
        rem = ci
        for a in range(len(cd)):
            ccoords.append(rem % cd[a])
            rem = rem // cd[a]
        levels.append(Level(Ac, cd, np.stack(ccoords, axis=1)))
    if coarse_solve:
        Ad = levels[-1].A.toarray()
        if pin:
            Ad[-1, :] = 0.0
            Ad[:, -1] = 0.0
            Ad[-1, -1] = 1.0
        Ainv = np.linalg.inv(Ad)
        if pin:   # the last unknown fixed at 0 and its (redundant) equation dropped:
            Ainv[-1, :] = 0.0   # e = [A_red^-1 b_red; 0] — B stays positive semidefinite with
            Ainv[:, -1] = 0.0   # B S~ = I on the mean-zero space for an exact solve
        levels[-1].Ainv = Ainv
    return levels


def vcycle(levels, b, nu=1, l=0):
    """One V-cycle x ~ A_l^-1 b from x = 0 (the approximation of S~^-1 when l = 0)."""
    lv = levels[l]
    if l == len(levels) - 1:
        return lv.Ainv @ b
    dl1inv = 1.0 / lv.l1
    x = np.zeros_like(b)
    for _ in range(nu):                       # pre-smoothing, l1-Jacobi
        x = x + dl1inv * (b - lv.A @ x)
    r = b - lv.A @ x                          # residual
    ec = vcycle(levels, lv.P.T @ r, nu, l + 1)   # restrict, coarse correction
    x = x + lv.P @ ec                         # prolongate
    for _ in range(nu):                       # post-smoothing
        x = x + dl1inv * (b - lv.A @ x)
    return x


class AMGSchur:
    """S^-1 = one V-cycle on S~ (drop-in for the Chebyshev polynomial in BlockDiagPrecond).

    slabs = [(z0, z1), ...] element-layer ranges along the last axis (reading A9c, the
    multi-rank build): S^-1 = block-Jacobi of one V-cycle per diagonal block S~[slab, slab]
    (slab-local aggregation of the block's own subcell grid; couplings between slabs dropped).
    In the element-contiguous L2 numbering every slab is one contiguous index range."""

    def __init__(self, asm, nu=2, max_coarse=512, pin=False, slabs=None, cheb_degree=1,
                 cheb_ratio=20.0, global_coarse=False):
        coords = l2_cell_coords(asm.dim, asm.N, asm.p)
        dims = [int(asm.N[a]) * asm.p for a in range(asm.dim)]
        self.nu = nu
        self.S = asm.S.tocsr()
        # cheb_degree >= 2 (reading A9d): S^-1 = the Chebyshev polynomial of degree cheb_degree
        # in B S~ (B = the V-cycle below, SPD with spectrum in (0, 1] for the symmetric l1-Jacobi
        # V-cycle) on [b / ratio, b], b = 1.1 — the Chebyshev-Jacobi recurrence of reading A10
        # with B in place of D^-1; degree 1 is the plain V-cycle.  With slabs (reading A9c) B is
        # block-Jacobi over a chain of slabs: two colours (even / odd slabs), each colour's
        # blocks decoupled, so the spectrum of B S~ is bounded by 2 (the additive-Schwarz
        # colouring bound, one per colour) and b = 2.2
        self.cheb_degree = int(cheb_degree)
        last = asm.dim - 1
        per_layer = int(np.prod(asm.N[:last])) * asm.p ** asm.dim
        if not slabs:
            slabs = [(0, int(asm.N[last]))]
        if self.cheb_degree >= 2:
            b_ = 1.1 if len(slabs) == 1 else 2.2
            a_ = b_ / float(cheb_ratio)
            self.theta, self.delta = 0.5 * (b_ + a_), 0.5 * (b_ - a_)
            self.sigma = self.theta / self.delta
        self.blocks = []
        S = asm.S.tocsr()
        for z0, z1 in slabs:
            a, b = z0 * per_layer, z1 * per_layer
            c = coords[a:b].copy()
            c[:, last] -= z0 * asm.p
            d = list(dims)
            d[last] = (z1 - z0) * asm.p
            # the pin only where the block is singular: a slab's diagonal block keeps the
            # interface couplings on its diagonal (S~_ii sums all face weights), so with two or
            # more slabs every block is nonsingular and is inverted as it is (reading A9c)
            lv = build_hierarchy(S[a:b, a:b], c, tuple(d), max_coarse=max_coarse,
                                 pin=pin and len(slabs) == 1)
            self.blocks.append((a, b, lv))
        self.levels = self.blocks[0][2] if len(self.blocks) == 1 else None
        # reading A9e (slabs only): a global coarse space couples the slabs — the indicator
        # vectors of the aggregates of a fixed coarse grid of the GLOBAL element grid (ceil(N_a /
        # C) elements per aggregate along axis a, C = 8 in 3D, 16 in 2D), R the aggregate-sum
        # restriction, A0 = R S~ R^T (the exact Galerkin operator, dense), B0 = R^T A0^-1 R, and
        # the inner preconditioner M (the block-Jacobi V-cycles, or their A9d polynomial) enters
        # the balancing (hybrid two-level) form, once per application of S^-1:
        #   S^-1 = B0 + (I - B0 S~) M (I - S~ B0),
        # symmetric, with S^-1 S~ = I on range(R^T) and its spectrum in (0, max(1, lam_max(M S~))].  The singular pure-Neumann S~ (pin) makes A0 singular
        # with the constants as its nullspace: its last unknown is fixed at 0 (as A21).
        self.global_coarse = bool(global_coarse) and len(slabs) > 1
        if self.global_coarse:
            C = 8 if asm.dim == 3 else 16
            ge = [max(1, -(-int(asm.N[a]) // C)) for a in range(asm.dim)]
            g = [gg * asm.p for gg in ge]
            cd = [-(-int(asm.N[a]) // gg) for a, gg in enumerate(ge)]
            agg = coords[:, 0] // g[0]
            stride = 1
            for a in range(1, asm.dim):
                stride *= cd[a - 1]
                agg = agg + stride * (coords[:, a] // g[a])
            n0 = int(np.prod(cd))
            self.R = sp.csr_matrix((np.ones(len(agg)), (agg, np.arange(len(agg)))),
                                   shape=(n0, len(agg)))
            A0 = (self.R @ S @ self.R.T).toarray()
            if pin:
                A0[-1, :] = 0.0
                A0[:, -1] = 0.0
                A0[-1, -1] = 1.0
            A0inv = np.linalg.inv(A0)
            if pin:
                A0inv[-1, :] = 0.0
                A0inv[:, -1] = 0.0
            self.A0inv = A0inv

    def B0(self, r):
        return self.R.T @ (self.A0inv @ (self.R @ r))

    def block_vcycles(self, r):
        out = np.empty_like(r)
        for a, b, lv in self.blocks:
            out[a:b] = vcycle(lv, r[a:b], self.nu)
        return out

    def vcycles(self, r):
        return self.block_vcycles(r)

    def __call__(self, r):
        """S^-1 r: the (block-Jacobi) V-cycles or their A9d polynomial M, wrapped in the balancing
        global coarse correction when global_coarse (A9e), step by step:
        e0 = B0 r, w = M (r - S~ e0), S^-1 r = e0 + w - B0 S~ w."""
        if not self.global_coarse:
            return self.inner(r)
        e0 = self.B0(r)
        w = self.inner(r - self.S @ e0)
        return e0 + w - self.B0(self.S @ w)

    def inner(self, r):
        if self.cheb_degree < 2:
            return self.vcycles(r)
        # r/d form, step by step: d_0 = B r / theta, y = d_0; r_i = r_{i-1} - S~ d_{i-1},
        # d_i = c1 d_{i-1} + c2 B r_i, y += d_i
        rho = 1.0 / self.sigma
        d = self.vcycles(r) / self.theta
        y = d.copy()
        res = r.copy()
        for _ in range(1, self.cheb_degree):
            res = res - self.S @ d
            rn = 1.0 / (2.0 * self.sigma - rho)
            d = (rn * rho) * d + (2.0 * rn / self.delta) * self.vcycles(res)
            y = y + d
            rho = rn
        return y
