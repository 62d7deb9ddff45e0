"""Preconditioner and MINRES (oracle; test infrastructure).

P:411-421 Remark: B = diag(tau M~, S~); S^-1 = approximate inverse of S~.
P:669 / P:889: S^-1 is one AMG V-cycle in the paper; this build's slice uses a fixed
Chebyshev-Jacobi polynomial in S~ (reading A9/A10), identical on the GPU.
P:169: MINRES; relative tolerance 1e-12 (preconditioned norm, reading A8).
"""
from __future__ import annotations

import math

import numpy as np


def chebyshev_jacobi(S, r, degree: int, ratio: float, lam_max: float = 2.0):
    """k-step Chebyshev semi-iteration for S y = r, Jacobi-scaled, y0 = 0, on the
    interval [lam_max/ratio, lam_max] (reading A10; Saad, Iterative Methods, Alg. 12.1)."""
    Dinv = 1.0 / S.diagonal()
    a, b = lam_max / ratio, lam_max
    theta, delta = 0.5 * (b + a), 0.5 * (b - a)
    sigma = theta / delta
    rho = 1.0 / sigma
    r = r.copy()
    y = np.zeros_like(r)
    d = Dinv * r / theta
    for k in range(degree):
        y = y + d
        if k == degree - 1:
            break
        r = r - S @ d
        rho_new = 1.0 / (2.0 * sigma - rho)
        d = rho_new * rho * d + (2.0 * rho_new / delta) * (Dinv * r)
        rho = rho_new
    return y


class BlockDiagPrecond:
    """P^-1 = diag((tau M~)^-1, S^-1)."""

    def __init__(self, asm, tau=1.0, degree=4, ratio=30.0, exact_schur=False, exact_blocks=False,
                 schur="chebyshev", amg_nu=2, amg_max_coarse=512, project_mean=None,
                 amg_cheb_degree=1, amg_cheb_ratio=20.0,
                 amg_slabs=None, amg_global_coarse=False):
        self.asm, self.tau, self.degree, self.ratio = asm, tau, degree, ratio
        # NEXT-3: with pure-Neumann (all-essential flux) Darcy and gamma = 0 the
        # Schur complement is singular with the constants as nullspace, so every application of
        # S^-1 is followed by an orthogonalization step: subtract the plain mean of the
        # coefficient vector (reading A11/A21)
        if project_mean is None:
            project_mean = bool(getattr(asm.prob, "project_mean", False))
        self.project_mean = project_mean
        self.amg = None
        if schur == "amg":   # NEXT-1: one AMG V-cycle on S~ (reading A9b)
            from .amg import AMGSchur
            self.amg = AMGSchur(asm, nu=amg_nu, max_coarse=amg_max_coarse, pin=project_mean,
                                cheb_degree=amg_cheb_degree, cheb_ratio=amg_cheb_ratio,
                                slabs=amg_slabs, global_coarse=amg_global_coarse)
        self.n_rt = asm.n_rt
        self.exact_schur = exact_schur
        self.exact_blocks = exact_blocks
        if exact_schur or exact_blocks:
            import scipy.sparse.linalg as spla
            if exact_blocks:   # Prop 2.1/2.2: A = M, S = C + D M^-1 D^T exactly
                Minv = np.linalg.inv(asm.M.toarray())
                Zd = np.zeros((asm.n_l2, asm.n_l2))
                nl = asm.p ** asm.dim
                for e, Ze in enumerate(asm.Z):
                    Zd[e * nl:(e + 1) * nl, e * nl:(e + 1) * nl] = Ze
                Dd = asm.D.toarray()
                self.Sfull = Zd + Dd @ Minv @ Dd.T
                self.Mfull = asm.M.toarray()
            else:
                self._lu = spla.splu(asm.S.tocsc())

    def apply(self, v):
        vu, vq = v[: self.n_rt], v[self.n_rt:]
        if self.exact_blocks:
            zu = np.linalg.solve(self.tau * self.Mfull, vu)
            zq = np.linalg.solve(self.Sfull, vq)
        else:
            zu = vu / (self.tau * self.asm.Mdiag)
            if self.exact_schur:
                zq = self._lu.solve(vq)
            elif self.amg is not None:
                zq = self.amg(vq)
            else:
                zq = chebyshev_jacobi(self.asm.S, vq, self.degree, self.ratio)
            if self.project_mean:
                zq = zq - zq.mean()
        return np.concatenate([zu, zq])


class Breakdown(RuntimeError):
    pass


def minres(apply_A, apply_Pinv, b, rtol=1e-12, maxit=1000):
    """Preconditioned MINRES, Elman-Silvester-Wathen form, x0 = 0
    (SURVEY.md §8(c) step 10). Returns x, iterations, converged, |eta|/gamma_1 history."""
    n = len(b)
    x = np.zeros(n)
    v_old = np.zeros(n)
    w_old = np.zeros(n)
    w = np.zeros(n)
    v = b.copy()
    z = apply_Pinv(v)
    g2 = float(np.dot(z, v))
    if g2 < 0:
        raise Breakdown("preconditioner not SPD")
    gamma = math.sqrt(g2)
    if gamma == 0.0:
        return x, 0, True, [0.0]
    gamma0 = gamma
    gamma_old = 1.0
    eta = gamma
    s_old = s = 0.0
    c_old = c = 1.0
    hist = [1.0]
    it = 0
    conv = False
    for j in range(1, maxit + 1):
        z = z / gamma
        Az = apply_A(z)
        delta = float(np.dot(Az, z))
        v_new = Az - (delta / gamma) * v - (gamma / gamma_old) * v_old
        z_new = apply_Pinv(v_new)
        g2 = float(np.dot(z_new, v_new))
        if g2 < 0:
            raise Breakdown("preconditioner not SPD")
        gamma_new = math.sqrt(g2)
        a0 = c * delta - c_old * s * gamma
        a1 = math.hypot(a0, gamma_new)
        a2 = s * delta + c_old * c * gamma
        a3 = s_old * gamma
        c_new = a0 / a1
        s_new = gamma_new / a1
        w_new = (z - a3 * w_old - a2 * w) / a1
        x = x + c_new * eta * w_new
        eta = -s_new * eta
        hist.append(abs(eta) / gamma0)
        it = j
        # rotate
        v_old, v = v, v_new
        z = z_new
        gamma_old, gamma = gamma, gamma_new
        w_old, w = w, w_new
        c_old, c = c, c_new
        s_old, s = s, s_new
        if abs(eta) <= rtol * gamma0:
            conv = True
            break
        if gamma_new == 0.0:
            conv = True
            break
    return x, it, conv, hist


# --------------------------------------------------------------------------------------------
# NEXT-4: block-triangular preconditioner + GMRES (P:423-438 Remark).
class BlockTriPrecond:
    """B = [tau M~, D^T; 0, -S^]  (upper block-triangular, P:427-433 with the sign of this
    build's A = [M, D^T; D, -Z], whose Schur complement is -(Z + D M^-1 D^T) = -S).
    B^-1 v:  z_q = -S^-1 v_q ;  z_u = (tau M~)^-1 (v_u - D^T z_q).
    With exact blocks (M, S) B^-1 A has the single eigenvalue 1 and a degree-2 minimal
    polynomial, so GMRES converges in at most two iterations."""

    def __init__(self, asm, tau=1.0, degree=4, ratio=30.0, schur="chebyshev", exact_blocks=False,
                 amg_nu=2, amg_max_coarse=512, amg_cheb_degree=1, amg_cheb_ratio=20.0):
        self.asm, self.tau = asm, tau
        self.diag = BlockDiagPrecond(asm, tau=tau, degree=degree, ratio=ratio, schur=schur,
                                     exact_blocks=exact_blocks, amg_nu=amg_nu,
                                     amg_max_coarse=amg_max_coarse, project_mean=False,
                                     amg_cheb_degree=amg_cheb_degree,
                                     amg_cheb_ratio=amg_cheb_ratio)
        self.exact_blocks = exact_blocks
        self.n_rt = asm.n_rt

    def apply(self, v):
        vu, vq = v[: self.n_rt], v[self.n_rt:]
        d = self.diag
        if self.exact_blocks:
            zq = -np.linalg.solve(d.Sfull, vq)
            zu = np.linalg.solve(self.tau * d.Mfull, vu - self.asm.D.T @ zq)
        else:
            zq = -d.apply(np.concatenate([np.zeros(self.n_rt), vq]))[self.n_rt:]
            zu = (vu - self.asm.D.T @ zq) / (self.tau * self.asm.Mdiag)
        return np.concatenate([zu, zq])


def gmres(apply_A, apply_Binv, b, rtol=1e-12, restart=30, maxit=1000):
    """Right-preconditioned restarted GMRES(m), x0 = 0 (Saad, Iterative Methods, Alg. 9.5):
    Arnoldi on A B^-1 with classical Gram-Schmidt applied twice, Givens rotations on the
    Hessenberg matrix; stops when the residual of the least-squares problem |g_{j+1}| (= the
    true residual norm ||b - A x|| in exact arithmetic, right preconditioning) <= rtol ||b||.
    Returns x, total iterations, converged, residual history."""
    n = len(b)
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return x, 0, True, [0.0]
    hist = [1.0]
    it = 0
    while it < maxit:
        r = b - apply_A(x)
        beta = float(np.linalg.norm(r))
        if beta <= rtol * bnorm:
            return x, it, True, hist
        m = restart
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        conv = False
        for j in range(m):
            w = apply_A(apply_Binv(V[j]))
            for _ in range(2):                      # CGS2
                h = V[: j + 1] @ w
                w = w - V[: j + 1].T @ h
                H[: j + 1, j] += h
            H[j + 1, j] = float(np.linalg.norm(w))
            if H[j + 1, j] > 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                       # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = math.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            k = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if abs(g[j + 1]) <= rtol * bnorm or it >= maxit:
                conv = abs(g[j + 1]) <= rtol * bnorm
                break
        # x += B^-1 V_k y,  H[:k,:k] y = g[:k]  (back substitution)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + apply_Binv(V[:k].T @ y)
        if conv:
            return x, it, True, hist
    return x, it, False, hist
