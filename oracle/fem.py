"""Element-level definitions by direct quadrature (oracle; test infrastructure).

P:84   Piola map:  V_h(kappa) = det(J)^-1 J V_h(kappa_hat)
P:85   reference RT space Q_{p,p-1,p-1} x Q_{p-1,p,p-1} x Q_{p-1,p-1,p}
P:117  L2: W_h(kappa) = det(J)^-1 W_h(kappa_hat)   (integral preserving)
P:133-139 eq.(matrices):  v^T M_beta u = (beta u, v);  q^T B_alpha u = (alpha div u, q);
                          r^T W_alpha q = (alpha q, r)
Quadrature: tensor Gauss-Legendre, Q = p+2 points per direction (reading A3).

Local numbering (reading A6):
  3D x-block  l_i(x) h_j(y) h_k(z) e_x   idx = i + (p+1)(j + p k)
     y-block  h_i(x) l_j(y) h_k(z) e_y   idx = i + p(j + (p+1)k)
     z-block  h_i(x) h_j(y) l_k(z) e_z   idx = i + p(j + p k)
  blocks stacked x, y(, z);  L2: h_a h_b h_c, idx = a + p(b + p c).
  2D analogous (x-block i + (p+1) j, y-block i + p j).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from . import basis1d


class RefTables:
    """Reference-element values of all local basis functions at the quadrature points."""

    def __init__(self, dim: int, p: int, Q: int):
        self.dim, self.p, self.Q = dim, p, Q
        xq, wq = basis1d.gl_rule(Q)
        xi = basis1d.gll_nodes(p)
        Bl = basis1d.lagrange(xi, xq)          # [Q, p+1]
        dBl = basis1d.lagrange_deriv(xi, xq)   # [Q, p+1]
        Bh = basis1d.histopolation(p, xq)      # [Q, p]
        self.xq, self.wq1 = xq, wq
        if dim == 2:
            # quad point q = qx + Q*qy
            qx, qy = np.meshgrid(np.arange(Q), np.arange(Q), indexing="xy")
            qx, qy = qx.ravel(), qy.ravel()
            self.pts = np.stack([xq[qx], xq[qy]], axis=1)
            self.w = wq[qx] * wq[qy]
            nq = Q * Q
            nx = (p + 1) * p
            Phi = np.zeros((nq, 2 * nx, 2))
            Div = np.zeros((nq, 2 * nx))
            for j in range(p):
                for i in range(p + 1):
                    m = i + (p + 1) * j
                    Phi[:, m, 0] = Bl[qx, i] * Bh[qy, j]
                    Div[:, m] = dBl[qx, i] * Bh[qy, j]
            for j in range(p + 1):
                for i in range(p):
                    m = nx + i + p * j
                    Phi[:, m, 1] = Bh[qx, i] * Bl[qy, j]
                    Div[:, m] = Bh[qx, i] * dBl[qy, j]
            Psi = np.zeros((nq, p * p))
            for b in range(p):
                for a in range(p):
                    Psi[:, a + p * b] = Bh[qx, a] * Bh[qy, b]
        else:
            qz, qy, qx = np.meshgrid(np.arange(Q), np.arange(Q), np.arange(Q), indexing="ij")
            qx, qy, qz = qx.ravel(), qy.ravel(), qz.ravel()   # q = qx + Q(qy + Q qz)
            self.pts = np.stack([xq[qx], xq[qy], xq[qz]], axis=1)
            self.w = wq[qx] * wq[qy] * wq[qz]
            nq = Q ** 3
            nc = (p + 1) * p * p
            Phi = np.zeros((nq, 3 * nc, 3))
            Div = np.zeros((nq, 3 * nc))
            for k in range(p):
                for j in range(p):
                    for i in range(p + 1):
                        m = i + (p + 1) * (j + p * k)
                        Phi[:, m, 0] = Bl[qx, i] * Bh[qy, j] * Bh[qz, k]
                        Div[:, m] = dBl[qx, i] * Bh[qy, j] * Bh[qz, k]
            for k in range(p):
                for j in range(p + 1):
                    for i in range(p):
                        m = nc + i + p * (j + (p + 1) * k)
                        Phi[:, m, 1] = Bh[qx, i] * Bl[qy, j] * Bh[qz, k]
                        Div[:, m] = Bh[qx, i] * dBl[qy, j] * Bh[qz, k]
            for k in range(p + 1):
                for j in range(p):
                    for i in range(p):
                        m = 2 * nc + i + p * (j + p * k)
                        Phi[:, m, 2] = Bh[qx, i] * Bh[qy, j] * Bl[qz, k]
                        Div[:, m] = Bh[qx, i] * Bh[qy, j] * dBl[qz, k]
            Psi = np.zeros((nq, p ** 3))
            for c in range(p):
                for b in range(p):
                    for a in range(p):
                        Psi[:, a + p * (b + p * c)] = Bh[qx, a] * Bh[qy, b] * Bh[qz, c]
        self.Phi, self.Div, self.Psi = Phi, Div, Psi
        self.n_rt = Phi.shape[1]
        self.n_l2 = Psi.shape[1]


@lru_cache(maxsize=32)
def ref_tables(dim: int, p: int, Q: int) -> RefTables:
    return RefTables(dim, p, Q)


def element_vertices(V: np.ndarray, dim: int, e_idx) -> np.ndarray:
    """Corner coordinates X[c][b][a] (3D) / X[b][a] (2D) of element (ex,ey[,ez])."""
    if dim == 2:
        ex, ey = e_idx
        return V[ey:ey + 2, ex:ex + 2, :]
    ex, ey, ez = e_idx
    return V[ez:ez + 2, ey:ey + 2, ex:ex + 2, :]


def jacobian(X: np.ndarray, pts: np.ndarray):
    """J[q] = dT/dx_hat at reference points for the (bi/tri)linear vertex map."""
    dim = pts.shape[1]
    N = [lambda t: 1.0 - t, lambda t: t]
    dN = [lambda t: -np.ones_like(t), lambda t: np.ones_like(t)]
    J = np.zeros((len(pts), dim, dim))
    if dim == 2:
        for b in range(2):
            for a in range(2):
                x = X[b, a]
                gx = dN[a](pts[:, 0]) * N[b](pts[:, 1])
                gy = N[a](pts[:, 0]) * dN[b](pts[:, 1])
                J[:, :, 0] += np.outer(gx, x)
                J[:, :, 1] += np.outer(gy, x)
    else:
        for c in range(2):
            for b in range(2):
                for a in range(2):
                    x = X[c, b, a]
                    gx = dN[a](pts[:, 0]) * N[b](pts[:, 1]) * N[c](pts[:, 2])
                    gy = N[a](pts[:, 0]) * dN[b](pts[:, 1]) * N[c](pts[:, 2])
                    gz = N[a](pts[:, 0]) * N[b](pts[:, 1]) * dN[c](pts[:, 2])
                    J[:, :, 0] += np.outer(gx, x)
                    J[:, :, 1] += np.outer(gy, x)
                    J[:, :, 2] += np.outer(gz, x)
    return J, np.linalg.det(J)


def physical_points(X: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """T(x_hat) for the vertex map (used for manufactured-solution loads)."""
    dim = pts.shape[1]
    N = [lambda t: 1.0 - t, lambda t: t]
    out = np.zeros((len(pts), dim))
    if dim == 2:
        for b in range(2):
            for a in range(2):
                out += np.outer(N[a](pts[:, 0]) * N[b](pts[:, 1]), X[b, a])
    else:
        for c in range(2):
            for b in range(2):
                for a in range(2):
                    out += np.outer(N[a](pts[:, 0]) * N[b](pts[:, 1]) * N[c](pts[:, 2]), X[c, b, a])
    return out


def check_geometry(detJ: np.ndarray):
    if np.any(detJ <= 0.0):
        raise ValueError("invalid mesh: det J <= 0 at a quadrature point")


def element_rt_mass(X, beta: float, ref: RefTables) -> np.ndarray:
    """M^e_mn = sum_q w_q beta phi_m(x_q) . phi_n(x_q) det J_q, with phi = J phi_hat / det J
    (P:84 Piola; P:135 eq. matrices)."""
    J, det = jacobian(X, ref.pts)
    check_geometry(det)
    A = np.einsum("qmc,qdc->qmd", ref.Phi, J)          # (J phi_hat)_d per basis function
    wt = ref.w * beta / det
    # sum over q and d written as one matrix product over the flattened (q, d) index
    Am = A.transpose(1, 0, 2).reshape(A.shape[1], -1)
    Aw = (A * wt[:, None, None]).transpose(1, 0, 2).reshape(A.shape[1], -1)
    return Aw @ Am.T


def element_l2_mass(X, c, ref: RefTables) -> np.ndarray:
    """W^e_ab = sum_q w_q c psi_a psi_b det J_q, psi = psi_hat / det J.
    c: a constant, or its values at the quadrature points (variable coefficient, NEXT-3)."""
    J, det = jacobian(X, ref.pts)
    check_geometry(det)
    wt = ref.w * c / det
    return (ref.Psi * wt[:, None]).T @ ref.Psi


def element_div_form(X, ref: RefTables) -> np.ndarray:
    """B^e_an = sum_q w_q psi_a (div phi_n) det J_q; div phi = div_hat phi_hat / det J
    (P:136 with alpha = 1)."""
    J, det = jacobian(X, ref.pts)
    check_geometry(det)
    wt = ref.w / det
    return (ref.Psi * wt[:, None]).T @ ref.Div
