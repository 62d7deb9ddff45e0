"""Assembled operators of the transformed saddle-point system (oracle; test infrastructure).

P:207-211 eq.(transformed-system):  A = [[M_beta, D^T], [D, -W_alpha^-1]]
P:517-520 eq.(transformed-system-darcy): A' = [[M_{1/eps}, D^T], [D, -W^-1 W_gamma W^-1]]
P:451-456 eq.(approx-schur): M~ = diag(M_beta), W~ = diag(W_alpha), S~ = W~^-1 + D M~^-1 D^T
P:466-471 eq.(approx-schur-entries) entry formula of S~
P:555  Darcy: W^-1 W_gamma W^-1 approximated by the product of the (reciprocal) diagonals
P:552, P:761 (NEXT-3): general (not piecewise-constant) gamma keeps the full (2,2) block
       W^-1 W_gamma W^-1 (two W^-1 per apply); reading A22: gamma is the trilinear (Q_1)
       field of per-vertex values, evaluated at the quadrature points
P:886  S~ via the sparse triple product D M~^-1 D^T
NEXT-3 (reading A21): essential flux conditions on whole domain sides by
elimination — identity rows/columns for the prescribed RT DOFs (u_b), which are dropped from
D's columns and from the face sets F(i) of S~; M~ = 1 there (the diagonal of the eliminated
(1,1) block).

Everything is assembled from dense element matrices computed by direct
quadrature (fem.py); library primitives used: scipy.sparse products,
scipy.linalg Cholesky (cho_factor/cho_solve).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import fem, space


def mass_weight(prob, e: int) -> float:
    """beta_e (grad-div) or 1/eps_e (Darcy, M_{1/eps})."""
    if prob.kind == "grad_div":
        return float(prob.beta[e])
    return 1.0 / float(prob.eps[e])


def _check_coeffs(prob):
    if prob.kind == "grad_div":
        if np.any(prob.alpha <= 0) or np.any(prob.beta <= 0):
            raise ValueError("coefficient error: alpha, beta must be > 0")
    else:
        if np.any(prob.eps <= 0) or np.any(prob.gamma < 0):
            raise ValueError("coefficient error: eps > 0, gamma >= 0 required")
        gv = getattr(prob, "gamma_vertex", None)
        if gv is not None and np.any(gv < 0):
            raise ValueError("coefficient error: gamma >= 0 required")


class Assembled:
    """Global objects for one Problem, all in canonical numbering."""

    def __init__(self, prob, with_schur: bool = True):
        _check_coeffs(prob)
        self.prob = prob
        dim, N, p = prob.dim, prob.N, prob.p
        self.dim, self.N, self.p = dim, N, p
        ref = fem.ref_tables(dim, p, prob.nq)
        s = space.sizes(dim, N, p)
        self.n_rt = s["n_rt"]
        E = prob.E
        nl = p ** dim
        self.n_l2 = E * nl
        rows, cols, vals = [], [], []
        self.Z = []          # dense per-element (2,2) block Z_e
        self.Wdiag = np.zeros(self.n_l2)   # diag of W_alpha (grad-div) / W (Darcy)
        self.Wgdiag = np.zeros(self.n_l2)  # diag of W_gamma (Darcy)
        for e in range(E):
            X = fem.element_vertices(prob.vertices, dim, space.element_index(dim, N, e))
            Me = fem.element_rt_mass(X, mass_weight(prob, e), ref)
            g = space.rt_local_to_global(dim, N, p, e)
            rows.append(np.repeat(g, len(g)))
            cols.append(np.tile(g, len(g)))
            vals.append(Me.ravel())
            sl = slice(e * nl, (e + 1) * nl)
            if prob.kind == "grad_div":
                We = fem.element_l2_mass(X, float(prob.alpha[e]), ref)
                cf = sla.cho_factor(We)
                Ze = sla.cho_solve(cf, np.eye(nl))          # W_alpha^-1
                self.Wdiag[sl] = np.diag(We)
            else:
                We = fem.element_l2_mass(X, 1.0, ref)
                Gv = getattr(prob, "gamma_vertex", None)
                if Gv is not None:   # general gamma (NEXT-3, reading A22): trilinear vertex
                    Ge = fem.element_vertices(Gv[..., None], dim, space.element_index(dim, N, e))
                    gq = fem.physical_points(Ge, ref.pts)[:, 0]    # field at the quadrature points
                    Wg = fem.element_l2_mass(X, gq, ref)
                else:
                    Wg = fem.element_l2_mass(X, float(prob.gamma[e]), ref)
                cf = sla.cho_factor(We)
                Ze = sla.cho_solve(cf, Wg @ sla.cho_solve(cf, np.eye(nl)))  # W^-1 W_g W^-1
                self.Wdiag[sl] = np.diag(We)
                self.Wgdiag[sl] = np.diag(Wg)
            self.Z.append(Ze)
        self.M = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                               shape=(self.n_rt, self.n_rt))
        I, J, A = space.divergence_csr(dim, N, p)
        self.D = sp.csr_matrix((A, J, I), shape=(self.n_l2, self.n_rt))
        self.Dptr, self.Dcol, self.Dval = I, J, A   # Algorithm 1's D (unmasked)
        # essential flux sides (NEXT-3): A_hat = [[F M F + B, F D^T], [D F, -Z]], F = diag(free),
        # B = diag(essential)
        self.essential = int(getattr(prob, "essential", 0) or 0)
        self.ess = space.essential_rt_mask(dim, N, p, self.essential)
        if self.ess.any():
            Fm = sp.diags((~self.ess).astype(float))
            self.M = (Fm @ self.M @ Fm + sp.diags(self.ess.astype(float))).tocsr()
            self.D = (self.D @ Fm).tocsr()
        self.Mdiag = self.M.diagonal().copy()                 # M~
        if prob.kind == "grad_div":
            self.Ctil = 1.0 / self.Wdiag                     # W~^-1
        else:
            self.Ctil = self.Wgdiag / self.Wdiag ** 2        # diag(W)^-1 diag(W_g) diag(W)^-1
        if with_schur:
            self.S = schur_entry_formula(self.Dptr, self.Dcol, self.Dval, self.Mdiag, self.Ctil,
                                         skip=self.ess)

    # --- block operator -------------------------------
    def apply_Z(self, q):
        nl = self.p ** self.dim
        out = np.empty_like(q)
        for e, Ze in enumerate(self.Z):
            out[e * nl:(e + 1) * nl] = Ze @ q[e * nl:(e + 1) * nl]
        return out

    def apply_block(self, x):
        u, q = x[: self.n_rt], x[self.n_rt:]
        yu = self.M @ u + self.D.T @ q
        yq = self.D @ u - self.apply_Z(q)
        return np.concatenate([yu, yq])

    def dense_block(self):
        n = self.n_rt + self.n_l2
        if n > 6000:
            raise ValueError("dense block only for tiny meshes")
        Zd = sla.block_diag(*self.Z)
        return np.block([[self.M.toarray(), self.D.T.toarray()],
                         [self.D.toarray(), -Zd]])


def schur_entry_formula(Dptr, Dcol, Dval, Mdiag, Ctil, skip=None) -> sp.csr_matrix:
    """S~ from eq.(approx-schur-entries):
    S_ii = C~_ii + sum_{k in F(i)} 1/M~_kk ; S_ij = -1/M~_kk if i, j share face k.
    F(i) and the cells of a face are read off the incidence D; columns sorted.
    skip: faces removed from every F(i) (eliminated essential-flux DOFs, NEXT-3)."""
    n_l2 = len(Dptr) - 1
    if skip is not None and np.any(skip):
        keep = ~skip[Dcol]
        Dcol, Dval = Dcol[keep], Dval[keep]
        cnt = np.add.reduceat(keep.astype(np.int64), Dptr[:-1]) if len(keep) else np.zeros(0, np.int64)
        Dptr = np.concatenate([[0], np.cumsum(cnt)])
    cells_of_face = {}
    for i in range(n_l2):
        for t in range(Dptr[i], Dptr[i + 1]):
            cells_of_face.setdefault(int(Dcol[t]), []).append(i)
    indptr = [0]
    indices, data = [], []
    for i in range(n_l2):
        row = {i: Ctil[i]}
        for t in range(Dptr[i], Dptr[i + 1]):
            k = int(Dcol[t])
            row[i] += 1.0 / Mdiag[k]
            for j in cells_of_face[k]:
                if j != i:
                    row[j] = row.get(j, 0.0) - 1.0 / Mdiag[k]
        for j in sorted(row):
            indices.append(j)
            data.append(row[j])
        indptr.append(len(indices))
    return sp.csr_matrix((np.array(data), np.array(indices, dtype=np.int64),
                          np.array(indptr, dtype=np.int64)), shape=(n_l2, n_l2))


def schur_triple_product(D: sp.csr_matrix, Mdiag, Ctil) -> sp.csr_matrix:
    """S~ = D diag(1/M~) D^T + diag(C~) by a sparse triple product."""
    S = (D @ sp.diags(1.0 / Mdiag) @ D.T + sp.diags(Ctil)).tocsr()
    S.sort_indices()
    return S
