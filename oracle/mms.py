"""Manufactured-solution load vector and L2 error (oracle; test infrastructure).

Grad-div: -grad(alpha div u) + beta u = f, natural BC alpha div u = 0.
Saddle form with q = div u; transformed: right-hand side (f, 0).
Load b_k = (f, phi_k) = sum_q w_q f(x_q) . (J_q phi_hat_k(x_hat_q))  (Piola, det J cancels).
"""
from __future__ import annotations

import numpy as np

from . import fem, space


def u_exact(dim, X):
    pi = np.pi
    if dim == 2:
        x, y = X[:, 0], X[:, 1]
        return np.stack([np.cos(pi * x) * np.sin(pi * y), np.sin(pi * x) * np.cos(pi * y)], 1)
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    return np.stack([np.cos(pi * x) * np.sin(pi * y) * np.sin(pi * z),
                     np.sin(pi * x) * np.cos(pi * y) * np.sin(pi * z),
                     np.sin(pi * x) * np.sin(pi * y) * np.cos(pi * z)], 1)


def f_exact(dim, X):
    """alpha = beta = 1: grad(div u*) = -dim pi^2 u*, so f = (1 + dim pi^2) u*."""
    return (1.0 + dim * np.pi ** 2) * u_exact(dim, X)


def load_vector(prob, Q=None):
    dim, N, p = prob.dim, prob.N, prob.p
    ref = fem.ref_tables(dim, p, Q or prob.nq + 2)
    b = np.zeros(prob.n_rt())
    for e in range(prob.E):
        X = fem.element_vertices(prob.vertices, dim, space.element_index(dim, N, e))
        J, det = fem.jacobian(X, ref.pts)
        xq = fem.physical_points(X, ref.pts)
        f = f_exact(dim, xq)
        A = np.einsum("qmc,qdc->qmd", ref.Phi, J)
        g = space.rt_local_to_global(dim, N, p, e)
        b[g] += np.einsum("q,qd,qmd->m", ref.w, f, A)
    return b


def l2_error(prob, u, Q=None):
    dim, N, p = prob.dim, prob.N, prob.p
    ref = fem.ref_tables(dim, p, Q or prob.nq + 2)
    err2 = 0.0
    for e in range(prob.E):
        X = fem.element_vertices(prob.vertices, dim, space.element_index(dim, N, e))
        J, det = fem.jacobian(X, ref.pts)
        xq = fem.physical_points(X, ref.pts)
        g = space.rt_local_to_global(dim, N, p, e)
        uh_hat = np.einsum("qmc,m->qc", ref.Phi, u[g])
        uh = np.einsum("qdc,qc->qd", J, uh_hat) / det[:, None]
        d = uh - u_exact(dim, xq)
        err2 += np.sum(ref.w * det * np.sum(d * d, axis=1))
    return np.sqrt(err2)
