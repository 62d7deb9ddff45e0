"""1D node sets and the interpolation-histopolation basis (oracle; test infrastructure).

P:178  "vertices are given by the d-fold Cartesian product of the p+1 Gauss--Lobatto points"
P:181  RT DOFs: "tensor-product of one-dimensional interpolation and histopolation operators"
P:182  L2 DOFs: "integrals over each subelement volume ... one-dimensional histopolation"

Reference interval [0,1] (elements are images of [0,1]^d).
"""
from __future__ import annotations

import numpy as np


def legendre_and_derivative(n: int, t):
    """P_n(t), P_n'(t) on [-1,1] by the three-term recurrence."""
    t = np.asarray(t, float)
    p0, p1 = np.ones_like(t), t.copy()
    if n == 0:
        return p0, np.zeros_like(t)
    for k in range(2, n + 1):
        p0, p1 = p1, ((2 * k - 1) * t * p1 - (k - 1) * p0) / k
    # derivative: (1-t^2) P_n' = n (P_{n-1} - t P_n); endpoints by closed form
    with np.errstate(divide="ignore", invalid="ignore"):
        d = n * (p0 - t * p1) / (1.0 - t * t)
    d = np.where(np.abs(t) == 1.0, np.sign(t) ** (n + 1) * n * (n + 1) / 2.0, d)
    return p1, d


def gll_nodes(p: int) -> np.ndarray:
    """p+1 Gauss-Lobatto(-Legendre) nodes on [0,1]: 0, roots of P_p'(2x-1), 1."""
    if p < 1:
        raise ValueError("p >= 1 required")
    if p == 1:
        return np.array([0.0, 1.0])
    # interior nodes: roots of P_p' ; Newton on f = P_p' using
    # f' = P_p'' = (2t P_p' - p(p+1) P_p) / (1 - t^2)
    t = -np.cos(np.pi * np.arange(1, p) / p)  # Chebyshev-Lobatto initial guess
    for _ in range(100):
        P, dP = legendre_and_derivative(p, t)
        d2P = (2 * t * dP - p * (p + 1) * P) / (1 - t * t)
        dt = dP / d2P
        t = t - dt
        if np.max(np.abs(dt)) < 1e-16:
            break
    x = np.concatenate([[0.0], 0.5 * (t + 1.0), [1.0]])
    return np.sort(x)


def gl_rule(Q: int):
    """Q-point Gauss-Legendre rule mapped to [0,1] (quadrature rule, reading A3)."""
    if Q < 1:
        raise ValueError("Q >= 1 required")
    t, w = np.polynomial.legendre.leggauss(Q)
    return 0.5 * (t + 1.0), 0.5 * w


def lagrange(nodes: np.ndarray, x) -> np.ndarray:
    """L[r, i] = l_i(x_r), Lagrange basis on `nodes` (product formula)."""
    x = np.atleast_1d(np.asarray(x, float))
    n = len(nodes)
    L = np.ones((len(x), n))
    for i in range(n):
        for m in range(n):
            if m != i:
                L[:, i] *= (x - nodes[m]) / (nodes[i] - nodes[m])
    return L


def lagrange_deriv(nodes: np.ndarray, x) -> np.ndarray:
    """dL[r, i] = l_i'(x_r) (product rule, no division by x - node)."""
    x = np.atleast_1d(np.asarray(x, float))
    n = len(nodes)
    dL = np.zeros((len(x), n))
    for i in range(n):
        for k in range(n):
            if k == i:
                continue
            term = np.full(len(x), 1.0 / (nodes[i] - nodes[k]))
            for m in range(n):
                if m != i and m != k:
                    term *= (x - nodes[m]) / (nodes[i] - nodes[m])
            dL[:, i] += term
    return dL


def _legendre01_antideriv(n: int, x):
    """F_n(x) = integral_0^x P_n(2s-1) ds."""
    t = 2.0 * np.asarray(x, float) - 1.0
    if n == 0:
        return 0.5 * (t + 1.0)
    Pn1, _ = legendre_and_derivative(n + 1, t)
    Pm1, _ = legendre_and_derivative(n - 1, t)
    # integral of P_n dt = (P_{n+1} - P_{n-1})/(2n+1); value at t=-1 is 0 for n>=1
    return 0.5 * (Pn1 - Pm1) / (2 * n + 1)


def histopolation_coeffs(p: int) -> np.ndarray:
    """C with h_j(x) = sum_n C[n, j] P_n(2x-1), defined by the histopolation DOFs
    integral_{xi_m}^{xi_{m+1}} h_j = delta_{mj}, h_j in Q_{p-1}."""
    xi = gll_nodes(p)
    A = np.zeros((p, p))
    for n in range(p):
        F = _legendre01_antideriv(n, xi)
        A[:, n] = F[1:] - F[:-1]          # A[m, n] = integral over subinterval m of P_n
    return np.linalg.solve(A, np.eye(p))  # A C = I


def histopolation(p: int, x) -> np.ndarray:
    """H[r, j] = h_j(x_r), j = 0..p-1."""
    x = np.atleast_1d(np.asarray(x, float))
    C = histopolation_coeffs(p)
    Pm = np.stack([legendre_and_derivative(n, 2.0 * x - 1.0)[0] for n in range(p)], axis=1)
    return Pm @ C


def mass_1d(p: int, Q: int | None = None):
    """1D reference masses M_l = B_l^T W B_l, M_h = B_h^T W B_h (used by pins only)."""
    Q = Q or p + 2
    xq, wq = gl_rule(Q)
    Bl = lagrange(gll_nodes(p), xq)
    Bh = histopolation(p, xq)
    return Bl.T @ (wq[:, None] * Bl), Bh.T @ (wq[:, None] * Bh)
