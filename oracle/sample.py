"""Element-local evaluation of the block operator for sampled outputs (oracle; test
infrastructure).  Used for parity at BASELINE sizes, where assembling the global
matrices is too slow: each sampled output row is computed from the dense
quadrature element matrices (fem.py) of the 1 or 2 elements that touch it.

y_u = M u + D^T q~ ,  y_q = D u - Z q~
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import fem, space
from .operators import mass_weight


def element_blocks(prob, e):
    """(M^e, Z^e) for element e by direct quadrature."""
    dim, N, p = prob.dim, prob.N, prob.p
    ref = fem.ref_tables(dim, p, prob.nq)
    X = fem.element_vertices(prob.vertices, dim, space.element_index(dim, N, e))
    Me = fem.element_rt_mass(X, mass_weight(prob, e), ref)
    nl = p ** dim
    if prob.kind == "grad_div":
        We = fem.element_l2_mass(X, float(prob.alpha[e]), ref)
        Ze = sla.cho_solve(sla.cho_factor(We), np.eye(nl))
    else:
        We = fem.element_l2_mass(X, 1.0, ref)
        Gv = getattr(prob, "gamma_vertex", None)
        if Gv is not None:   # general gamma (NEXT-3, reading A22), as in operators.Assembled
            Ge = fem.element_vertices(Gv[..., None], dim, space.element_index(dim, N, e))
            Wg = fem.element_l2_mass(X, fem.physical_points(Ge, ref.pts)[:, 0], ref)
        else:
            Wg = fem.element_l2_mass(X, float(prob.gamma[e]), ref)
        cf = sla.cho_factor(We)
        Ze = sla.cho_solve(cf, Wg @ sla.cho_solve(cf, np.eye(nl)))
    return Me, Ze


def rt_row_elements(dim, N, p, f):
    """Elements containing global RT DOF f and f's local index in each."""
    s = space.sizes(dim, N, p)
    n, offs = s["n"], s["offs"]
    comp = max(c for c in range(dim) if f >= offs[c])
    r = f - offs[comp]
    ext = [n[a] + (1 if a == comp else 0) for a in range(dim)]
    idx = []
    for a in range(dim):
        idx.append(r % ext[a])
        r //= ext[a]
    cands = []
    for a in range(dim):
        I = idx[a]
        if a == comp:
            opts = []
            if I % p == 0:
                if I // p - 1 >= 0:
                    opts.append((I // p - 1, p))
                if I // p < N[a]:
                    opts.append((I // p, 0))
            else:
                opts.append((I // p, I % p))
        else:
            opts = [(I // p, I % p)]
        cands.append(opts)
    out = []
    import itertools
    for combo in itertools.product(*cands):
        eidx = [c[0] for c in combo]
        e = eidx[0] + N[0] * eidx[1] + (N[0] * N[1] * eidx[2] if dim == 3 else 0)
        g = space.rt_local_to_global(dim, N, p, e)
        jl = int(np.nonzero(g == f)[0][0])
        out.append((e, jl))
    return out


def block_apply_rows(prob, x, rt_rows, l2_rows):
    """Exact y[rows] of the block operator from element matrices of touching elements."""
    dim, N, p = prob.dim, prob.N, prob.p
    nl = p ** dim
    n_rt = prob.n_rt()
    u, q = x[:n_rt], x[n_rt:]
    v2f, sig = space.volume_to_face(dim, p)
    cache = {}

    def blocks(e):
        if e not in cache:
            cache[e] = element_blocks(prob, e)
        return cache[e]

    yu = np.zeros(len(rt_rows))
    for t, f in enumerate(rt_rows):
        acc = 0.0
        for e, jl in rt_row_elements(dim, N, p, int(f)):
            Me, _ = blocks(e)
            g = space.rt_local_to_global(dim, N, p, e)
            acc += Me[jl, :] @ u[g]
            ks, ils = np.nonzero(v2f == jl)
            for k, il in zip(ks, ils):
                acc += sig[k, il] * q[e * nl + il]
        yu[t] = acc
    yq = np.zeros(len(l2_rows))
    for t, i in enumerate(l2_rows):
        e, il = int(i) // nl, int(i) % nl
        _, Ze = blocks(e)
        g = space.rt_local_to_global(dim, N, p, e)
        acc = 0.0
        for k in range(2 * dim):
            acc += sig[k, il] * u[g[v2f[k, il]]]
        acc -= Ze[il, :] @ q[e * nl:(e + 1) * nl]
        yq[t] = acc
    return yu, yq


def element_apply(prob, x, elements):
    """Matrix-free-style oracle apply restricted to `elements` (each element matrix
    formed by quadrature, multiplied, scattered).  Returns the partial y; used to time
    the oracle on a bounded sample (bench cpu_baseline)."""
    dim, N, p = prob.dim, prob.N, prob.p
    nl = p ** dim
    n_rt = prob.n_rt()
    u, q = x[:n_rt], x[n_rt:]
    v2f, sig = space.volume_to_face(dim, p)
    y = np.zeros(x.shape)   # calloc: untouched pages stay unmapped (no full-size memset)
    for e in elements:
        Me, Ze = element_blocks(prob, int(e))
        g = space.rt_local_to_global(dim, N, p, int(e))
        ue = u[g]
        qe = q[e * nl:(e + 1) * nl]
        De = np.zeros((nl, len(g)))
        De[np.arange(nl)[None, :].repeat(2 * dim, 0), v2f] = sig
        y[g] += Me @ ue + De.T @ qe
        y[n_rt + e * nl:n_rt + (e + 1) * nl] += De @ ue - Ze @ qe
    return y
