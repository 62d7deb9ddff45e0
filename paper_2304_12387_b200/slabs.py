"""Host-side logic of the element-slab decomposition.

Rank r of P owns element layers [z0, z1) along the last axis (z in 3D, y in 2D).  Its vectors
use the canonical numbering of the slab sub-mesh; the interface face plane between ranks r and
r+1 is replicated (local last-axis faces at K = 0 and K = n_last).  These helpers are the
single statement of the conventions libhdiv's comm.cu implements:

  * interface planes of an RT vector: lo = [off_last, off_last + plane) (r > 0),
    hi = [off_last + n_last*plane, + plane) (r < P-1), plane = n_x n_y (3D) or n_x (2D);
  * dot products exclude the lo plane on r > 0 (the lower rank owns the interface);
  * S~ ghost columns: n_l2 + (X + n_x Y) for the cell layer below, n_l2 + plane + (X + n_x Y)
    for the layer above (X, Y subcell coordinates in the plane).
No arithmetic of the method lives here (index bookkeeping only).
"""
from __future__ import annotations

import numpy as np


def slab_bounds(n_layers: int, nranks: int, rank: int):
    base, rem = divmod(int(n_layers), int(nranks))
    z0 = rank * base + min(rank, rem)
    return z0, z0 + base + (1 if rank < rem else 0)


def slab_inputs(prob, z0: int, z1: int):
    """Vertex layers z0..z1 (inclusive) and per-element coefficients of the slab."""
    dim = prob.dim
    V = prob.vertices[z0:z1 + 1]
    per_layer = prob.N[0] * (prob.N[1] if dim == 3 else 1)
    sl = slice(z0 * per_layer, z1 * per_layer)
    pick = (lambda a: None if a is None else np.ascontiguousarray(a[sl]))
    return V, pick(prob.alpha), pick(prob.beta), pick(prob.gamma), pick(prob.eps)


def _sizes(dim, n):
    if dim == 2:
        nxf = (n[0] + 1) * n[1]
        return [0, nxf], nxf + n[0] * (n[1] + 1)
    nxf = (n[0] + 1) * n[1] * n[2]
    nyf = n[0] * (n[1] + 1) * n[2]
    return [0, nxf, nxf + nyf], nxf + nyf + n[0] * n[1] * (n[2] + 1)


def local_to_global_rt(dim, N, p, z0, z1) -> np.ndarray:
    """Global canonical RT index of every local RT index of slab [z0, z1)."""
    n_g = [N[a] * p for a in range(dim)]
    n_l = list(n_g)
    n_l[dim - 1] = (z1 - z0) * p
    offs_g, _ = _sizes(dim, n_g)
    offs_l, nrt_l = _sizes(dim, n_l)
    out = np.empty(nrt_l, dtype=np.int64)
    shift = z0 * p
    for c in range(dim):
        ext_l = [n_l[a] + (1 if a == c else 0) for a in range(dim)]
        ext_g = [n_g[a] + (1 if a == c else 0) for a in range(dim)]
        idx = np.indices(ext_l[::-1]).reshape(dim, -1)[::-1]   # (I, J[, K]) with I fastest
        idx[dim - 1] += shift
        g = idx[0] + ext_g[0] * (idx[1] + (ext_g[1] * idx[2] if dim == 3 else 0))
        n_c = int(np.prod(ext_l))
        out[offs_l[c]:offs_l[c] + n_c] = offs_g[c] + g
    return out


def local_to_global_l2(dim, N, p, z0, z1) -> np.ndarray:
    per_layer = N[0] * (N[1] if dim == 3 else 1)
    pd = p ** dim
    return np.arange(z0 * per_layer * pd, z1 * per_layer * pd, dtype=np.int64)


def interface_planes(dim, N, p, z0, z1, rank, nranks):
    """(lo, hi) slices of the local RT vector holding the replicated interface planes."""
    n_l = [N[a] * p for a in range(dim)]
    n_l[dim - 1] = (z1 - z0) * p
    offs_l, _ = _sizes(dim, n_l)
    plane = n_l[0] * (n_l[1] if dim == 3 else 1)
    o = offs_l[dim - 1]
    lo = slice(o, o + plane) if rank > 0 else None
    hi = slice(o + n_l[dim - 1] * plane, o + (n_l[dim - 1] + 1) * plane) if rank < nranks - 1 else None
    return lo, hi


def dot_mask(dim, N, p, z0, z1, rank, nranks) -> np.ndarray:
    """Boolean mask over the local block vector [u; q]: entries counted in global dots."""
    n_l = [N[a] * p for a in range(dim)]
    n_l[dim - 1] = (z1 - z0) * p
    _, nrt = _sizes(dim, n_l)
    per_layer = N[0] * (N[1] if dim == 3 else 1)
    nl2 = (z1 - z0) * per_layer * p ** dim
    m = np.ones(nrt + nl2, dtype=bool)
    lo, _ = interface_planes(dim, N, p, z0, z1, rank, nranks)
    if lo is not None:
        m[lo] = False
    return m


def ghost_columns_to_global(dim, N, p, z0, z1, rank, nranks) -> dict:
    """Map ghost column -> global L2 index of the neighbour cell across the interface."""
    per_layer = N[0] * (N[1] if dim == 3 else 1)
    nl2 = (z1 - z0) * per_layer * p ** dim
    nx = N[0] * p
    plane = nx * (N[1] * p if dim == 3 else 1)
    out = {}
    for k in range(plane):
        X = k % nx
        Y = k // nx
        for side, zc in (("lo", z0 * p - 1), ("hi", z1 * p)):
            if side == "lo" and rank == 0:
                continue
            if side == "hi" and rank == nranks - 1:
                continue
            col = nl2 + k + (plane if side == "hi" else 0)
            if dim == 3:
                e = X // p + N[0] * (Y // p + N[1] * (zc // p))
                g = e * p ** 3 + X % p + p * (Y % p + p * (zc % p))
            else:
                e = X // p + N[0] * (zc // p)
                g = e * p ** 2 + X % p + p * (zc % p)
            out[col] = g
    return out
