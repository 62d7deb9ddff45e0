"""Canonical global numbering and Algorithm 1 (oracle; test infrastructure).

Canonical numbering (reading A6), n_a = N_a p subcells per axis:
  3D RT: x-faces (I,J,K), I in [0,n_x]:  I + (n_x+1)(J + n_y K)
         y-faces (offset N_xf):          I + n_x (J + (n_y+1) K)
         z-faces (offset N_xf+N_yf):     I + n_x (J + n_y K)
  2D RT: x-faces I + (n_x+1) J ; y-faces N_xf + I + n_x J
  L2:    element-contiguous  e p^d + (a + p(b + p c))   (Alg. 1 element_map)
Orientation (reading A5): every global face normal points along +x/+y/+z, so
global_orientation = +1; the local sign is +1 on the positive side of a cell.
"""
from __future__ import annotations

import numpy as np


def sizes(dim, N, p):
    n = [N[a] * p for a in range(dim)]
    if dim == 2:
        nxf = (n[0] + 1) * n[1]
        nyf = n[0] * (n[1] + 1)
        return dict(n=n, offs=[0, nxf], n_rt=nxf + nyf)
    nxf = (n[0] + 1) * n[1] * n[2]
    nyf = n[0] * (n[1] + 1) * n[2]
    nzf = n[0] * n[1] * (n[2] + 1)
    return dict(n=n, offs=[0, nxf, nxf + nyf], n_rt=nxf + nyf + nzf)


def element_index(dim, N, e):
    if dim == 2:
        return (e % N[0], e // N[0])
    return (e % N[0], (e // N[0]) % N[1], e // (N[0] * N[1]))


def rt_local_to_global(dim, N, p, e) -> np.ndarray:
    """rt_local_to_global[e, j_loc] (Alg. 1 table), local order as in fem.py."""
    s = sizes(dim, N, p)
    n, offs = s["n"], s["offs"]
    out = []
    if dim == 2:
        ex, ey = element_index(dim, N, e)
        for j in range(p):
            for i in range(p + 1):
                I, J = ex * p + i, ey * p + j
                out.append(offs[0] + I + (n[0] + 1) * J)
        for j in range(p + 1):
            for i in range(p):
                I, J = ex * p + i, ey * p + j
                out.append(offs[1] + I + n[0] * J)
        return np.array(out, dtype=np.int64)
    ex, ey, ez = element_index(dim, N, e)
    for k in range(p):
        for j in range(p):
            for i in range(p + 1):
                I, J, K = ex * p + i, ey * p + j, ez * p + k
                out.append(offs[0] + I + (n[0] + 1) * (J + n[1] * K))
    for k in range(p):
        for j in range(p + 1):
            for i in range(p):
                I, J, K = ex * p + i, ey * p + j, ez * p + k
                out.append(offs[1] + I + n[0] * (J + (n[1] + 1) * K))
    for k in range(p + 1):
        for j in range(p):
            for i in range(p):
                I, J, K = ex * p + i, ey * p + j, ez * p + k
                out.append(offs[2] + I + n[0] * (J + n[1] * K))
    return np.array(out, dtype=np.int64)


def l2_local_to_global(dim, p, e) -> np.ndarray:
    nl = p ** dim
    return e * nl + np.arange(nl, dtype=np.int64)


def volume_to_face(dim, p):
    """volume_to_face[k, i_loc] and the orientation of that face seen from the cell,
    k = (-x,+x,-y,+y[,-z,+z])  (Alg. 1; reading of local_orientation in DESIGN.md)."""
    nl = p ** dim
    v2f = np.zeros((2 * dim, nl), dtype=np.int64)
    sig = np.zeros((2 * dim, nl), dtype=np.int64)
    if dim == 2:
        nx = (p + 1) * p
        for b in range(p):
            for a in range(p):
                il = a + p * b
                v2f[0, il], sig[0, il] = a + (p + 1) * b, -1
                v2f[1, il], sig[1, il] = (a + 1) + (p + 1) * b, +1
                v2f[2, il], sig[2, il] = nx + a + p * b, -1
                v2f[3, il], sig[3, il] = nx + a + p * (b + 1), +1
        return v2f, sig
    nc = (p + 1) * p * p
    for c in range(p):
        for b in range(p):
            for a in range(p):
                il = a + p * (b + p * c)
                v2f[0, il], sig[0, il] = a + (p + 1) * (b + p * c), -1
                v2f[1, il], sig[1, il] = (a + 1) + (p + 1) * (b + p * c), +1
                v2f[2, il], sig[2, il] = nc + a + p * (b + (p + 1) * c), -1
                v2f[3, il], sig[3, il] = nc + a + p * ((b + 1) + (p + 1) * c), +1
                v2f[4, il], sig[4, il] = 2 * nc + a + p * (b + p * c), -1
                v2f[5, il], sig[5, il] = 2 * nc + a + p * (b + p * (c + 1)), +1
    return v2f, sig


def divergence_csr(dim, N, p):
    """Algorithm 1 literally: row i has 2d entries, I[i] = 2 d i."""
    E = int(np.prod(N[:dim]))
    nl = p ** dim
    n_l2 = E * nl
    element_map = np.arange(n_l2) // nl
    l2_global_to_local = np.arange(n_l2) % nl
    v2f, sig_loc = volume_to_face(dim, p)
    n_rt = sizes(dim, N, p)["n_rt"]
    global_orientation = np.ones(n_rt, dtype=np.int64)  # reading A5
    l2g = [rt_local_to_global(dim, N, p, e) for e in range(E)]
    Iptr = np.zeros(n_l2 + 1, dtype=np.int64)
    Jcol = np.zeros(2 * dim * n_l2, dtype=np.int64)
    Aval = np.zeros(2 * dim * n_l2, dtype=np.float64)
    for i in range(n_l2):                     # "parallel for" (sequential here)
        Iptr[i] = 2 * dim * i
        e = element_map[i]
        iloc = l2_global_to_local[i]
        for k in range(2 * dim):
            jloc = v2f[k, iloc]
            s_loc = sig_loc[k, iloc]
            j = l2g[e][jloc]
            s_glob = global_orientation[j]
            Jcol[2 * dim * i + k] = j
            Aval[2 * dim * i + k] = s_loc * s_glob
    Iptr[n_l2] = 2 * dim * n_l2
    return Iptr, Jcol, Aval


def essential_rt_mask(dim, N, p, sides: int) -> np.ndarray:
    """Boolean mask of the RT DOFs on the domain sides selected by the bitmask `sides`
    (bit 2a: the side x_a = min, bit 2a+1: x_a = max; a = 0..dim-1) — the faces where the
    normal flux u.n is prescribed (essential flux condition, SPE10 P:1035; NEXT-3).
    In the canonical numbering a face of component c lies on a side of axis c iff its
    subcell-face coordinate along c is 0 or n_c."""
    s = sizes(dim, N, p)
    n, offs = s["n"], s["offs"]
    mask = np.zeros(s["n_rt"], dtype=bool)
    for c in range(dim):
        ext = [n[a] + (1 if a == c else 0) for a in range(dim)]
        cnt = int(np.prod(ext))
        idx = np.arange(cnt, dtype=np.int64)
        # coordinate along c of face r (x fastest)
        stride = int(np.prod(ext[:c])) if c > 0 else 1
        coord = (idx // stride) % ext[c]
        if sides >> (2 * c) & 1:
            mask[offs[c] + idx[coord == 0]] = True
        if sides >> (2 * c + 1) & 1:
            mask[offs[c] + idx[coord == n[c]]] = True
    return mask
