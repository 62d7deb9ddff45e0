"""Counter-based seeded generators for meshes, coefficients and vectors.

Recipe:
  * random numbers: splitmix64 finaliser of (seed, index) -> 53-bit uniform in [0,1)
  * structured meshes: (N_x+1)(N_y+1)(N_z+1) vertices, x fastest, element
    e = ex + N_x (ey + N_y ez)
  * config 3 perturbation: interior vertices += U(-0.2h, 0.2h) per coordinate (A17)
  * config 3 coefficients: eps_e = 10^U(-2,2) (contrast 1e4), gamma = 0 (A18)
  * config 5: tensor-product graded two-material "crooked pipe" analogue

Nothing here evaluates a basis function, a quadrature rule or an operator.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def counter_uniform(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """n uniforms in [0,1): u_i = splitmix64(seed*G + (offset+i+1)*G) >> 11 * 2^-53."""
    out = np.empty(n, dtype=np.float64)
    chunk = 1 << 24
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _GOLDEN
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            idx = np.arange(offset + c0 + 1, offset + c1 + 1, dtype=np.uint64)
            z = _splitmix(s + idx * _GOLDEN)
            out[c0:c1] = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return out


def random_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    u = counter_uniform(seed, n)
    u *= (hi - lo)
    u += lo
    return u


def cartesian_vertices(dim: int, N, lo=None, hi=None) -> np.ndarray:
    """Uniform box vertices, array [(Nz+1),(Ny+1),(Nx+1),3] (3D) or [(Ny+1),(Nx+1),2]."""
    N = tuple(int(n) for n in N[:dim])
    lo = np.zeros(dim) if lo is None else np.asarray(lo, float)
    hi = np.ones(dim) if hi is None else np.asarray(hi, float)
    axes = [lo[a] + (hi[a] - lo[a]) * np.arange(N[a] + 1) / N[a] for a in range(dim)]
    return tensor_vertices(axes)


def tensor_vertices(axes) -> np.ndarray:
    """Vertices of the tensor grid of 1D node sequences axes=[x_nodes, y_nodes(, z_nodes)]."""
    dim = len(axes)
    if dim == 2:
        Y, X = np.meshgrid(axes[1], axes[0], indexing="ij")
        return np.ascontiguousarray(np.stack([X, Y], axis=-1))
    Z, Y, X = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    return np.ascontiguousarray(np.stack([X, Y, Z], axis=-1))


def perturbed_vertices(N, amp: float = 0.2, seed: int = 3) -> np.ndarray:
    """Unit cube, interior vertices jittered by U(-amp*h, amp*h) per coordinate (A17)."""
    V = cartesian_vertices(3, N)
    nz1, ny1, nx1, _ = V.shape
    h = np.array([1.0 / N[0], 1.0 / N[1], 1.0 / N[2]])
    r = counter_uniform(seed, V.size).reshape(V.shape)
    d = (2.0 * r - 1.0) * amp * h
    interior = np.zeros((nz1, ny1, nx1), bool)
    interior[1:-1, 1:-1, 1:-1] = True
    V = V + d * interior[..., None]
    return np.ascontiguousarray(V)


# ----------------------------------------------------------------------------
# config 5: graded two-material "crooked pipe" analogue
_DUCT = [((0.0, 0.35), (0.2, 0.35), (0.35, 0.65)),
         ((0.3, 0.45), (0.2, 0.8), (0.35, 0.65)),
         ((0.4, 1.0), (0.65, 0.8), (0.35, 0.65))]
ALPHA_IN, BETA_IN = 1.641, 0.2        # P:915 inner region
ALPHA_OUT, BETA_OUT = 1.88e-3, 2000.0  # P:915 outer region


def _graded_axis(breaks, n: int, ratio: float = 1.35) -> np.ndarray:
    breaks = np.unique(np.asarray(breaks, float))
    L = np.diff(breaks)
    if n < len(L):   # every interface plane must be a mesh plane
        raise ValueError(f"graded axis needs at least {len(L)} intervals, got {n}")
    want = L / L.sum() * n
    m = np.maximum(np.floor(want).astype(int), 1)
    while m.sum() < n:
        m[np.argmax(want - m)] += 1
    while m.sum() > n:
        k = np.argmax(np.where(m > 1, m - want, -np.inf))
        m[k] -= 1
    nodes = [breaks[0]]
    for a, b, k in zip(breaks[:-1], breaks[1:], m):
        i = np.arange(k)
        s = ratio ** np.minimum(i, k - 1 - i).astype(float)
        s = s / s.sum() * (b - a)
        nodes.extend(list(a + np.cumsum(s)))
    x = np.array(nodes)
    x[-1] = breaks[-1]
    return x


def graded_two_material(N):
    """Axis-aligned graded box mesh + per-element two-material alpha/beta."""
    bx = [0, 1] + [v for box in _DUCT for v in box[0]]
    by = [0, 1] + [v for box in _DUCT for v in box[1]]
    bz = [0, 1] + [v for box in _DUCT for v in box[2]]
    axes = [_graded_axis(bx, N[0]), _graded_axis(by, N[1]), _graded_axis(bz, N[2])]
    V = tensor_vertices(axes)
    cx = 0.5 * (axes[0][1:] + axes[0][:-1])
    cy = 0.5 * (axes[1][1:] + axes[1][:-1])
    cz = 0.5 * (axes[2][1:] + axes[2][:-1])
    CZ, CY, CX = np.meshgrid(cz, cy, cx, indexing="ij")
    inner = np.zeros(CX.shape, bool)
    for (x0, x1), (y0, y1), (z0, z1) in _DUCT:
        inner |= (CX > x0) & (CX < x1) & (CY > y0) & (CY < y1) & (CZ > z0) & (CZ < z1)
    inner = inner.ravel()
    alpha = np.where(inner, ALPHA_IN, ALPHA_OUT)
    beta = np.where(inner, BETA_IN, BETA_OUT)
    return V, alpha, beta


# ----------------------------------------------------------------------------
@dataclass
class Problem:
    """One synthetic workload: mesh + degree + coefficients (inputs only)."""
    name: str
    dim: int
    N: tuple            # (Nx, Ny, Nz); Nz = 1 in 2D
    p: int
    kind: str           # "grad_div" | "darcy"
    vertices: np.ndarray
    alpha: Optional[np.ndarray] = None   # grad-div  W_alpha weight, per element
    beta: Optional[np.ndarray] = None    # grad-div  M_beta weight,  per element
    eps: Optional[np.ndarray] = None     # Darcy     M_{1/eps},       per element
    gamma: Optional[np.ndarray] = None   # Darcy     W_gamma,         per element
    gamma_vertex: Optional[np.ndarray] = None   # Darcy general gamma: per-vertex values of a
                                         # trilinear field (shape vertices.shape[:-1]), NEXT-3
    affine: bool = True                  # axis-aligned boxes (generator knows it)
    Q: int = 0                           # 0 -> p+2 (A3)
    essential: int = 0                   # essential-flux sides bitmask (bit 2a: x_a = min,
                                         # bit 2a+1: x_a = max), NEXT-3
    project_mean: bool = False           # orthogonalize after every S^-1
    extra: dict = field(default_factory=dict)

    @property
    def E(self) -> int:
        return int(np.prod(self.N[: self.dim]))

    @property
    def nq(self) -> int:
        return self.Q if self.Q > 0 else self.p + 2

    def n_rt(self) -> int:
        n = [self.N[a] * self.p for a in range(self.dim)]
        if self.dim == 2:
            return (n[0] + 1) * n[1] + n[0] * (n[1] + 1)
        return ((n[0] + 1) * n[1] * n[2] + n[0] * (n[1] + 1) * n[2]
                + n[0] * n[1] * (n[2] + 1))

    def n_l2(self) -> int:
        return self.E * self.p ** self.dim


CONFIG_NAMES = ("c1", "c2", "c3", "c3s", "c4", "c5")


def make_config(name: str, N=None, p=None, seed: int = 0) -> Problem:
    """BASELINE.json configs 1..5; N/p override sizes."""
    if name == "c1":   # 2D 4x4, RT p=2 / L2 p=1, Darcy eps=gamma=1
        N = tuple(N or (4, 4)) + (1,)
        p = p or 2
        E = N[0] * N[1]
        return Problem("c1", 2, N[:3], p, "darcy", cartesian_vertices(2, N),
                       eps=np.ones(E), gamma=np.ones(E))
    if name == "c2":   # 3D 8^3, p=3, grad-div alpha=beta=1
        N = tuple(N or (8, 8, 8))
        p = p or 3
        E = int(np.prod(N))
        return Problem("c2", 3, N, p, "grad_div", cartesian_vertices(3, N),
                       alpha=np.ones(E), beta=np.ones(E))
    if name == "c3":   # 3D 64^3 perturbed, p=4, Darcy eps=10^U(-2,2), gamma=0
        N = tuple(N or (64, 64, 64))
        p = p or 4
        E = int(np.prod(N))
        eps = 10.0 ** (-2.0 + 4.0 * counter_uniform(4 + seed, E))
        return Problem("c3", 3, N, p, "darcy", perturbed_vertices(N, 0.2, 3 + seed),
                       eps=eps, gamma=np.zeros(E), affine=False)
    if name == "c3s":  # SPE10-shaped: c3 with u.n prescribed on every side, gamma = 0,
        pr = make_config("c3", N=N, p=p, seed=seed)   # singular S~ -> projection
        pr.name, pr.essential, pr.project_mean = "c3s", (1 << (2 * pr.dim)) - 1, True
        return pr
    if name == "c4":   # 3D 128^3, p=4, grad-div alpha=beta=1
        N = tuple(N or (128, 128, 128))
        p = p or 4
        E = int(np.prod(N))
        return Problem("c4", 3, N, p, "grad_div", cartesian_vertices(3, N),
                       alpha=np.ones(E), beta=np.ones(E))
    if name == "c5":   # graded two-material crooked-pipe analogue
        N = tuple(N or (24, 24, 25))
        p = p or 4
        V, a, b = graded_two_material(N)
        return Problem("c5", 3, N, p, "grad_div", V, alpha=a, beta=b)
    raise ValueError(name)
