"""Pins of the oracle's numbering and Algorithm-1 divergence."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import space


def _D(dim, N, p):
    I, J, A = space.divergence_csr(dim, N, p)
    s = space.sizes(dim, N, p)
    return sp.csr_matrix((A, J, I), shape=(len(I) - 1, s["n_rt"])), I, J, A


def test_single_element_rows():
    D, *_ = _D(2, (1, 1), 1)
    assert np.array_equal(D.toarray(), [[-1, 1, -1, 1]])
    D, *_ = _D(3, (1, 1, 1), 1)
    assert np.array_equal(D.toarray(), [[-1, 1, -1, 1, -1, 1]])


@pytest.mark.parametrize("dim,N,p", [(2, (4, 4), 2), (2, (3, 2), 3), (3, (2, 2, 2), 2),
                                     (3, (3, 2, 4), 3), (3, (1, 2, 1), 4)])
def test_incidence_structure(dim, N, p):
    """2d nonzeros per row, <=2 per column with opposite signs, sorted columns,
    and counts: interior faces 2, boundary faces 1."""
    D, I, J, A = _D(dim, N, p)
    assert np.array_equal(np.diff(I), np.full(len(I) - 1, 2 * dim))
    for i in range(len(I) - 1):
        assert np.all(np.diff(J[I[i]:I[i + 1]]) > 0)   # canonical order ascending
    Dc = D.tocsc()
    n = [N[a] * p for a in range(dim)]
    s = space.sizes(dim, N, p)
    for f in range(s["n_rt"]):
        vals = Dc.data[Dc.indptr[f]:Dc.indptr[f + 1]]
        assert len(vals) in (1, 2)
        if len(vals) == 2:
            assert sorted(vals) == [-1, 1]
    # number of boundary faces = surface subfaces
    ncol = np.diff(Dc.indptr)
    if dim == 2:
        nb = 2 * n[0] + 2 * n[1]
    else:
        nb = 2 * (n[0] * n[1] + n[1] * n[2] + n[0] * n[2])
    assert np.sum(ncol == 1) == nb


@pytest.mark.parametrize("dim,N,p", [(2, (2, 3), 3), (3, (2, 1, 2), 2), (3, (1, 1, 1), 3)])
def test_equals_lowest_order_on_refined_mesh(dim, N, p):
    """D coincides with the lowest-order D on the GLL-refined mesh."""
    D, *_ = _D(dim, N, p)
    Nref = tuple(N[a] * p for a in range(dim))
    D1, *_ = _D(dim, Nref, 1)
    # same RT (face-grid) numbering; map L2 rows via subcell coordinates
    E = int(np.prod(N))
    perm = np.zeros(D.shape[0], dtype=int)
    for e in range(E):
        eidx = space.element_index(dim, N, e)
        for il in range(p ** dim):
            loc = [(il // p ** a) % p for a in range(dim)]
            g = [eidx[a] * p + loc[a] for a in range(dim)]
            row1 = g[0] + Nref[0] * g[1] + (Nref[0] * Nref[1] * g[2] if dim == 3 else 0)
            perm[e * p ** dim + il] = row1
    assert (D - D1[perm]).nnz == 0


@pytest.mark.parametrize("n,p", [(1, 1), (2, 1), (2, 3), (4, 2), (3, 4)])
def test_rt_dof_count_2d(n, p):
    np_ = n * p
    assert space.sizes(2, (n, n), p)["n_rt"] == 2 * np_ * (np_ + 1)


def test_counts_3d():
    # p=3 single hex: 27 volumes, 108 faces
    v2f, _ = space.volume_to_face(3, 3)
    assert v2f.shape == (6, 27)
    assert len(space.rt_local_to_global(3, (1, 1, 1), 3, 0)) == 108
    # BASELINE configs (SURVEY §8 size table)
    assert space.sizes(3, (8, 8, 8), 3)["n_rt"] == 43200
    assert space.sizes(3, (64, 64, 64), 4)["n_rt"] == 50528256
    assert space.sizes(3, (128, 128, 128), 4)["n_rt"] == 403439616
