"""The oracle's element-local sampled rows agree with its global assembly (the sampled
path is what full-size GPU parity compares against)."""
import numpy as np
import pytest

from oracle import operators, sample
from synth import make_config, random_vector


@pytest.mark.parametrize("name,N,p", [("c1", (3, 2), 2), ("c2", (2, 3, 2), 2), ("c3", (2, 2, 2), 3),
                                      ("c5", (5, 5, 3), 2), ("c3gv", (2, 3, 2), 2),
                                      ("c3gv", (2, 2, 2), 3)])
def test_sampled_rows_match_assembly(name, N, p):
    if name == "c3gv":   # general vertex-field gamma (NEXT-3, reading A22), as in the GPU tests
        pr = make_config("c3", N=N, p=p)
        pr.gamma_vertex = (10.0 ** random_vector(pr.vertices[..., 0].size, 42)).reshape(
            pr.vertices.shape[:-1])
    else:
        pr = make_config(name, N=N, p=p)
    A = operators.Assembled(pr, with_schur=False)
    x = random_vector(A.n_rt + A.n_l2, 21)
    y = A.apply_block(x)
    rt_rows = np.arange(A.n_rt)
    l2_rows = np.arange(A.n_l2)
    yu, yq = sample.block_apply_rows(pr, x, rt_rows, l2_rows)
    assert np.abs(yu - y[:A.n_rt]).max() <= 1e-13 * np.abs(y[:A.n_rt]).max()
    assert np.abs(yq - y[A.n_rt:]).max() <= 1e-13 * np.abs(y[A.n_rt:]).max()
    ye = sample.element_apply(pr, x, range(pr.E))
    assert np.abs(ye - y).max() <= 1e-13 * np.abs(y).max()
