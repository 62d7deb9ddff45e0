"""GPU parity of the general-gamma Darcy block (NEXT-3: P:552; reading A22): the full
W^-1 W_gamma W^-1 by two passes of the element-local CG with the W_gamma sum-factorised apply
in between, C~ = diag(W_gamma)/diag(W)^2 with the variable coefficient, and MINRES — CUDA path
through the C-ABI vs the CPU oracle."""
import numpy as np
import pytest

from synth import make_config, random_vector

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _rel(a, b):
    d = np.abs(np.asarray(a) - np.asarray(b)).max()
    s = np.abs(np.asarray(b)).max()
    return d / s if s > 0 else d


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _problem(name, N, p):
    pr = make_config(name, N=N, p=p)
    pr.kind = "darcy"
    pr.eps = 10.0 ** random_vector(pr.E, 41)
    pr.gamma = np.zeros(pr.E)
    nv = pr.vertices[..., 0].size
    pr.gamma_vertex = (10.0 ** random_vector(nv, 42)).reshape(pr.vertices.shape[:-1])
    return pr


CASES = [("c3", (2, 2, 2), 1), ("c3", (3, 2, 2), 2), ("c3", (2, 3, 2), 3), ("c3", (2, 2, 2), 4),
         ("c3", (2, 2, 1), 5), ("c3", (1, 2, 2), 6), ("c2", (3, 2, 2), 3), ("c5", (5, 5, 3), 2)]


@pytest.mark.parametrize("name,N,p", CASES)
def test_general_gamma_apply(name, N, p):
    from oracle import operators
    from paper_2304_12387_b200 import from_problem
    pr = _problem(name, N, p)
    A = operators.Assembled(pr)
    op = from_problem(pr)
    s = op.sizes
    x = random_vector(s.n, 17)
    y = _host(op.apply_block(_dev(x)))
    yo = A.apply_block(x)
    assert _rel(y[:s.n_rt], yo[:s.n_rt]) < TOL
    assert _rel(y[s.n_rt:], yo[s.n_rt:]) < TOL
    q = x[s.n_rt:]
    assert _rel(_host(op.apply_z(_dev(q))), A.apply_Z(q)) < TOL      # the (2,2) block alone
    assert _rel(_host(op.schur_diag_term()), A.Ctil) < TOL
    op.close()


def test_general_gamma_minres():
    from oracle import operators, solvers
    from paper_2304_12387_b200 import from_problem
    pr = _problem("c3", (3, 3, 2), 2)
    A = operators.Assembled(pr)
    n = A.n_rt + A.n_l2
    b = A.apply_block(random_vector(n, 1))
    P = solvers.BlockDiagPrecond(A)
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=3000)
    op = from_problem(pr)
    x, rep = op.minres(_dev(b), rtol=1e-12, maxit=3000)
    assert conv_o and rep.converged and abs(rep.iters - it_o) <= 1, (rep.iters, it_o)
    assert _rel(_host(x), xo) < 1e-9
    op.close()
