"""GPU parity of the multi-rank slab path on ONE GPU: P ranks of one
process (one host thread and stream each) joined by libhdiv's loopback communicator, which moves
the same interface planes, L2 ghost layers and all-gathered scalars as the NCCL path by
device-to-device copies.  Every rank's slab result must match the single-rank result on the same
global problem: block applies (reverse-added interface planes), M~, S~ with ghost columns inside
S^-1, and MINRES (masked dots, rank-ordered sums: iteration counts +-1, solutions 1e-9)."""
import threading

import numpy as np
import pytest

from synth import make_config, random_vector

pytestmark = pytest.mark.gpu


def _rel(a, b):
    d = np.abs(np.asarray(a) - np.asarray(b)).max()
    s = np.abs(np.asarray(b)).max()
    return d / s if s > 0 else d


def _run_slabs(pr, P, fn, key, **kw):
    """fn(rank, op, rt_map, l2_map) on every rank (threads); returns the per-rank results."""
    import torch
    from paper_2304_12387_b200 import HdivOperator, slabs
    from paper_2304_12387_b200.binding import loopback_id
    uid = loopback_id(key)
    out, errs = [None] * P, []
    last = pr.dim - 1

    def work(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                z0, z1 = slabs.slab_bounds(pr.N[last], P, r)
                V, a, b, g, e = slabs.slab_inputs(pr, z0, z1)
                op = HdivOperator(pr.dim, pr.N, pr.p, pr.kind, vertices=V, alpha=a, beta=b,
                                  gamma=g, eps=e, essential=pr.essential,
                                  project_mean=pr.project_mean, slab=(z0, z1), nccl_id=uid,
                                  rank=r, nranks=P, **{"amg_cheb_degree": 1, "amg_global_coarse": 2, **kw})
                rt = slabs.local_to_global_rt(pr.dim, pr.N, pr.p, z0, z1)
                l2 = slabs.local_to_global_l2(pr.dim, pr.N, pr.p, z0, z1)
                out[r] = fn(r, op, rt, l2)
                torch.cuda.current_stream().synchronize()
                op.close()
        except Exception as ex:   # pragma: no cover - surfaced below
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


def _problem(name, N, p, ess=0, project=False):
    pr = make_config(name, N=N, p=p)
    if name == "c2":
        pr.alpha = 10.0 ** random_vector(pr.E, 31)
        pr.beta = 10.0 ** random_vector(pr.E, 32)
    pr.essential, pr.project_mean = ess, project
    return pr


# the last three have >= 3 z-tile layers per slab: the interface exchange runs on the comm
# stream while the interior tile layers compute (apply_block_dev's overlapped path)
CASES = [("c2", (4, 3, 6), 3, 2, 0), ("c2", (3, 4, 7), 2, 3, 0), ("c3", (3, 3, 4), 2, 2, 0),
         ("c1", (4, 6), 2, 3, 0), ("c2", (4, 3, 5), 4, 2, 63), ("c5", (5, 5, 6), 2, 2, 0),
         ("c2", (4, 3, 12), 3, 2, 0), ("c2", (4, 3, 10), 4, 2, 63), ("c2", (5, 3, 27), 2, 3, 0)]


@pytest.mark.parametrize("name,N,p,P,ess", CASES)
def test_slab_apply_and_diag(name, N, p, P, ess):
    import torch
    from paper_2304_12387_b200 import from_problem
    pr = _problem(name, N, p, ess)
    ref = from_problem(pr)
    n_rt = ref.sizes.n_rt
    x = random_vector(ref.sizes.n, 11)
    y = ref.apply_block(torch.from_numpy(x).cuda()).cpu().numpy()
    md = ref.mass_diag().cpu().numpy()
    ref.close()

    def fn(r, op, rt, l2):
        xl = np.concatenate([x[:n_rt][rt], x[n_rt:][l2]])
        yl = op.apply_block(torch.from_numpy(xl).cuda()).cpu().numpy()
        return yl, op.mass_diag().cpu().numpy(), rt, l2

    res = _run_slabs(pr, P, fn, key=1000 + hash((name, N, p, P, ess)) % 1000)
    planes = {}
    for yl, mdl, rt, l2 in res:
        nrl = len(rt)
        assert _rel(yl[:nrl], y[:n_rt][rt]) < 1e-12
        assert _rel(yl[nrl:], y[n_rt:][l2]) < 1e-12
        assert _rel(mdl, md[rt]) < 1e-12
        for i, g in enumerate(rt):   # replicated interface faces: bitwise equal on both ranks
            if g in planes:
                assert planes[g] == yl[i]
            planes[g] = yl[i]


@pytest.mark.parametrize("name,N,p,P,ess,project", [("c2", (4, 3, 6), 3, 2, 0, False),
                                                    ("c2", (4, 3, 12), 3, 2, 0, False),
                                                    ("c2", (4, 3, 10), 4, 2, 63, False),
                                                    ("c3", (3, 3, 4), 2, 2, 0, False),
                                                    ("c1", (4, 6), 2, 3, 0, False),
                                                    ("c3", (3, 3, 4), 2, 2, 63, True)])
def test_slab_minres(name, N, p, P, ess, project):
    import torch
    from paper_2304_12387_b200 import from_problem
    pr = _problem(name, N, p, ess, project)
    if project:
        pr.gamma = np.zeros(pr.E)
    ref = from_problem(pr)
    n_rt = ref.sizes.n_rt
    xs = random_vector(ref.sizes.n, 3)
    b = ref.apply_block(torch.from_numpy(xs).cuda())
    x1, rep1 = ref.minres(b, rtol=1e-12, maxit=3000)
    b = b.cpu().numpy()
    x1 = x1.cpu().numpy()
    ref.close()

    def fn(r, op, rt, l2):
        bl = np.concatenate([b[:n_rt][rt], b[n_rt:][l2]])
        xl, rep = op.minres(torch.from_numpy(bl).cuda(), rtol=1e-12, maxit=3000)
        return xl.cpu().numpy(), rep.iters, rep.converged, rt, l2

    res = _run_slabs(pr, P, fn, key=2000 + hash((name, N, p, P, ess)) % 1000)
    its = {r[1] for r in res}
    assert len(its) == 1, its                     # every rank takes the same decisions
    assert all(r[2] for r in res) and abs(res[0][1] - rep1.iters) <= 1, (res[0][1], rep1.iters)
    dqs = []
    for xl, _, _, rt, l2 in res:
        nrl = len(rt)
        assert _rel(xl[:nrl], x1[:n_rt][rt]) < 1e-9
        dqs.append(xl[nrl:] - x1[n_rt:][l2])
    c = np.concatenate(dqs).mean() if project else 0.0   # p~ unique up to ONE global constant
    for dq in dqs:
        assert np.abs(dq - c).max() < 1e-9 * np.abs(x1[n_rt:]).max()


@pytest.mark.parametrize("name,N,p,P,ess,project,k,gc", [("c2", (4, 3, 7), 3, 2, 0, False, 1, False),
                                                         ("c3", (3, 3, 6), 2, 3, 0, False, 1, False),
                                                         ("c5", (5, 5, 6), 2, 2, 0, False, 1, False),
                                                         ("c3", (3, 3, 4), 2, 2, 63, True, 1, False),
                                                         ("c3", (3, 3, 6), 2, 3, 0, False, 3, False),
                                                         ("c1", (5, 8), 2, 2, 0, False, 2, False),
                                                         ("c3", (3, 3, 4), 2, 2, 63, True, 2, False),
                                                         ("c3", (3, 3, 6), 2, 3, 0, False, 1, True),
                                                         ("c3", (4, 3, 8), 2, 4, 0, False, 3, True),
                                                         ("c2", (4, 3, 7), 3, 2, 0, False, 3, True),
                                                         ("c3", (3, 3, 4), 2, 2, 63, True, 3, True),
                                                         ("c5", (5, 5, 6), 2, 3, 0, False, 1, True),
                                                         ("c3", (3, 3, 6), 2, 3, 3 | 16, False, 3, True),
                                                         ("c2", (3, 4, 6), 4, 2, 32, False, 2, True)])
def test_slab_minres_amg(name, N, p, P, ess, project, k, gc):
    """Multi-rank S^-1 = block-Jacobi of per-slab AMG V-cycles (reading A9c) — plain, inside the
    A9d polynomial (k > 1), and in the A9e balancing form with the global coarse space (gc):
    each rank's preconditioner output and the MINRES iteration counts (+-1) against the
    oracle's on the same slabs."""
    import torch
    from oracle import operators, solvers
    from paper_2304_12387_b200 import slabs as sl
    pr = _problem(name, N, p, ess, project)
    if project:
        pr.gamma = np.zeros(pr.E)
    A = operators.Assembled(pr)
    last = pr.dim - 1
    bounds = [sl.slab_bounds(pr.N[last], P, r) for r in range(P)]
    Po = solvers.BlockDiagPrecond(A, schur="amg", amg_max_coarse=16, amg_slabs=bounds,
                                  amg_cheb_degree=k, amg_global_coarse=gc)
    n_rt = A.n_rt
    v = random_vector(A.n_rt + A.n_l2, 8)
    if project:
        v[n_rt:] -= v[n_rt:].mean()
    zo = Po.apply(v)
    xs = random_vector(A.n_rt + A.n_l2, 3)
    b = A.apply_block(xs)
    xo, it_o, conv_o, _ = solvers.minres(A.apply_block, Po.apply, b, rtol=1e-12, maxit=3000)

    def fn(r, op, rt, l2):
        vl = np.concatenate([v[:n_rt][rt], v[n_rt:][l2]])
        zl = op.apply_precond(torch.from_numpy(vl).cuda()).cpu().numpy()
        bl = np.concatenate([b[:n_rt][rt], b[n_rt:][l2]])
        xl, rep = op.minres(torch.from_numpy(bl).cuda(), rtol=1e-12, maxit=3000)
        return zl, xl.cpu().numpy(), rep.iters, rep.converged, rt, l2

    res = _run_slabs(pr, P, fn, key=3000 + hash((name, N, p, P, ess, k, gc)) % 1000,
                     schur="amg", amg_max_coarse=16, amg_cheb_degree=k,
                     amg_global_coarse=1 if gc else 2)
    assert conv_o
    its = {r[2] for r in res}
    assert len(its) == 1 and all(r[3] for r in res), its
    assert abs(res[0][2] - it_o) <= 1, (res[0][2], it_o)
    for zl, xl, _, _, rt, l2 in res:
        nrl = len(rt)
        assert _rel(zl[:nrl], zo[:n_rt][rt]) < 1e-12
        assert _rel(zl[nrl:], zo[n_rt:][l2]) < 1e-10   # (projection: the global mean)
        assert _rel(xl[:nrl], xo[:n_rt][rt]) < 1e-8


@pytest.mark.parametrize("name,N,p,P,schur", [("c2", (4, 3, 6), 3, 2, "chebyshev"),
                                              ("c2", (4, 3, 12), 3, 2, "amg"),
                                              ("c3", (3, 3, 6), 2, 3, "chebyshev"),
                                              ("c5", (5, 5, 6), 2, 2, "amg"),
                                              ("c3", (3, 3, 6), 2, 3, "amg3"),
                                              ("c3", (4, 3, 8), 2, 4, "amg3gc"),
                                              ("c2", (4, 3, 7), 3, 2, "amggc")])
def test_slab_gmres(name, N, p, P, schur):
    """NEXT-4 on slabs: block-triangular preconditioner (D^T reverse-added) + GMRES with
    all-gathered projections — every rank takes the same decisions; iteration counts +-1 and
    solutions vs the single-rank GPU solve (Chebyshev S^-1) or vs the oracle's GMRES with the
    block-Jacobi AMG S^-1 (reading A9c)."""
    import torch
    from oracle import operators, solvers
    from paper_2304_12387_b200 import from_problem, slabs as sl
    pr = _problem(name, N, p)
    # amg3: the A9d polynomial over the block-Jacobi V-cycles; ...gc: the A9e global coarse space
    k = 3 if schur.startswith("amg3") else 1
    gc = schur.endswith("gc")
    schur = "amg" if schur.startswith("amg") else schur
    kw = {"schur": schur, "amg_max_coarse": 16, "amg_cheb_degree": k,
          "amg_global_coarse": 1 if gc else 2}
    ref = from_problem(pr, **kw)
    n_rt = ref.sizes.n_rt
    xs = random_vector(ref.sizes.n, 3)
    b = ref.apply_block(torch.from_numpy(xs).cuda())
    if schur == "chebyshev":
        x1, r1 = ref.gmres(b, rtol=1e-10, restart=20, maxit=2000)
        x1, it1 = x1.cpu().numpy(), r1.iters
    b = b.cpu().numpy()
    ref.close()
    if schur == "amg":
        A = operators.Assembled(pr)
        last = pr.dim - 1
        bounds = [sl.slab_bounds(pr.N[last], P, r) for r in range(P)]
        B = solvers.BlockTriPrecond(A, schur="amg", amg_max_coarse=16)
        B.diag = solvers.BlockDiagPrecond(A, schur="amg", amg_max_coarse=16, amg_slabs=bounds,
                                          project_mean=False, amg_cheb_degree=k,
                                          amg_global_coarse=gc)
        x1, it1, conv, _ = solvers.gmres(A.apply_block, B.apply, b, rtol=1e-10, restart=20)
        assert conv

    def fn(r, op, rt, l2):
        bl = np.concatenate([b[:n_rt][rt], b[n_rt:][l2]])
        xl, rep = op.gmres(torch.from_numpy(bl).cuda(), rtol=1e-10, restart=20, maxit=2000)
        return xl.cpu().numpy(), rep.iters, rep.converged, rt, l2

    res = _run_slabs(pr, P, fn, key=4000 + hash((name, N, p, P, schur, k, gc)) % 1000, **kw)
    its = {r[1] for r in res}
    assert len(its) == 1 and all(r[2] for r in res), its
    assert abs(res[0][1] - it1) <= 1, (res[0][1], it1)
    for xl, _, _, rt, l2 in res:
        nrl = len(rt)
        assert _rel(xl[:nrl], x1[:n_rt][rt]) < 1e-8
        assert _rel(xl[nrl:], x1[n_rt:][l2]) < 1e-7


@pytest.mark.gpu
def test_slab_amg_iterations_vs_P():
    """Iteration counts vs the slab count (loopback ranks on one GPU, 10^4-contrast config-3
    mesh): the A9d polynomial (b = 2.2 with slabs) stays below the plain block-Jacobi V-cycle's
    count, and with the A9e global coarse space (the default for 3D slabs) the count no longer
    grows from 2 to 8 slabs on this mesh — at 24^3 p = 4 (profiles/r02_slab_iterations.txt) with
    the polynomial 256 / 265 / 287 at P = 2 / 4 / 8 against 265 / 287 / 316 block-Jacobi, with the
    plain V-cycle 491 / 501 / 478 against 527 / 578 / 637."""
    import torch
    from paper_2304_12387_b200 import from_problem
    pr = _problem("c3", (4, 4, 8), 2)
    its = {}
    op = from_problem(pr, schur="amg", amg_max_coarse=16, amg_cheb_degree=1)
    b = op.apply_block(torch.from_numpy(random_vector(op.sizes.n, 3)).cuda()).cpu().numpy()
    op.close()
    for k in (1, 3):
        op = from_problem(pr, schur="amg", amg_max_coarse=16, amg_cheb_degree=k)
        _, rep = op.minres(torch.from_numpy(b).cuda(), rtol=1e-12, maxit=3000)
        op.close()
        assert rep.converged
        its[(k, 1, 0)] = rep.iters
        for gc in (0, 1):
            for P in (2, 4, 8):
                def fn(r, op, rt, l2):
                    nrt_g = len(b) - pr.E * pr.p ** 3
                    bl = np.concatenate([b[:nrt_g][rt], b[nrt_g:][l2]])
                    _, rep = op.minres(torch.from_numpy(bl).cuda(), rtol=1e-12, maxit=3000)
                    return rep.iters, rep.converged
                res = _run_slabs(pr, P, fn, key=4000 + 100 * gc + 10 * k + P, schur="amg",
                                 amg_max_coarse=16, amg_cheb_degree=k,
                                 amg_global_coarse=1 if gc else 2)
                assert all(r[1] for r in res)
                its[(k, P, gc)] = res[0][0]
    for P in (2, 4, 8):
        assert its[(3, P, 0)] < its[(1, P, 0)], its
        assert its[(3, P, 1)] <= its[(3, P, 0)], its
    assert its[(3, 8, 1)] <= 1.1 * its[(3, 2, 1)] + 3, its
    assert its[(1, 8, 1)] <= 1.1 * its[(1, 2, 1)] + 3, its
