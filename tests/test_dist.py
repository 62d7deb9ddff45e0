"""Multi-process (gloo, world_size 2, CPU) tests of the element-slab decomposition that
libhdiv's multi-GPU path implements: every rank applies the oracle operator of
its own slab in slab-local canonical numbering, the replicated interface planes are exchanged
and reverse-added over torch.distributed, and the result must equal the global operator; the
masked dot products must sum to the global ones; the S~ ghost-column convention must reproduce
the global S~ rows; and the reverse-added planes must be bitwise identical on both ranks."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import operators
    from paper_2304_12387_b200 import slabs
    from synth import make_config, random_vector, Problem
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for name, N, p in cases:
            pr = make_config(name, N=N, p=p)
            dim = pr.dim
            last = dim - 1
            z0, z1 = slabs.slab_bounds(pr.N[last], world, rank)
            V, al, be, ga, ep = slabs.slab_inputs(pr, z0, z1)
            Nl = list(pr.N)
            Nl[last] = z1 - z0
            loc = Problem(name + f"_r{rank}", dim, tuple(Nl), p, pr.kind, V, alpha=al, beta=be,
                          gamma=ga, eps=ep)
            A_g = operators.Assembled(pr)
            A_l = operators.Assembled(loc)
            rt_map = slabs.local_to_global_rt(dim, pr.N, p, z0, z1)
            l2_map = slabs.local_to_global_l2(dim, pr.N, p, z0, z1)
            assert len(rt_map) == A_l.n_rt and len(l2_map) == A_l.n_l2
            x = random_vector(A_g.n_rt + A_g.n_l2, 5)
            xl = np.concatenate([x[:A_g.n_rt][rt_map], x[A_g.n_rt:][A_g.n_rt * 0 + l2_map]])
            yl = A_l.apply_block(xl)
            dl = A_l.Mdiag.copy()
            # reverse-add of the replicated interface planes (what comm_reverse_add does)
            lo, hi = slabs.interface_planes(dim, pr.N, p, z0, z1, rank, world)
            for vec in (yl, dl):
                reqs, bufs = [], {}
                for sl, peer in ((lo, rank - 1), (hi, rank + 1)):
                    if sl is None:
                        continue
                    send = torch.from_numpy(vec[sl].copy())
                    recv = torch.empty_like(send)
                    reqs += [dist.isend(send, peer), dist.irecv(recv, peer)]
                    bufs[peer] = (sl, recv)
                for r in reqs:
                    r.wait()
                for peer, (sl, recv) in bufs.items():
                    vec[sl] = vec[sl] + recv.numpy()
            yg = A_g.apply_block(x)
            ref = np.concatenate([yg[:A_g.n_rt][rt_map], yg[A_g.n_rt:][l2_map]])
            err = np.abs(yl - ref).max() / np.abs(ref).max()
            assert err < 1e-13, (name, rank, err)
            assert np.abs(dl - A_g.Mdiag[rt_map]).max() <= 1e-14 * np.abs(A_g.Mdiag).max()
            # bitwise identical replicas of the interface plane
            if hi is not None:
                t = torch.from_numpy(yl[hi].copy())
                dist.send(t, rank + 1)
            if lo is not None:
                t = torch.empty(lo.stop - lo.start, dtype=torch.float64)
                dist.recv(t, rank - 1)
                assert np.array_equal(t.numpy(), yl[lo])
            # masked dots: sum over ranks == global dot
            m = slabs.dot_mask(dim, pr.N, p, z0, z1, rank, world)
            part = torch.tensor([float(np.dot(yl[m], xl[m]))], dtype=torch.float64)
            allp = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(allp, part)
            tot = sum(float(t.item()) for t in allp)
            assert abs(tot - float(np.dot(yg, x))) <= 1e-12 * abs(float(np.dot(yg, x)))
            # S~ ghost-column convention: local rows with ghosts == global rows
            S = A_g.S.tocsr()
            gh = slabs.ghost_columns_to_global(dim, pr.N, p, z0, z1, rank, world)
            nl2 = A_l.n_l2
            for i_loc in range(nl2):
                g = l2_map[i_loc]
                cols = set(S.indices[S.indptr[g]:S.indptr[g + 1]].tolist())
                local_cols = set()
                for gc in cols:
                    hits = np.nonzero(l2_map == gc)[0]
                    if len(hits):
                        local_cols.add(int(hits[0]))
                    else:
                        inv = [c for c, gg in gh.items() if gg == gc]
                        assert len(inv) == 1, (i_loc, gc)
                        local_cols.add(inv[0])
                assert len(local_cols) == len(cols)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cases", [[("c2", (2, 3, 4), 2), ("c1", (3, 4), 2), ("c3", (2, 2, 3), 2),
                                    ("c5", (5, 5, 4), 1)]])
def test_slab_decomposition_world2(cases):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_slab_bounds_cover():
    from paper_2304_12387_b200 import slabs
    for n in (1, 5, 16, 128):
        for P in (1, 2, 3, 8):
            if P > n:
                continue
            b = [slabs.slab_bounds(n, P, r) for r in range(P)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(P - 1))
            assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1
