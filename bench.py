"""bench.py — BASELINE.json metric: GDOF/s of the fp64 matrix-free H(div) block-operator apply
(plus MINRES time-to-solve), on synthetic inputs, through libhdiv's C-ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--p 4] [--impl reference]

A step is one block-operator apply y = A x over the whole workload (default
config 4: 128^3 Cartesian hexes, p = 4, grad-div, 537.7M DOFs; inputs 4.3 GB per vector,
i.e. much larger than the 126 MB L2, so no flush is needed).  N > 1: element slabs along z,
one rank per GPU (torchrun), interface reverse-add over NCCL inside each apply; the timed
region is bracketed by barrier + synchronize and the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDOF/s of matrix-free H(div) block-operator apply, p=2–6; MINRES time-to-solve"
WORKLOADS = {
    "c4": "config 4: 3D 128^3 Cartesian hex mesh, RT p / L2 p-1 (default p=4), grad-div "
          "alpha=beta=1, block-operator apply [M, D^T; D, -W_alpha^-1]",
    "c3": "config 3: 3D 64^3 randomly perturbed hex mesh, p=4, Darcy eps=10^U(-2,2), gamma=0",
    "c5": "config 5: graded two-material crooked-pipe analogue, grad-div",
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def torchrun_argv(argv, nproc: int, port: int, python=None):
    """Command line that relaunches this script under torchrun, one rank per GPU (the driver's
    own N > 1 launch form: --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1)."""
    return [python or sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port", str(port),
            os.path.abspath(__file__)] + list(argv)


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def nccl_log_env(env):
    """NCCL communicator init logged (NCCL_DEBUG=INFO) to stderr, so stdout keeps the JSON line."""
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return env


def make_problem(cfg: str, p: int):
    from synth import make_config
    return make_config(cfg, p=p)


# V100 local-CG solve times for 100 applies of W^-1 (Table dg-mass-inv), context
_PAPER_WINV_S = {1: 0.1937, 2: 0.0841, 3: 0.0556, 4: 0.0598, 5: 0.0697, 6: 0.0770}


def winv_bench(torch):
    import numpy as np
    from synth import make_config, random_vector
    from paper_2304_12387_b200 import from_problem
    out = {"workload": "W^-1 q (the (2,2) block) by the fused element-local CG in the GL-nodal "
                       "basis (p <= 4 also by the precomputed explicit element inverses, "
                       "explicit_*); config-3 jittered hex mesh sized to ~1.7e6 L2 DOFs, grad-div "
                       "alpha = 1 (Z = W^-1); 100 applies (Table dg-mass-inv shape, P:773-822)",
           "paper_v100_context": "P:792-794 local-CG solve x100: " +
                                 ", ".join(f"p{p} {t} s" for p, t in _PAPER_WINV_S.items())}
    def run(pr):
        t0 = time.perf_counter()
        op = from_problem(pr, schur="chebyshev")   # (the (2,2) block alone: no S^-1 needed)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        q = torch.from_numpy(random_vector(op.sizes.n_l2, 5)).cuda()
        y = torch.empty_like(q)
        for _ in range(3):
            op.apply_z(q, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(100):
            op.apply_z(q, y)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        n = op.sizes.n_l2
        op.close()
        del q, y
        torch.cuda.empty_cache()
        return n, t, setup

    for p in range(1, 7):
        ne = max(2, int(round((1.7e6 / p ** 3) ** (1.0 / 3.0))))
        pr = make_config("c3", N=(ne, ne, ne), p=p)
        pr.kind = "grad_div"
        pr.alpha = np.ones(pr.E)
        pr.beta = np.ones(pr.E)
        os.environ["HDIV_WINV"] = "cg"      # the local CG (explicit inverses not built)
        n, t, _ = run(pr)
        os.environ.pop("HDIV_WINV")
        out[f"p{p}"] = {"N": ne, "l2_dofs": n, "solve_x100_s": t, "GDOF_s": 100 * n / t / 1e9}
        if p <= 4:   # the precomputed explicit inverses, the default at p <= 4
            n, t, setup = run(pr)
            out[f"p{p}"].update({"explicit_x100_s": t, "explicit_GDOF_s": 100 * n / t / 1e9,
                                 "explicit_setup_s": setup})
    return out


def build_operator(pr, ws, rank, dist, nccl_id=None):
    from paper_2304_12387_b200 import HdivOperator
    if ws == 1:
        from paper_2304_12387_b200 import from_problem
        return from_problem(pr, schur="chebyshev")   # (apply timing: no AMG hierarchy needed)
    from paper_2304_12387_b200.slabs import slab_bounds, slab_inputs
    z0, z1 = slab_bounds(pr.N[pr.dim - 1], ws, rank)
    V, a, b, g, e = slab_inputs(pr, z0, z1)
    return HdivOperator(pr.dim, pr.N, pr.p, pr.kind, vertices=V, alpha=a, beta=b, gamma=g, eps=e,
                        essential=pr.essential, project_mean=pr.project_mean, schur="chebyshev",
                        slab=(z0, z1), nccl_id=nccl_id, rank=rank, nranks=ws)


def time_applies(op, x, y, steps, warmup, dist, torch):
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        op.apply_block(x, y)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        op.apply_block(x, y)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def _oracle_sample_worker(job):
    """One host process of the parallel oracle sample (BLAS pinned to one thread)."""
    cfg, p, elems, budget_s = job
    from threadpoolctl import threadpool_limits
    import numpy as np
    from oracle import sample
    pr = make_problem(cfg, p)
    n = pr.n_rt() + pr.n_l2()
    x = np.zeros(n)   # only the sampled elements' entries matter for the timing
    done = 0
    with threadpool_limits(1):
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < budget_s and done < len(elems):
            sample.element_apply(pr, x, elems[done:done + 8])
            done += 8
        dt = time.perf_counter() - t0
    return done, dt


def cpu_baseline(pr, budget_s: float = 15.0, cfg: str = "c4", parallel: bool = True):
    """The oracle (as it stands) on a bounded sample of the workload's elements: element matrices
    by direct quadrature + multiply, scaled to whole-apply DOFs.  Honest core accounting: one
    process with BLAS pinned to 1 thread (cores = 1), and the same element loop split over all
    host cores (one process per core, each with 1 BLAS thread) -> cores = #processes."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import sample
    n = pr.n_rt() + pr.n_l2()
    E = pr.E
    x = np.zeros(n)
    rng = np.random.default_rng(0)
    elems = rng.integers(0, E, 100000)
    one_budget = budget_s / 2 if parallel else budget_s
    t0 = time.perf_counter()
    done = 0
    with threadpool_limits(1):
        while time.perf_counter() - t0 < one_budget and done < len(elems):
            sample.element_apply(pr, x, elems[done:done + 8])
            done += 8
    dt = time.perf_counter() - t0
    v1 = n * done / E / dt / 1e9
    out = {"value": v1, "unit": "GDOF/s", "cores": 1, "kind": "oracle",
           "sample": f"{done} of {E} elements of {pr.name} p={pr.p} (element matrices by direct "
                     f"quadrature + multiply), {dt:.1f} s on 1 thread, scaled to whole-apply DOFs",
           "single_thread_value": v1}
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    ncpu = min(ncpu, 32)
    if parallel and ncpu > 1:
        import multiprocessing as mp
        jobs = [(cfg, pr.p, rng.integers(0, E, 20000), budget_s / 2) for _ in range(ncpu)]
        t1 = time.perf_counter()
        with mp.get_context("spawn").Pool(ncpu) as pool:
            res = pool.map(_oracle_sample_worker, jobs)
        wall = time.perf_counter() - t1
        tot = sum(r[0] for r in res)
        busy = max(r[1] for r in res)
        vp = n * tot / E / busy / 1e9
        out.update({"value": vp, "cores": ncpu,
                    "sample": f"{tot} of {E} elements of {pr.name} p={pr.p} over {ncpu} processes "
                              f"x 1 BLAS thread ({busy:.1f} s each, {wall:.1f} s wall incl. "
                              f"spawn); 1 thread alone: {v1:.3g} GDOF/s; element matrices by "
                              f"direct quadrature + multiply, scaled to whole-apply DOFs"})
    return out


def oracle_minres(name: str):
    """The oracle's MINRES (reading A8/A10: Chebyshev-Jacobi S^-1) on a full config, one
    thread: setup (dense element matrices, assembly, S~) and time-to-solve, rtol 1e-12."""
    from threadpoolctl import threadpool_limits
    from oracle import operators, solvers
    from synth import make_config, random_vector
    pr = make_config(name)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        A = operators.Assembled(pr)
        P = solvers.BlockDiagPrecond(A)
        t1 = time.perf_counter()
        n = A.n_rt + A.n_l2
        b = A.apply_block(random_vector(n, 2 if name == "c2" else 1))
        t2 = time.perf_counter()
        _, it, conv, _ = solvers.minres(A.apply_block, P.apply, b, rtol=1e-12, maxit=5000)
        t3 = time.perf_counter()
    return {"iters": it, "converged": bool(conv), "setup_s": t1 - t0, "time_to_solve_s": t3 - t2,
            "cores": 1, "dofs": n}


def run_reference(args, ws, rank):
    """--impl reference: the oracle, as it stands, on the host cores; rank 0 only."""
    if rank != 0:
        return
    pr = make_problem(args.config, args.p)
    n = pr.n_rt() + pr.n_l2()
    per_step_budget = max(0.2, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    if args.ref_seconds is not None:
        per_step_budget = args.ref_seconds
    for _ in range(args.warmup):
        cpu_baseline(pr, budget_s=min(1.0, per_step_budget), cfg=args.config, parallel=False)
    vals = [cpu_baseline(pr, budget_s=per_step_budget, cfg=args.config)
            for _ in range(args.steps)]
    v = sorted(x["value"] for x in vals)[len(vals) // 2]
    cb = dict(vals[0])
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GDOF/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": n / (v * 1e9) * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "p": pr.p,
                       "N_RT": pr.n_rt(), "N_L2": pr.n_l2(),
                       "note": "each step: oracle element-by-element apply on a bounded "
                               "sample, scaled to the whole workload"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--impl", default="hdiv", choices=["hdiv", "reference"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-minres", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-seconds", type=float, default=None,
                    help="--impl reference: oracle seconds per step (default: ~120 s total)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: relaunch under torchrun (one process per GPU)
        import torch
        nvis = torch.cuda.device_count()
        if args.impl != "reference" and nvis < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {nvis} "
                              "CUDA devices are visible", "n_gpus": nvis}), flush=True)
            sys.exit(2)
        env = nccl_log_env(dict(os.environ))
        cmd = torchrun_argv(sys.argv[1:], args.gpus, _free_port())
        sys.exit(subprocess.call(cmd, env=env))
    if ws > 1 and args.gpus != ws:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws} ranks",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if ws > 1:
        nccl_log_env(os.environ)
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = td
        from paper_2304_12387_b200.binding import nccl_unique_id
        idl = [nccl_unique_id() if rank == 0 else None]
        td.broadcast_object_list(idl, src=0)
        nccl_id = idl[0]

    from paper_2304_12387_b200.binding import nccl_unique_id  # noqa: F401 (import check)
    pr = make_problem(args.config, args.p)
    n_glob = pr.n_rt() + pr.n_l2()
    t0 = time.time()
    op = build_operator(pr, ws, rank, dist, nccl_id)
    t_setup = time.time() - t0
    s = op.sizes
    x = torch.rand(s.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)

    clk = ClockSampler(local)
    clk.start()
    ms = time_applies(op, x, y, args.steps, args.warmup, dist, torch)
    clocks = clk.stop()
    ms_step = ms / args.steps
    value = n_glob / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel (the block-apply kernel: 1 launch per step on one GPU)
    peak, peak_src = _peaks()
    E_loc = op.sizes.n_l2 // (pr.p ** pr.dim)
    alg_bytes = 16 * s.n + 32 * E_loc        # read x, write y, 4 coefficients per element
    launches = op.apply_launches()
    achieved = alg_bytes / (ms_step * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        key = f"{args.config}_p{pr.p}"
        if key in tr and ws == 1:
            traffic = tr[key]["dram_bytes_per_launch"]
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "affine_apply_kernel (fused block apply)" if pr.affine else
                          "general_kernel (quadrature block apply)",
                "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src}

    # end-to-end through the C-ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if args.e2e_steps > 0:
        xh = torch.empty(s.n, dtype=torch.float64, pin_memory=True)
        yh = torch.empty(s.n, dtype=torch.float64, pin_memory=True)
        xh.copy_(x.cpu())
        op.apply_block_host(xh, yh)
        if dist is not None:
            dist.barrier()
        t1 = time.perf_counter()
        for _ in range(args.e2e_steps):
            op.apply_block_host(xh, yh)
        te = time.perf_counter() - t1
        if dist is not None:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": n_glob * args.e2e_steps / te / 1e9, "unit": "GDOF/s",
               "h2d_bytes_per_step": 8 * s.n, "d2h_bytes_per_step": 8 * s.n,
               "note": "hdiv_apply_block_host: pinned host x -> device, apply, device -> pinned "
                       "host y every step; box meshes pipeline ~32 z-chunks (H2D of chunk c+1 "
                       "and D2H of chunk c-1 overlap the fused apply of chunk c, three streams)"}
        # the PCIe ceiling of that number: the same bytes copied both ways at once (torch
        # copies on two streams, no apply) -> the e2e value a zero-cost apply would reach
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        ycp = torch.empty_like(x)

        def both():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                ycp.copy_(xh, non_blocking=True)
            with torch.cuda.stream(s2):
                yh.copy_(x, non_blocking=True)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        both()
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(2):
            both()
        c1.record()
        torch.cuda.synchronize()
        tc = c0.elapsed_time(c1) / 2 / 1e3
        e2e["pcie_ceiling"] = {"value": n_glob / tc / 1e9, "unit": "GDOF/s",
                               "copy_gbs_per_direction": 8 * s.n / tc / 1e9,
                               "frac": e2e["value"] / (n_glob / tc / 1e9)}
        del xh, yh, ycp

    result = {"metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": ws,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
              "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
              "dtype": "f64", "data": "synthetic",
              "config": {"workload": WORKLOADS.get(args.config, args.config), "p": pr.p,
                         "N": list(pr.N), "N_RT": pr.n_rt(), "N_L2": pr.n_l2(),
                         "global_dofs": n_glob, "parallelism": f"z-slabs x{ws}",
                         "l2_flush": "inputs larger than L2 (%.2f GB per vector vs 126 MB)"
                                     % (8 * n_glob / 1e9),
                         "setup_s": round(t_setup, 2)},
              "roofline": roofline, "e2e": e2e, "gpu_launches": launches * args.steps,
              "clocks": clocks}

    del x, y
    op.close()
    torch.cuda.empty_cache()

    # p sweep (1 GPU): GDOF/s for p = 2..6 on meshes that fill a similar memory footprint
    if not args.no_sweep and ws == 1 and args.config == "c4":
        sweep = {}
        for p in (2, 3, 4, 5, 6):
            Nn = {2: 160, 3: 128, 4: 128, 5: 96, 6: 80}[p]
            from synth import make_config
            prp = make_config("c4", N=(Nn, Nn, Nn), p=p)
            opp = build_operator(prp, 1, 0, None)
            xs = torch.rand(opp.sizes.n, dtype=torch.float64, device="cuda")
            ys = torch.empty_like(xs)
            msp = time_applies(opp, xs, ys, 30, 5, None, torch) / 30
            nn = opp.sizes.n
            ab = 16 * nn + 32 * prp.E
            sweep[f"p{p}"] = {"N": Nn, "dofs": nn, "ms": msp, "GDOF_s": nn / msp / 1e6,
                              "hbm_frac": ab / (msp * 1e-3) / 1e9 / peak}
            del xs, ys
            opp.close()
            torch.cuda.empty_cache()
        result["sweep"] = sweep

    # MINRES time-to-solve (config 2: 8^3 p=3 grad-div, rtol 1e-12, x0 = 0) with both S^-1
    # (Chebyshev-Jacobi, reading A10; one AMG V-cycle, P:889-891 / reading A9b), and at the
    # bench workload (config 4) the AMG solve to 1e-12 plus the per-iteration cost of both
    if not args.no_minres and ws == 1:
        from synth import make_config, random_vector
        from paper_2304_12387_b200 import from_problem
        pr2 = make_config("c2")
        mres = {"workload": "config 2: 8^3 Cartesian, p=3, grad-div alpha=beta=1, "
                            "b = A x*, rtol 1e-12 (P:899), x0 = 0"}
        for schur in ("chebyshev", "amg"):
            op2 = from_problem(pr2, schur=schur)
            xs = torch.from_numpy(random_vector(op2.sizes.n, 2)).cuda()
            b = op2.apply_block(xs)
            op2.minres(b, rtol=1e-12, maxit=5000)   # warm-up (graph build)
            # a ~5 ms solve is host-latency bound: the best of three
            rep = min((op2.minres(b, rtol=1e-12, maxit=5000)[1] for _ in range(3)),
                      key=lambda r: r.t_solve_ms)
            key = "" if schur == "chebyshev" else "amg_"
            mres[key + "iters"] = rep.iters
            mres[key + "converged"] = bool(rep.converged)
            mres[key + "time_to_solve_s"] = rep.t_solve_ms / 1e3
            op2.close()
            del xs, b
            torch.cuda.empty_cache()
        # config 1 (2D 4x4, p = 2, Darcy) on the GPU, and the oracle's MINRES on configs 1 and 2
        # in full, timed beside it on one host thread
        pr1 = make_config("c1")
        op1 = from_problem(pr1)
        xs1 = torch.from_numpy(random_vector(op1.sizes.n, 1)).cuda()
        b1 = op1.apply_block(xs1)
        op1.minres(b1, rtol=1e-12, maxit=5000)
        rep1 = min((op1.minres(b1, rtol=1e-12, maxit=5000)[1] for _ in range(3)),
                   key=lambda r: r.t_solve_ms)   # best of three (host-latency bound)
        mres["c1_iters"] = rep1.iters
        mres["c1_time_to_solve_s"] = rep1.t_solve_ms / 1e3
        op1.close()
        if not args.no_cpu:
            for nm in ("c1", "c2"):
                mres["oracle_" + nm] = oracle_minres(nm)
        mres["preconditioner"] = "diag(tau M~) + Chebyshev-Jacobi(S~), degree 4"
        mres["amg_preconditioner"] = ("diag(tau M~) + one smoothed-aggregation V-cycle on S~ "
                                      "(3^3 aggregates, 2+2 l1-Jacobi sweeps, Galerkin)")
        result["minres"] = mres
        # NEXT-4: GMRES(30) + block-triangular vs MINRES + block-diagonal (both with the AMG
        # S^-1) on config 5 at p=4 (graded two-material, 3.7M DOFs)
        pr5 = make_config("c5", p=4)
        op5 = from_problem(pr5, schur="amg")
        xs5 = torch.from_numpy(random_vector(op5.sizes.n, 5)).cuda()
        b5 = op5.apply_block(xs5)
        _, rm = op5.minres(b5, rtol=1e-12, maxit=5000)
        _, rg = op5.gmres(b5, rtol=1e-12, maxit=5000, restart=30)
        result["gmres"] = {"workload": "config 5 (24x24x25 graded two-material, p=4, grad-div), "
                                       "S^-1 = AMG V-cycle, rtol 1e-12, x0 = 0",
                           "gmres_tri_iters": rg.iters, "gmres_tri_time_s": rg.t_solve_ms / 1e3,
                           "gmres_converged": bool(rg.converged),
                           "minres_diag_iters": rm.iters, "minres_diag_time_s": rm.t_solve_ms / 1e3,
                           "note": "GMRES stops on the true residual (right preconditioning), "
                                   "MINRES on the preconditioned residual (reading A8)"}
        op5.close()
        del xs5, b5
        torch.cuda.empty_cache()
        if args.config == "c4":
            for schur in ("chebyshev", "amg"):
                op4 = from_problem(pr, schur=schur)
                n4 = op4.sizes.n
                xs4 = torch.rand(n4, dtype=torch.float64, device="cuda") * 2 - 1
                b4 = op4.apply_block(xs4)
                op4.minres(b4, rtol=1e-30, maxit=6)
                _, r4 = op4.minres(b4, rtol=1e-30, maxit=30)
                key = "c4_" if schur == "chebyshev" else "c4_amg_"
                mres[key + "ms_per_iteration"] = r4.t_solve_ms / max(r4.iters, 1)
                if schur == "amg":   # the full solve at the bench workload (537.7M DOFs)
                    x4, r5 = op4.minres(b4, rtol=1e-12, maxit=1000)
                    mres["c4_amg_iters"] = r5.iters
                    mres["c4_amg_converged"] = bool(r5.converged)
                    mres["c4_amg_time_to_solve_s"] = r5.t_solve_ms / 1e3
                    mres["c4_amg_solution_err"] = ((x4 - xs4).abs().max() / xs4.abs().max()).item()
                    del x4
                op4.close()
                del b4, xs4
                torch.cuda.empty_cache()

    # Crooked-pipe-shaped p sweep (config 5a, paper scale: 24x24x25 graded two-material hexes,
    # grad-div with the P:915 coefficients), MINRES + one AMG V-cycle for S^-1, rtol 1e-12, next
    # to the paper's own saddle-point solver on 4 V100 (Table crooked-pipe-gpu) as
    # context: same method and problem shape, different hardware, mesh and right-hand side
    if not args.no_minres and ws == 1:
        from synth import make_config, random_vector
        from paper_2304_12387_b200 import from_problem
        paper = {2: (193, 0.85, 356500), 3: (251, 1.52, 1190115), 4: (298, 2.19, 2805520),
                 5: (335, 3.49, 5461375), 6: (360, 4.01, 9416340)}
        cp = {"workload": "config 5a: 24x24x25 graded two-material box mesh (crooked-pipe analogue, "
                          "alpha/beta of P:915), grad-div, b = A x* (x* = U(-1,1), seed 5), x0 = 0, "
                          "rtol 1e-12, S^-1 = AMG V-cycle; paper: 4x V100, 14,370 hexes of the real "
                          "crooked pipe, constant forcing (context, not the target)"}
        for p in (2, 3, 4, 5, 6):
            prc = make_config("c5", p=p)
            opc = from_problem(prc, schur="amg", amg_cheb_degree=1)   # one V-cycle, as the paper
            bc = opc.apply_block(torch.from_numpy(random_vector(opc.sizes.n, 5)).cuda())
            opc.minres(bc, rtol=1e-12, maxit=6)   # warm-up (graph build)
            _, rc = opc.minres(bc, rtol=1e-12, maxit=5000)
            cp[f"p{p}"] = {"rt_dofs": opc.sizes.n_rt, "dofs": opc.sizes.n, "iters": rc.iters,
                           "converged": bool(rc.converged), "time_s": rc.t_solve_ms / 1e3,
                           "paper_4xV100": {"iters": paper[p][0], "time_s": paper[p][1],
                                            "rt_dofs": paper[p][2]}}
            opc.close()
            del bc
            torch.cuda.empty_cache()
        result["crooked_pipe_like"] = cp

    # NEXT-3: the SPE10-shaped pure-Neumann Darcy solve: config 3's jittered
    # 64^3 p=4 mesh and eps = 10^U(-2,2), u.n prescribed on every side (eliminated), gamma = 0,
    # singular S~ with the projection after every S^-1 (one AMG V-cycle); b = A x*
    if not args.no_minres and ws == 1:
        from synth import make_config, random_vector
        from paper_2304_12387_b200 import from_problem
        prs = make_config("c3s")
        t0s = time.time()
        ops = from_problem(prs, schur="amg", amg_cheb_degree=1)
        t_setup_s = time.time() - t0s
        xs = torch.rand(ops.sizes.n, dtype=torch.float64, device="cuda") * 2 - 1
        bs = ops.apply_block(xs)
        ops.minres(bs, rtol=1e-12, maxit=6)   # warm-up (graph build)
        xo, rs = ops.minres(bs, rtol=1e-12, maxit=5000)
        nrt = ops.sizes.n_rt
        dq = xo[nrt:] - xs[nrt:]
        result["spe10_like"] = {
            "workload": "config 3 mesh/coefficients (64^3 jittered hexes, p=4, eps=10^U(-2,2)), "
                        "u.n prescribed on all six sides, gamma=0: singular S~, projection "
                        "after every S^-1 (P:1035-1040); S^-1 = AMG V-cycle; rtol 1e-12",
            "dofs": ops.sizes.n, "iters": rs.iters, "converged": bool(rs.converged),
            "time_to_solve_s": rs.t_solve_ms / 1e3, "setup_s": round(t_setup_s, 2),
            "u_err": ((xo[:nrt] - xs[:nrt]).abs().max() / xs[:nrt].abs().max()).item(),
            "q_err_mod_const": ((dq - dq.mean()).abs().max() / xs[nrt:].abs().max()).item()}
        ops.close()
        del xo, dq
        torch.cuda.empty_cache()
        # reading A9d: S^-1 = degree-3 Chebyshev polynomial in (V-cycle) S~ — fewer MINRES
        # iterations for three V-cycles and two S~ applies per S^-1
        ops = from_problem(prs, schur="amg", amg_cheb_degree=3)
        ops.minres(bs, rtol=1e-12, maxit=6)
        xo, rs = ops.minres(bs, rtol=1e-12, maxit=5000)
        dq = xo[nrt:] - xs[nrt:]
        result["spe10_like"]["amg_chebyshev3"] = {
            "iters": rs.iters, "converged": bool(rs.converged),
            "time_to_solve_s": rs.t_solve_ms / 1e3,
            "u_err": ((xo[:nrt] - xs[:nrt]).abs().max() / xs[:nrt].abs().max()).item(),
            "q_err_mod_const": ((dq - dq.mean()).abs().max() / xs[nrt:].abs().max()).item()}
        ops.close()
        del xs, bs, xo, dq
        torch.cuda.empty_cache()
        # config 3 itself (Darcy, gamma = 0 but natural conditions: S~ nonsingular), b = A x*
        prc3 = make_config("c3")
        c3m = {"workload": WORKLOADS["c3"] + ", MINRES b = A x* (x* = U(-1,1)), x0 = 0, rtol 1e-12"}
        for k in (1, 3):
            opm = from_problem(prc3, schur="amg", amg_cheb_degree=k)
            xs = torch.rand(opm.sizes.n, dtype=torch.float64, device="cuda") * 2 - 1
            bs = opm.apply_block(xs)
            opm.minres(bs, rtol=1e-12, maxit=6)
            xo, rs = opm.minres(bs, rtol=1e-12, maxit=5000)
            c3m["amg" if k == 1 else "amg_chebyshev3"] = {
                "iters": rs.iters, "converged": bool(rs.converged),
                "time_to_solve_s": rs.t_solve_ms / 1e3,
                "solution_err": ((xo - xs).abs().max() / xs.abs().max()).item()}
            opm.close()
            del xs, bs, xo
            torch.cuda.empty_cache()
        result["config3_minres"] = c3m

    # Config 3's own apply (trilinear hexes: quadrature kernel, FP64-ALU-class):
    # GDOF/s and the fraction of the measured FP64 FMA peak (profiles/r01_fp64_peak.txt) for the
    # analytic flop count of the sum-factorised kernel
    if not args.no_minres and ws == 1:
        from synth import make_config
        from paper_2304_12387_b200 import from_problem
        pr3 = make_config("c3")
        P3_, Q3_ = pr3.p, pr3.p + 2
        fma = 0
        for c in range(3):   # forward interpolation of component c + its transpose
            E3 = [P3_ + 1 if a == c else P3_ for a in range(3)]
            fma += E3[1] * E3[2] * E3[0] * Q3_ + Q3_ * E3[2] * E3[1] * Q3_ + Q3_ * Q3_ * E3[2] * Q3_
        fp64_peak = 34.116   # measured, profiles/r01_fp64_peak.txt
        c3 = {}
        # tri_geometry 2: the paper's partial assembly (G_q = w_q mw / det J J^T J stored at the
        # Q^3 points, 48 B each: P:684); 1: J recomputed from the vertices every apply
        for geo, key in ((2, "stored_geometry"), (1, "on_the_fly_jacobian")):
            op3 = from_problem(pr3, tri_geometry=geo, schur="chebyshev")
            x3 = torch.rand(op3.sizes.n, dtype=torch.float64, device="cuda")
            y3 = torch.empty_like(x3)
            ms3 = time_applies(op3, x3, y3, 20, 5, None, torch) / 20
            pw = 18 if geo == 2 else 60   # pointwise flops per point: 3x3 G u | J, det, J^T J u
            flops_el = 2 * 2 * fma + pw * Q3_ ** 3 + 6 * P3_ ** 3 + 2 * 3 * P3_ ** 2 * (P3_ + 1)
            tf = flops_el * pr3.E / (ms3 * 1e-3) / 1e12
            alg = 16 * op3.sizes.n + (48 * Q3_ ** 3 if geo == 2 else 0) * pr3.E
            c3[key] = {"ms": ms3, "dofs": op3.sizes.n, "GDOF_s": op3.sizes.n / ms3 / 1e6,
                       "alu": {"achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                               "frac": tf / fp64_peak, "flops_per_element": flops_el},
                       "hbm": {"alg_bytes_per_launch": alg, "achieved": alg / (ms3 * 1e-3) / 1e9,
                               "frac": alg / (ms3 * 1e-3) / 1e9 / peak}}
            op3.close()
            del x3, y3
            torch.cuda.empty_cache()
        best = min(c3, key=lambda k: c3[k]["ms"])
        b = c3[best]
        result["config3_apply"] = {
            "workload": WORKLOADS["c3"] + " (block apply; gamma = 0: no W^-1)",
            "variant": best, "dofs": b["dofs"], "ms": b["ms"],
            "GDOF_s": b["GDOF_s"],
            "roofline": {"bound": "alu", "achieved": b["alu"]["achieved"], "peak": fp64_peak,
                         "unit": "TFLOP/s", "frac": b["alu"]["frac"],
                         "flops_per_element": b["alu"]["flops_per_element"],
                         "peak_source": "measured FP64 FMA microbenchmark (scripts/fp64_peak.cu)"},
            "hbm_frac": b["hbm"]["frac"], "variants": c3}
        # the same mesh with a nonzero (2,2) block (grad-div, alpha/beta = 10^U(-2,2)): Z by the
        # precomputed explicit element inverses fused into the batched kernel;
        # HBM roofline with the inverses' 8 p^3 B per L2 DOF counted as algorithmic bytes
        try:
            import numpy as np
            from synth import random_vector
            pr3.kind = "grad_div"
            pr3.alpha = 10.0 ** random_vector(pr3.E, 33, -2.0, 2.0)
            pr3.beta = 10.0 ** random_vector(pr3.E, 34, -2.0, 2.0)
            op3 = from_problem(pr3, schur="chebyshev")
            x3 = torch.rand(op3.sizes.n, dtype=torch.float64, device="cuda")
            y3 = torch.empty_like(x3)
            ms3 = time_applies(op3, x3, y3, 20, 5, None, torch) / 20
            alg = 16 * op3.sizes.n + 8 * P3_ ** 3 * op3.sizes.n_l2
            result["config3_graddiv_apply"] = {
                "workload": "config 3 mesh, grad-div alpha, beta = 10^U(-2,2) (block apply with "
                            "Z = W_alpha^-1 by the explicit element inverses)",
                "dofs": op3.sizes.n, "ms": ms3, "GDOF_s": op3.sizes.n / ms3 / 1e6,
                "roofline": {"bound": "hbm", "achieved": alg / (ms3 * 1e-3) / 1e9, "peak": peak,
                             "unit": "GB/s", "frac": alg / (ms3 * 1e-3) / 1e9 / peak,
                             "alg_bytes_per_launch": alg}}
            op3.close()
            del x3, y3
        except Exception as ex:   # reported, never fatal to the bench line
            result["config3_graddiv_apply"] = {"error": str(ex)[:200]}
        torch.cuda.empty_cache()

    # W^-1 benchmark of Table dg-mass-inv (NEXT-2): ~1.7e6 L2 DOFs on a jittered
    # hex mesh, 100 applications of the (2,2)-block inverse by the fused element-local CG
    if not args.no_minres and ws == 1:
        result["winv"] = winv_bench(torch)

    if rank == 0 and ws == 1 and not args.no_cpu:   # (the oracle baseline: N = 1 only)
        result["cpu_baseline"] = cpu_baseline(pr)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
