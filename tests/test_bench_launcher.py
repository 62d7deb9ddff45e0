"""bench.py's multi-GPU launcher plumbing (CPU): `--gpus N` without WORLD_SIZE relaunches the
script under torchrun with N ranks; under torchrun rank 0 alone prints the reference line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_torchrun_argv():
    import bench
    cmd = bench.torchrun_argv(["--gpus", "4", "--steps", "5"], 4, 29555, python="py")
    assert cmd[:3] == ["py", "-m", "torch.distributed.run"]
    assert "--nnodes=1" in cmd and "--nproc-per-node=4" in cmd
    i = cmd.index("--master-addr")
    assert cmd[i + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29555"
    assert cmd[-5:] == [os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "5"]


def test_nccl_log_env_keeps_user_settings():
    import bench
    env = bench.nccl_log_env({"NCCL_DEBUG": "WARN"})
    assert env["NCCL_DEBUG"] == "WARN" and env["NCCL_DEBUG_FILE"] == "/dev/stderr"


def test_relaunch_two_ranks_reference_line():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "3", "--config", "c2",
                        "--ref-seconds", "0.3"], capture_output=True, text=True, env=env,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout           # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
