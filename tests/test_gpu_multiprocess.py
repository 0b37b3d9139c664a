"""The multi-process path (pk_comm_init: VMM + POSIX-fd exchange over Unix
sockets) under torchrun, world 2. On a single-GPU box both ranks share
cuda:0 (their kernels time-slice); with >= 2 GPUs each rank gets its own."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_torchrun_world2():
    env = dict(os.environ)
    if torch.cuda.device_count() < 2:
        env["PK_TEST_DEVICE"] = "0"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "mp_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("multiprocess ok") == 2, r.stdout


@pytest.mark.parametrize("impl", ["pk", "reference"])
def test_bench_under_torchrun_world2(impl):
    """bench.py's N > 1 contract path (as the driver launches it): one JSON line
    from rank 0 with the whole-job value, e2e and roofline keys."""
    import json
    env = dict(os.environ)
    if torch.cuda.device_count() < 2:
        env.update(PK_BENCH_DEVICE="0", PK_BENCH_BACKEND="gloo")
    root = os.path.dirname(HERE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--size", "4096", "--impl", impl, "--cpu-seconds", "1"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    if impl == "pk":
        assert line["roofline"]["overlapped"]["t_roof_ms"] > 0 and line["gpu_launches"] == 6
    else:
        assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port"


def test_full_size_on_distinct_gpus():
    """World = every visible GPU, one rank each (needs >= 2): NVLS must be on,
    and the 1 GiB all-reduce, AG-GEMM / GEMM-RS at 16384, ring attention at
    32K and MoE at T 4096 must match NCCL + torch (mp_full_worker.py)."""
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip(f"needs >= 2 GPUs on distinct devices (this box has {ngpu}); the emulated and "
                    "same-GPU multi-process tests cover the single-GPU case")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpu}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "mp_full_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    import json
    reps = [json.loads(x.split("full-size ok ", 1)[1]) for x in r.stdout.splitlines() if "full-size ok " in x]
    assert len(reps) == ngpu, r.stdout
    assert all(x["distinct_devices"] for x in reps)
    assert all(x["nvls"] for x in reps), "NVLS multicast was not available on distinct GPUs"


def test_full_size_worker_logic_on_one_gpu():
    """The distinct-GPU worker above, at small sizes with both ranks on cuda:0
    and gloo collectives (PK_FULL_SMOKE=1): keeps its checks honest on a
    1-GPU box."""
    env = dict(os.environ, PK_FULL_SMOKE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "mp_full_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("full-size ok ") == 2, r.stdout
