"""bench.py's contract on the GPU (C1, a few steps): the single-GPU line and
the N > 1 z-slab path over NCCL, exercised with one rank (APRGPU_BENCH_SLAB=1)
since a one-GPU box cannot run two."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out: str) -> dict:
    return json.loads(out.strip().splitlines()[-1])


@pytest.mark.gpu
def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--rl-iters", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["gpu_launches"] > 0 and d["value"] > 0
    assert d["clocks"]["reasons"] != ["unsampled"]


@pytest.mark.gpu
def test_bench_slab_path_over_nccl():
    env = dict(os.environ, APRGPU_BENCH_SLAB="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1",
                        "--config", "c1", "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    for k in KEYS:
        assert k in d, k
    assert d["scaling"] == "strong" and d["gpu_launches"] > 0 and "z-slabs" in d["parallelism"]


@pytest.mark.gpu
def test_bench_weak_scaling_slab_workload():
    # the N > 1 workload (C3 tiled N times along z, one slab per GPU), at N = 2 on one rank
    env = dict(os.environ, APRGPU_BENCH_SLAB="1", APRGPU_BENCH_TILEZ="2")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1",
                        "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["scaling"] == "weak" and "2048 x 1024 x 1024" in d["config"]["workload"]
    assert d["config"]["particles"] > 30_000_000


@pytest.mark.gpu
def test_bench_c4_slab_path():
    # BASELINE config 4 through the N > 1 path (strong scaling of the C4 APR
    # over z-slabs; one rank here), as `bench.py --gpus N --config c4` runs it
    env = dict(os.environ, APRGPU_BENCH_SLAB="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1",
                        "--config", "c4", "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True,
                       timeout=1200, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["scaling"] == "strong" and d["config"]["particles"] == 547570496
    assert d["value"] > 0 and d["gpu_launches"] > 0
