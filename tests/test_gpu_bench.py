"""bench.py end to end on the device (marked gpu): the single-process line
and the ShardedAdamWGS path under torch.distributed.run on one NCCL rank
(the multi-rank code: side-stream statistics all-reduce captured in the
step graph), on a small cloud."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
ARGS = ["--steps", "3", "--warmup", "3", "--no-cpu", "--no-legs", "--rows", "300000",
        "--e2e-steps", "3"]


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _check(d, n_gpus):
    assert d["n_gpus"] == n_gpus and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["frac"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["n_per_gpu"] == 300000


def test_bench_single_process():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *ARGS], capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    _check(_line(r.stdout), 1)


def test_bench_sharded_nccl_rank():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=1", "--master-addr", "127.0.0.1",
                        f"--master-port={_port()}", str(ROOT / "bench.py"), "--gpus", "1",
                        "--sharded", *ARGS], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    _check(d, 1)
    assert "index-sharded x1" in d["config"]["parallelism"]
