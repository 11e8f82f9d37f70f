"""bench.py's launch contract on a host without GPUs (CPU): --gpus N outside
torchrun launches N ranks itself only when the node has N GPUs, and under a
launcher --gpus must equal WORLD_SIZE; both fail loudly otherwise."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, env=e, timeout=300)


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") not in (None, ""), reason="CPU check")
def test_gpus_without_enough_devices_fails_loudly():
    import torch
    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        pytest.skip("this host has the GPUs")
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 2
    assert "needs 2 GPUs" in r.stderr


def test_gpus_must_match_world_size():
    r = _run(["--gpus", "1"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=2" in r.stderr
