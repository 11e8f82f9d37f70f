"""The fused kernels' alternative dealings, forced through the library's
measurement switches (environment, read once per process, hence one
subprocess per case): the two-phase kernel on i.i.d. masks of every size
(GS_FUSED_MODE=2), per-CTA mask slices on a big cloud (GS_MASK_SLICES=1),
tiles dealt grid-stride on a small one (GS_MASK_SLICES=2), the bias warp on
both (GS_TMA4_BW=1), the 3-CTA-per-SM sparse-mask shape on any cloud
(GS_LOWVIS_SHAPE), and dynamic tails of the tile dealing from one to seven
eighths (GS_DYN_TAIL).  Each equals K1 + K2 bit for bit (marked
gpu)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BODY = Path(__file__).resolve().parent / "_fused_env_check.py"


@pytest.mark.parametrize("env,n,kind,mode,p", [
    ({"GS_FUSED_MODE": "2"}, 100_003, "bool", "adamw-gs", 0.3),
    ({"GS_FUSED_MODE": "2"}, 5_000_011, "bool", "adamw-gs", 0.05),
    ({"GS_FUSED_MODE": "2"}, 1_300_001, "radii", "adamw-const", 0.3),
    ({"GS_FUSED_MODE": "2", "GS_TMA4_BW": "0"}, 300_007, "bool", "sparse-adam", 0.3),
    ({"GS_MASK_SLICES": "1"}, 5_000_011, "bool", "adamw-gs", 0.3),
    ({"GS_MASK_SLICES": "1"}, 5_000_011, "radii", "adamw-gs", 0.01),
    ({"GS_MASK_SLICES": "2"}, 300_007, "bool", "adamw-gs", 0.3),
    ({"GS_TMA4_BW": "1"}, 300_007, "bool", "adamw-gs", 0.5),
    ({"GS_TMA4_BW": "1", "GS_MASK_SLICES": "2"}, 5_000_011, "bool", "adamw-gs", 0.3),
    ({"GS_TMA4_BW": "1", "GS_LOWVIS_SHAPE": "1"}, 5_000_011, "bool", "adamw-gs", 0.02),
    ({"GS_TMA4_BW": "1", "GS_LOWVIS_SHAPE": "1"}, 200_003, "bool", "sparse-adam", 0.02),
    ({"GS_TMA4_BW": "1", "GS_LOWVIS_SHAPE": "2"}, 1_000_003, "bool", "adamw-const", 0.3),
    ({"GS_DYN_TAIL": "1"}, 5_000_011, "bool", "adamw-gs", 0.3),
    ({"GS_DYN_TAIL": "7"}, 5_000_011, "radii", "adamw-const", 0.1),
    ({"GS_DYN_TAIL": "4", "GS_TMA4_BW": "1"}, 5_000_011, "bool", "sparse-adam", 0.02),
])
def test_forced_fused_dealing_equals_index_path(env, n, kind, mode, p):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, str(BODY), str(n), kind, mode, str(p)], env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]
