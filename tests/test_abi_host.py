"""CPU tests: the C-ABI library loads and exports every declared symbol, and
the host-side logic (bias LUT, thresholds, N_I rounding, RSR sampling,
sharding) matches the reference / oracle.  No kernel is launched here."""

import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

from _golden import GOLDEN
from oracle import adamw_gs_oracle as O

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "adamw_gs.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2601_16736_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes binding out of sync with the header"
    assert lib.gs_abi_version() == _lib.GS_ABI_VERSION


def test_library_is_sm100a():
    import subprocess
    from paper_2601_16736_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_ctypes_struct_layout_matches_header(tmp_path):
    """Compile the header with gcc and compare every field offset and the
    struct sizes with the ctypes mirror."""
    import subprocess
    from paper_2601_16736_b200 import _lib
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "adamw_gs.h"',
             'int main(void) {']
    for cname, py in (("gs_group", _lib.GsGroup), ("gs_step_cfg", _lib.GsStepCfg)):
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(HEADER.parent), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in (("gs_group", _lib.GsGroup), ("gs_step_cfg", _lib.GsStepCfg)):
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_workspace_queries_without_gpu():
    from paper_2601_16736_b200 import _lib
    lib = _lib.load()
    assert lib.gs_compact_workspace_bytes(0) >= 4
    assert lib.gs_compact_workspace_bytes(6_000_000) == 4 * (((6_000_000 + 8191) // 8192) * 257 + 1)
    assert lib.gs_step_workspace_bytes() > 0


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_16736_b200._lib import ExtensionMissing
    from paper_2601_16736_b200.engine import StepEngine
    with pytest.raises(ExtensionMissing):
        StepEngine(10, torch.device("cpu"), 0.9, 0.999)


def test_active_threshold_product_equals_oracle():
    from paper_2601_16736_b200.engine import active_logit_threshold
    assert np.float32(active_logit_threshold()) == O.active_logit_threshold_f32()


def test_bias_lut_matches_oracle_and_saturates():
    from paper_2601_16736_b200.engine import bias_lut
    lut = bias_lut(0.9, 0.999)
    ref = O.bias_lut_f32(0.9, 0.999, lut.shape[0] - 1)
    assert np.array_equal(lut, ref)
    assert lut[-1, 0] == 1.0 and lut[-1, 1] == 1.0   # clamping the clock is exact
    t = np.arange(lut.shape[0], lut.shape[0] + 1000, dtype=np.float64)
    assert np.all((1.0 / (1.0 - np.power(0.999, t))).astype(np.float32) == 1.0)


def test_round_pixel_count_known_answers():
    from paper_2601_16736_b200.engine import ConfigError, round_pixel_count
    meta = json.loads(str(np.load(GOLDEN / "rsr_stats.npz")["meta"]))
    for k, want in meta["round_pixel_count"]:
        assert round_pixel_count(k) == want
    assert round_pixel_count(1024, enabled=False) == 1024.0
    with pytest.raises(ConfigError):
        round_pixel_count(0)


def test_stss_sample_product_bit_exact_with_reference():
    from paper_2601_16736_b200.sampling import StSSchedule, stream, stss_sample
    z = np.load(GOLDEN / "rsr_stats.npz")
    meta = json.loads(str(z["meta"]))
    for i, (seed, boundary, n_p, ratio) in enumerate(meta["stss"]):
        sched = StSSchedule(milestones=((0, ratio),), interval=10)
        idx = stss_sample(sched, boundary, n_p, stream(seed, "stss", boundary))
        assert np.array_equal(idx, z[f"stss_{i}"])


def test_stss_schedule_validation():
    from paper_2601_16736_b200.engine import ConfigError
    from paper_2601_16736_b200.sampling import RsrConfig, StSSchedule
    with pytest.raises(ConfigError):
        StSSchedule(milestones=((10, 0.1), (5, 0.2)))
    with pytest.raises(ConfigError):
        StSSchedule(milestones=((0, 1.5),))
    with pytest.raises(ConfigError):
        RsrConfig(alpha1=1.0)
    s = StSSchedule(milestones=((0, 0.05), (775, 0.25)))
    assert s.ratio_at(774) == 0.05 and s.ratio_at(775) == 0.25


def test_shard_rows_partition():
    from paper_2601_16736_b200.sampling import shard_rows
    from paper_2601_16736_b200.sharded import shard_range
    rng = np.random.default_rng(0)
    n = 1_000_003
    idx = np.sort(rng.choice(n, 250_000, replace=False))
    for world in (1, 2, 3, 8):
        parts = []
        for r in range(world):
            lo, hi = shard_range(n, r, world)
            loc = shard_rows(idx, lo, hi)
            assert loc.size == 0 or (loc.min() >= 0 and loc.max() < hi - lo)
            parts.append(loc + lo)
        assert np.array_equal(np.concatenate(parts), idx)


def test_optimizer_config_validation():
    from paper_2601_16736_b200.optimizer import ConfigError, OptimizerConfig
    with pytest.raises(ConfigError):
        OptimizerConfig(mode="sgd")
    with pytest.raises(ConfigError):
        OptimizerConfig(beta1=1.0)
    with pytest.raises(ConfigError):
        OptimizerConfig(ct_opacity=0.0)
    cfg = OptimizerConfig(lr_extra={"f_rest": 1e-4})
    assert cfg.lr("xyz") == cfg.lr_mu and cfg.lr("opacity") == cfg.lr_tau
    assert cfg.lr("f_rest") == 1e-4


def test_algorithmic_bytes_matches_baseline_md():
    from paper_2601_16736_b200.synthetic import algorithmic_bytes
    # 6M at 30% -> 3.001 GB; 1,664 B per visible primitive
    assert algorithmic_bytes(6_000_000, 1_800_000) == 6_000_000 + 1_800_000 * 1664
