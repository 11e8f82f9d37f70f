"""Seeded synthetic Gaussian clouds for tests and benchmarks.

Parameters (SH-3 layout, fp32):
    xyz ~ N(0, 5^2), f_dc ~ N(0, 0.5^2), f_rest ~ N(0, 0.05^2),
    opacity logit ~ N(-1, 2^2), scaling ~ U(ln 1e-3, ln 0.5), rotation ~ N(0, 1)
Gradients: g = z * s, z ~ N(0, 1), s ~ logU(1e-7, 1e-2); invisible rows are
exactly 0 (the renderer contract, renderer.py:222).
Visibility: i.i.d. Bernoulli(p) rows, or index-coherent 64-row blocks.

Host (NumPy, seeded per (label, step)) generators serve the parity tests;
the ``*_device`` generators build the large benchmark clouds directly in
HBM with a seeded torch CUDA generator.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .sampling import stream

SH3_LAYOUT = (("xyz", 3), ("f_dc", 3), ("f_rest", 45), ("opacity", 1), ("scaling", 3),
              ("rotation", 4))
SH3_WIDTH = sum(w for _, w in SH3_LAYOUT)  # 59 floats per primitive
EXTENT = 5.0
# optimizer.py:76-80, config.py:210; f_rest = f_dc / 20 as in 3DGS
LR_SH3 = {"xyz": 1.6e-4 * EXTENT, "f_dc": 2.5e-3, "f_rest": 2.5e-3 / 20.0, "opacity": 0.05,
          "scaling": 5e-3, "rotation": 1e-3}


@dataclass(frozen=True)
class WorkloadConfig:
    n: int
    p_vis: float = 0.3
    mask_family: str = "bernoulli"  # or "coherent" (64-row blocks)
    seed: int = 0
    lambda_o: float = 1e-3          # presets.py:42-46
    lambda_s: float = 1e-5
    n_pixels: int = 1_000_000       # N_I' = 100,000
    block: int = 64


def make_params(cfg: WorkloadConfig) -> dict:
    n = cfg.n
    r = lambda lab: stream(cfg.seed, "param-" + lab)  # noqa: E731
    f32 = np.float32
    return {
        "xyz": r("xyz").normal(0.0, 5.0, (n, 3)).astype(f32),
        "f_dc": r("f_dc").normal(0.0, 0.5, (n, 3)).astype(f32),
        "f_rest": r("f_rest").normal(0.0, 0.05, (n, 45)).astype(f32),
        "opacity": r("opacity").normal(-1.0, 2.0, (n, 1)).astype(f32),
        "scaling": r("scaling").uniform(math.log(1e-3), math.log(0.5), (n, 3)).astype(f32),
        "rotation": r("rotation").normal(0.0, 1.0, (n, 4)).astype(f32),
    }


def param_groups(params: dict, cfg: WorkloadConfig | None = None) -> list:
    return [{"params": [params[name]], "lr": LR_SH3[name], "name": name} for name, _ in SH3_LAYOUT]


def visibility(cfg: WorkloadConfig, step: int) -> np.ndarray:
    rng = stream(cfg.seed, "vis", step)
    if cfg.mask_family == "coherent":
        nb = (cfg.n + cfg.block - 1) // cfg.block
        return np.repeat(rng.random(nb) < cfg.p_vis, cfg.block)[: cfg.n]
    return rng.random(cfg.n) < cfg.p_vis


def step_grads(cfg: WorkloadConfig, step: int, vis: np.ndarray) -> dict:
    rng = stream(cfg.seed, "grad", step)
    out = {}
    for name, w in SH3_LAYOUT:
        s = np.exp(rng.uniform(math.log(1e-7), math.log(1e-2), (cfg.n, w)))
        g = (rng.standard_normal((cfg.n, w)) * s).astype(np.float32)
        g[~vis] = 0.0
        out[name] = g
    return out


# ---------------------------------------------------------------- device-side
def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def make_params_device(cfg: WorkloadConfig, device) -> dict:
    g = _gen(device, cfg.seed * 7919 + 1)
    n = cfg.n
    kw = dict(device=device, dtype=torch.float32, generator=g)
    return {
        "xyz": torch.randn((n, 3), **kw) * 5.0,
        "f_dc": torch.randn((n, 3), **kw) * 0.5,
        "f_rest": torch.randn((n, 45), **kw) * 0.05,
        "opacity": torch.randn((n, 1), **kw) * 2.0 - 1.0,
        "scaling": torch.rand((n, 3), **kw) * (math.log(0.5) - math.log(1e-3)) + math.log(1e-3),
        "rotation": torch.randn((n, 4), **kw),
    }


def visibility_device(cfg: WorkloadConfig, step: int, device) -> torch.Tensor:
    g = _gen(device, cfg.seed * 1_000_003 + 17 + step)
    if cfg.mask_family == "coherent":
        nb = (cfg.n + cfg.block - 1) // cfg.block
        blocks = torch.rand(nb, device=device, generator=g) < cfg.p_vis
        return blocks.repeat_interleave(cfg.block)[: cfg.n].contiguous()
    return torch.rand(cfg.n, device=device, generator=g) < cfg.p_vis


def grads_device(cfg: WorkloadConfig, step: int, device, vis: torch.Tensor | None = None) -> dict:
    g = _gen(device, cfg.seed * 104_729 + 31 + step)
    out = {}
    lo, hi = math.log(1e-7), math.log(1e-2)
    for name, w in SH3_LAYOUT:
        s = torch.exp(torch.rand((cfg.n, w), device=device, generator=g) * (hi - lo) + lo)
        x = torch.randn((cfg.n, w), device=device, generator=g) * s
        if vis is not None:
            x.mul_(vis.view(-1, 1).to(x.dtype))
        out[name] = x.contiguous()
    return out


def algorithmic_bytes(n: int, n_visible: int, width: int = SH3_WIDTH, mask_bytes: int = 1) -> int:
    """Bytes one step must move: N*m_b + N_v*(28*P + 12).

    28*P: read theta, g, m, v and write theta, m, v (fp32); +8 clock r/w;
    +4 the int32 index written by the compaction.
    """
    return n * mask_bytes + n_visible * (28 * width + 12)
