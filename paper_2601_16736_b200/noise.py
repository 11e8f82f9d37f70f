"""Opacity-gated position noise (optimizer.py:453-486) on the GPU.

The pipeline adds the returned perturbation to the positions of every alive
row after the step (pipeline.py:334-336).  The reference draws gamma from a
host NumPy Generator; here gamma comes from a counter-based Philox stream
keyed by (seed, row, iteration) inside ``gs_noise_perturb`` — statistically
equivalent, reproducible, and free of a host round trip.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .engine import ConfigError, row_stride


@dataclass(frozen=True)
class NoiseConfig:
    """optimizer.py:453-460."""

    enabled: bool = False
    lambda_mu: float = 100.0  # gate sharpness
    lambda_t: float = 0.005   # gate centre opacity
    eta_ratio: float = 1.0    # eta_Ro / eta_mu


def _check(name, t, n, w) -> int:
    """Row stride of a CUDA fp32 [n, w] tensor (dense or a record view)."""
    if t.dtype != torch.float32 or not t.is_cuda:
        raise ConfigError(f"{name} must be a CUDA fp32 tensor with {n} x {w} values")
    return row_stride(name, t, n, w)


@torch.no_grad()
def noise_perturb(position: torch.Tensor, log_scale: torch.Tensor, rotation: torch.Tensor,
                  opacity_logit: torch.Tensor, lr_position: float, cfg: NoiseConfig, seed: int,
                  iteration: int, alive: torch.Tensor | None = None,
                  add: bool = False) -> torch.Tensor:
    """Delta ``[N, D]`` (D = 2: angle rotation; D = 3: quaternion rotation);
    with ``add=True`` it is also added to ``position`` in place."""
    n = int(position.shape[0])
    dims = position.numel() // max(n, 1) if n else (2 if rotation.dim() == 1 else 3)
    if dims not in (2, 3):
        raise ConfigError("positions must be 2-D or 3-D")
    strides = (C.c_int64 * 4)(_check("position", position, n, dims),
                              _check("log_scale", log_scale, n, dims),
                              _check("rotation", rotation, n, 1 if dims == 2 else 4),
                              _check("opacity_logit", opacity_logit, n, 1))
    if alive is not None:
        alive = alive.to(torch.uint8).contiguous() if alive.dtype == torch.bool else alive
    delta = torch.empty((n, dims), dtype=torch.float32, device=position.device)
    lib = L.load()
    rc = lib.gs_noise_perturb(position.data_ptr(), log_scale.data_ptr(), rotation.data_ptr(),
                              opacity_logit.data_ptr(),
                              None if alive is None else alive.data_ptr(), n, dims,
                              float(lr_position), float(cfg.eta_ratio), float(cfg.lambda_mu),
                              float(cfg.lambda_t), int(seed) & (2**64 - 1),
                              int(iteration) & 0xFFFFFFFF, delta.data_ptr(), int(bool(add)),
                              strides, torch.cuda.current_stream(position.device).cuda_stream)
    L.check(rc, "gs_noise_perturb")
    return delta


def seed_from_generator(rng: np.random.Generator) -> int:
    """A 64-bit Philox key drawn from the caller's stream (the reference's
    ``hub.stream("noise", it)``, pipeline.py:335), so the noise stays a pure
    function of the experiment seed and iteration."""
    return int(rng.integers(0, 2**63 - 1, dtype=np.int64))
