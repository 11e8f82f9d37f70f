"""Structural row operations around the step: MCMC relocation.

``mcmc_relocate`` (pipeline.py:197-233) respawns dead primitives (alive,
opacity <= 1/255) at opacity-weighted live targets. The decision stays on
the host with the caller's Generator, so the drawn targets are identical to
the reference's: which rows are dead, ``rng.choice`` over the live rows, and
the blend-preserving opacity 1 - (1 - o)^(1/(k+1)) in float64. The row
movement runs on the GPU in ``gs_relocate_rows``: copy every attribute from
the target, write the shared opacity logit to target and respawn, and zero
the respawns' moments and clock (reset_rows, optimizer.py:159-165).

Pruning, cloning and splitting (``densify_adc``) are row gathers and
concatenations of the parameter and state records: ``MomentState.select``
/ ``concatenate`` and torch indexing of the parameter record.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

from .engine import ConfigError, DomainError

ACTIVE_OPACITY = 1.0 / 255.0  # primitives.py:33


class SceneCollapseError(RuntimeError):
    """Relocation has no alive primitives left to respawn from (pipeline.py:57-58)."""


def opacity_f64(tau) -> np.ndarray:
    """activate_opacity (primitives.py:51-59) in float64, branch-stable."""
    t = np.asarray(tau, np.float64).reshape(-1)
    out = np.empty_like(t)
    pos = t >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-t[pos]))
    e = np.exp(t[~pos])
    out[~pos] = e / (1.0 + e)
    return out


@dataclass
class RelocationPlan:
    dead: np.ndarray      # int64, ascending
    targets: np.ndarray   # int64, one live row per dead row
    tau_new: np.ndarray   # float64 logit shared by each dead row and its target

    @property
    def count(self) -> int:
        return int(self.dead.size)

    def ids_hash(self) -> str:
        """The reference's event hash of the relocated rows (pipeline.py:94-96)."""
        data = np.sort(self.dead.astype(np.int64)).tobytes()
        return hashlib.blake2b(data, digest_size=8).hexdigest()


def mcmc_plan(tau, alive, rng: np.random.Generator) -> RelocationPlan:
    """The reference's relocation decision (pipeline.py:205-219) on host opacity logits."""
    o = opacity_f64(tau)
    alive = np.ones(o.size, bool) if alive is None else np.asarray(alive, bool).reshape(-1)
    if alive.size != o.size:
        raise ConfigError("alive must have one entry per row")
    dead = np.flatnonzero(alive & (o <= ACTIVE_OPACITY))
    live = np.flatnonzero(alive & (o > ACTIVE_OPACITY))
    if live.size == 0:
        raise SceneCollapseError("no alive primitives to relocate onto")
    if dead.size == 0:
        e = np.empty(0, np.int64)
        return RelocationPlan(e, e, np.empty(0, np.float64))
    probs = o[live] / o[live].sum()
    targets = live[rng.choice(live.size, size=dead.size, p=probs)]
    uniq, inverse, counts = np.unique(targets, return_inverse=True, return_counts=True)
    k = np.asarray(counts + 1.0, dtype=np.float64)
    o_new = 1.0 - np.power(1.0 - o[uniq], 1.0 / k)          # _clone_opacity, pipeline.py:110-113
    if np.any(o_new <= 0.0) or np.any(o_new >= 1.0):       # inverse_opacity's domain
        raise DomainError("opacity must lie strictly inside (0, 1)", uniq[(o_new <= 0.0) |
                                                                           (o_new >= 1.0)])
    tau_new = np.log(o_new / (1.0 - o_new))                  # inverse_opacity, primitives.py:69-75
    return RelocationPlan(dead.astype(np.int64), targets.astype(np.int64), tau_new[inverse])
