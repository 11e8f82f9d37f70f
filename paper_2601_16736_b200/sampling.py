"""Host-side state sampling for Re-State Regularization (RSR).

Transcription note: ``_label_key``, ``stream``, ``RngHub``, ``StSSchedule``,
``RsrConfig``, ``AiuConfig`` and ``stss_sample`` restate the reference's
definitions (rng.py:17-43, optimizer.py:343-422) nearly line for line, error
strings included: the reference's config schema is the API, and the RNG /
selection contract must be bit-identical for the sampled rows to match.
``shard_rows``, ``aiu_shard_select`` and ``device_bernoulli`` are new.

The sampled row set must be bit-identical to the reference's, so it is drawn
on the host with the reference's counter-based stream contract — Philox
keyed by (seed, blake2b-4(label), indices) (rng.py:17-30) — and uploaded to
the GPU as a sorted int32 index list for ``gs_rsr_apply``.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from .engine import ConfigError


def _label_key(label: str) -> int:
    """rng.py:12-14 — 32-bit little-endian blake2b digest of the label."""
    return int.from_bytes(hashlib.blake2b(label.encode("utf-8"), digest_size=4).digest(), "little")


def stream(seed: int, label: str, *indices: int) -> np.random.Generator:
    """rng.py:17-30 — the same (seed, label, indices) always yield the same draws."""
    key = (_label_key(label), *(int(i) & 0xFFFFFFFF for i in indices))
    ss = np.random.SeedSequence(entropy=int(seed), spawn_key=key)
    return np.random.Generator(np.random.Philox(ss))


class RngHub:
    """rng.py:33-43 — stream factory bound to one experiment seed."""

    def __init__(self, seed: int):
        self.seed = int(seed)

    def stream(self, label: str, *indices: int) -> np.random.Generator:
        return stream(self.seed, label, *indices)


@dataclass(frozen=True)
class StSSchedule:
    """Milestone sampling ratios (optimizer.py:343-364); ratio 0 before the first."""

    milestones: tuple = ()
    interval: int = 10

    def __post_init__(self):
        iters = [it for it, _ in self.milestones]
        if any(b <= a for a, b in zip(iters, iters[1:])):
            raise ConfigError("milestones must be strictly increasing")
        if any(not (0.0 <= r <= 1.0) for _, r in self.milestones):
            raise ConfigError("sampling ratios must lie in [0, 1]")
        if self.interval < 1:
            raise ConfigError("interval must be >= 1")

    def ratio_at(self, iteration: int) -> float:
        out = 0.0
        for it, ratio in self.milestones:
            if iteration >= it:
                out = ratio
        return out


@dataclass(frozen=True)
class RsrConfig:
    """optimizer.py:367-376."""

    alpha1: float = 0.2
    alpha2: float = 0.04
    schedule: StSSchedule = field(default_factory=StSSchedule)
    enabled: bool = False

    def __post_init__(self):
        if not (0.0 <= self.alpha1 < 1.0 and 0.0 <= self.alpha2 < 1.0):
            raise ConfigError("RSR factors must lie in [0, 1)")


@dataclass(frozen=True)
class AiuConfig:
    """Artificial implicit updates for sampled invisible primitives
    (optimizer.py:389-422)."""

    start: int = 0
    end: int = -1  # inclusive; -1 disables
    prob_schedule: tuple = ()  # ((iteration, probability), ...)
    eta_schedule: tuple = ()  # ((iteration, step scale), ...)
    enabled: bool = False

    def __post_init__(self):
        for sched in (self.prob_schedule, self.eta_schedule):
            iters = [it for it, _ in sched]
            if any(b <= a for a, b in zip(iters, iters[1:])):
                raise ConfigError("schedule milestones must be strictly increasing")
        if any(not (0.0 <= p <= 1.0) for _, p in self.prob_schedule):
            raise ConfigError("sampling probabilities must lie in [0, 1]")

    def active(self, iteration: int) -> bool:
        return self.enabled and self.start <= iteration <= self.end

    @staticmethod
    def _at(schedule, iteration: int) -> float:
        out = 0.0
        for it, val in schedule:
            if iteration >= it:
                out = val
        return out

    def prob_at(self, iteration: int) -> float:
        return self._at(self.prob_schedule, iteration)

    def eta_at(self, iteration: int) -> float:
        return self._at(self.eta_schedule, iteration)


def stss_sample(schedule: StSSchedule, iteration: int, n_p: int,
                rng: np.random.Generator) -> np.ndarray:
    """optimizer.py:379-386 — floor(ratio*N_p) distinct rows, sorted, int64."""
    ratio = schedule.ratio_at(iteration)
    k = int(math.floor(ratio * n_p))
    if k <= 0:
        return np.empty(0, dtype=np.int64)
    return np.sort(rng.choice(n_p, size=k, replace=False).astype(np.int64))


def shard_rows(indices: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Rows of a sorted global sample that fall in the shard [lo, hi), made local.

    Every rank draws the same global sample (same seed/label/boundary) and
    keeps its slice — no communication.
    """
    a = np.searchsorted(indices, lo, side="left")
    b = np.searchsorted(indices, hi, side="left")
    return indices[a:b] - lo


def aiu_shard_select(rng: np.random.Generator, prob: float, counts, rank: int) -> np.ndarray:
    """AIU Bernoulli picks of one index shard, bit-identical to the
    single-process draw (optimizer.py:437-440).

    The reference draws ``rng.random(invisible.size) < prob`` over the global
    invisible list. With contiguous row shards that list is the rank-ordered
    concatenation of the local lists. So every rank draws the same global
    vector from the same stream and keeps its slice at the exclusive scan of
    ``counts``, the per-rank invisible counts (one all-gather).
    """
    counts = [int(c) for c in counts]
    off = sum(counts[:rank])
    draw = rng.random(sum(counts)) < prob
    return draw[off:off + counts[rank]]


def device_bernoulli(rng: np.random.Generator, n_total: int, prob: float, first: int, n: int,
                     device):
    """``(rng.random(n_total) < prob)[first:first + n]`` as a uint8 CUDA
    tensor, and ``rng`` advanced exactly as that host draw advances it.

    With the reference's Philox streams (rng.py:17-30) the draws are made
    on the device by gs_philox_bernoulli, bit for bit (the numbers the
    buffered outputs still hold come from the host); any other bit
    generator is drawn on the host and uploaded."""
    import torch

    from . import _lib as L
    n_total, first, n = int(n_total), int(first), int(n)
    out = torch.empty(max(n, 0), dtype=torch.uint8, device=device)
    if n_total <= 0:
        return out
    st = rng.bit_generator.state
    if st.get("bit_generator") != "Philox":
        sel = rng.random(n_total) < prob
        out.copy_(torch.from_numpy(sel[first:first + n].view(np.uint8)))
        return out
    pos = int(st["buffer_pos"])
    pre = min(4 - pos, n_total) if pos < 4 else 0
    head = (rng.random(pre) < prob) if pre else np.empty(0, bool)   # the buffered draws
    a, b = first, min(first + n, pre)
    if b > a:
        out[: b - a].copy_(torch.from_numpy(head[a:b].view(np.uint8)))
    rest = n_total - pre
    if rest <= 0:
        return out
    st2 = rng.bit_generator.state           # buffer empty now: draw j >= pre is block (j-pre)/4
    ctr = np.asarray(st2["state"]["counter"], np.uint64)
    key = np.asarray(st2["state"]["key"], np.uint64)
    d0 = max(first, pre)
    dn = first + n - d0
    if dn > 0:
        lib = L.load()
        c = (L.C.c_uint64 * 4)(*[int(x) for x in ctr])
        k = (L.C.c_uint64 * 2)(*[int(x) for x in key])
        with torch.cuda.device(out.device):
            rc = lib.gs_philox_bernoulli(c, k, d0 - pre, dn, float(prob),
                                         out[d0 - first:].data_ptr(),
                                         torch.cuda.current_stream(out.device).cuda_stream)
        L.check(rc, "gs_philox_bernoulli")
    # advance the host generator past the `rest` device draws: the counter
    # moves by all but the last block, which a host draw regenerates into
    # the buffer with the right position
    blocks = (rest + 3) // 4
    v = sum(int(x) << (64 * i) for i, x in enumerate(ctr)) + blocks - 1
    st2["state"]["counter"] = np.array([(v >> (64 * i)) & ((1 << 64) - 1) for i in range(4)],
                                       dtype=np.uint64)
    st2["buffer_pos"] = 4
    rng.bit_generator.state = st2
    rng.random(rest - 4 * (blocks - 1))
    return out
