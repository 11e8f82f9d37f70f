"""Index-sharded multi-GPU AdamW-GS (one process per GPU, NCCL).

Rows are independent (the step never reads another row,
optimizer.py:252-265), so rank r of G owns the contiguous rows
[floor(rN/G), floor((r+1)N/G)) with their parameters, gradients, moments
and clocks.  The data path needs no exchange:

* compaction is local; the global index list is the rank-ordered
  concatenation of the local lists offset by each shard's base, i.e.
  bit-identical to np.flatnonzero of the global mask;
* RSR / relocation samples are drawn identically on every rank from the
  reference RNG contract and sliced with ``searchsorted``;
* only scalar statistics cross NVLink: one all-reduce(sum) of the step
  statistics (10 doubles), off the critical path.

The one real exchange is the coupled modes' normaliser N_v (loss.py:190):
the visible count is summed across ranks between compaction and the step,
on the compute stream, without a host sync.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .optimizer import AdamWGS
from .sampling import shard_rows


def shard_range(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range of a rank: [floor(rN/G), floor((r+1)N/G))."""
    return (n_global * rank) // world, (n_global * (rank + 1)) // world


def allreduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-step statistics of all ranks (every field is additive)."""
    out = stats.clone()
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def global_visible_count(count: torch.Tensor, group=None) -> torch.Tensor:
    """N_v over all shards (int32 sum), for the coupled normaliser."""
    out = count.clone()
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


class ShardedAdamWGS:
    """AdamWGS over this rank's shard of a globally indexed Gaussian cloud.

    ``param_groups`` hold the rank-local rows only (shape [hi-lo, ...]).
    """

    def __init__(self, param_groups, n_global: int, *, group=None, **kw):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n_global = int(n_global)
        self.lo, self.hi = shard_range(self.n_global, self.rank, self.world)
        self.opt = AdamWGS(param_groups, **kw)
        if self.opt.n_rows != self.hi - self.lo:
            raise ValueError(f"rank {self.rank} holds {self.opt.n_rows} rows, shard is "
                             f"[{self.lo}, {self.hi})")
        self.stats = torch.zeros_like(self.opt.engine.stats)

    def step(self, visibility_local: torch.Tensor, n_pixels=None, **kw):
        opt = self.opt
        if opt.mode in ("sparse-adam", "coupled-adam") and (opt.lambda_o or opt.lambda_s or
                                                             kw.get("lambda_o") or
                                                             kw.get("lambda_s")):
            _, count = opt.engine.compact(visibility_local)
            kw["n_visible"] = global_visible_count(count, self.group)
        opt.step(visibility_local, n_pixels, **kw)
        self.stats = allreduce_stats(opt.engine.stats, self.group)
        return self.stats

    def global_rows(self) -> torch.Tensor:
        """This shard's visible rows in global numbering (after a step)."""
        eng = self.opt.engine
        c = int(eng.count.item())
        return eng.idx[:c].to(torch.int64) + self.lo

    def rsr_apply(self, global_indices, alpha1: float, alpha2: float):
        import numpy as np
        local = shard_rows(np.asarray(global_indices, dtype=np.int64), self.lo, self.hi)
        self.opt.rsr_apply(local, alpha1, alpha2)

    def reset_rows(self, global_indices):
        import numpy as np
        local = shard_rows(np.asarray(global_indices, dtype=np.int64), self.lo, self.hi)
        self.opt.reset_rows(local)

    def aiu_apply(self, visibility_local: torch.Tensor, aiu, rng, iteration: int,
                  alive_local: torch.Tensor | None = None):
        """Sharded AIU (optimizer.py:425-450), picks bit-identical to one process.

        One all-gather of the per-rank invisible counts; every rank draws the
        global Bernoulli vector from the same stream and keeps its slice
        (sampling.aiu_shard_select). Returns this shard's picks in global
        numbering."""
        import numpy as np

        from .sampling import aiu_shard_select

        def draw(n_local, prob):
            dev = self.opt.device if dist.get_backend(self.group) == "nccl" else "cpu"
            mine = torch.tensor([n_local], dtype=torch.int64, device=dev)
            allc = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(allc, mine, group=self.group)
            return aiu_shard_select(rng, prob, [int(c.item()) for c in allc], self.rank)

        picked = self.opt.aiu_apply(visibility_local, aiu, rng, iteration, alive_local, draw=draw)
        return np.asarray(picked, np.int64) + self.lo

