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
* only scalars cross NVLink: one all-reduce(sum) of the step statistics (10
  doubles).  In the decoupled modes it runs on a side stream behind an
  event, off the step's critical path.

Two exchanges sit on the critical path because the reference's semantics
need them: the coupled modes' normaliser N_v (loss.py:190) is summed across
ranks between compaction and the step (an int32 all-reduce on the compute
stream, no host sync), and the strict check's abort flag is max-reduced
between the all-row pre-check and the step, so a non-finite gradient on any
shard aborts the step on every shard (optimizer.py:248: nothing is mutated).

Errors are decided on the all-reduced statistics, so every rank raises the
same GradientError / DomainError (with the global row ids) at the same step;
no rank can leave the others blocked in a collective.
"""

from __future__ import annotations

import collections

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .engine import ConfigError, DomainError, GradientError
from .optimizer import ERRORS, AdamWGS, _stats_dict
from .sampling import shard_rows


def shard_range(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range of a rank: [floor(rN/G), floor((r+1)N/G))."""
    return (n_global * rank) // world, (n_global * (rank + 1)) // world


def _host_collective(group) -> bool:
    """gloo moves host tensors: device tensors go through a host copy."""
    return dist.get_backend(group) != "nccl"


def _all_reduce_(t: torch.Tensor, op=dist.ReduceOp.SUM, group=None) -> torch.Tensor:
    """In-place all-reduce on the current stream (NCCL), or through a host
    copy for host-side backends (gloo, the CPU tests)."""
    if t.is_cuda and _host_collective(group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def allreduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-step statistics of all ranks (every field is additive)."""
    return _all_reduce_(stats.clone(), dist.ReduceOp.SUM, group)


def global_visible_count(count: torch.Tensor, group=None) -> torch.Tensor:
    """N_v over all shards (int32 sum), for the coupled normaliser."""
    return _all_reduce_(count.clone(), dist.ReduceOp.SUM, group)


class ShardedAdamWGS:
    """AdamWGS over this rank's shard of a globally indexed Gaussian cloud.

    ``param_groups`` hold the rank-local rows only (shape [hi-lo, ...]);
    ``**kw`` are AdamWGS's options (``errors`` applies to the whole job).
    """

    STAT_SLOTS = 4  # per-step statistics buffers in flight on the side stream

    def __init__(self, param_groups, n_global: int, *, group=None, errors: str = "defer", **kw):
        if errors not in ERRORS:
            raise ConfigError(f"errors must be one of {ERRORS}")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n_global = int(n_global)
        self.lo, self.hi = shard_range(self.n_global, self.rank, self.world)
        self.errors = errors
        # the wrapper decides errors on the reduced statistics; the shard
        # optimizer only counts
        self.opt = AdamWGS(param_groups, errors="ignore", **kw)
        if self.opt.n_rows != self.hi - self.lo:
            raise ValueError(f"rank {self.rank} holds {self.opt.n_rows} rows, shard is "
                             f"[{self.lo}, {self.hi})")
        opt = self.opt
        opt._nv_reduce = lambda count: global_visible_count(count, self.group)
        opt._abort_reduce = lambda flag: _all_reduce_(flag, dist.ReduceOp.MAX, self.group)
        dev = opt.device
        self._side = torch.cuda.Stream(dev) if not _host_collective(group) else None
        self._bufs = [torch.zeros_like(opt.engine.stats) for _ in range(self.STAT_SLOTS)]
        self._free = [None] * self.STAT_SLOTS  # event: the side stream is done with the slot
        self._slot = 0
        self._host = [(torch.zeros(L.GS_STEP_STATS, dtype=torch.float64, pin_memory=True),
                       torch.zeros(1, dtype=torch.int32, pin_memory=True))
                      for _ in range(self.STAT_SLOTS)]
        self._pending = collections.deque()
        self.stats = self._bufs[0]
        self.stats_event = None

    # ------------------------------------------------------------------- step
    def step(self, visibility_local: torch.Tensor, n_pixels=None, **kw) -> torch.Tensor:
        """One step of this shard (AdamWGS.step arguments); returns the device
        tensor of the step statistics summed over all ranks.  In the
        decoupled modes the sum runs on a side stream: :meth:`wait_stats`
        orders it before work on the current stream."""
        self._poll(block=self.errors == "raise" or
                   (self.opt.mode == "coupled-adam" and self.opt.check == "strict"))
        self.opt.step(visibility_local, n_pixels, **kw)
        return self._reduce_stats()

    def _reduce_stats(self) -> torch.Tensor:
        """Copy the shard's statistics into a slot on the compute stream and
        sum it over the ranks.  Decoupled modes: on the side stream, behind an
        event (the compute stream joins it only when the caller reads the
        result); the coupled modes already sit behind an all-reduce."""
        opt = self.opt
        dev = opt.device
        cur = torch.cuda.current_stream(dev)
        i = self._slot
        self._slot = (i + 1) % self.STAT_SLOTS
        buf = self._bufs[i]
        if self._free[i] is not None:
            cur.wait_event(self._free[i])  # the side stream's reduce of this slot is done
        buf.copy_(opt.engine.stats)
        if self._side is not None and opt.mode not in ("sparse-adam", "coupled-adam"):
            ready = torch.cuda.Event()
            ready.record(cur)
            self._side.wait_event(ready)
            with torch.cuda.stream(self._side):
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
                done = torch.cuda.Event()
                done.record(self._side)
            self._free[i] = done
            self.stats_event = done
        else:
            _all_reduce_(buf, dist.ReduceOp.SUM, self.group)
            self._free[i] = None
            self.stats_event = None
        self.stats = buf
        if self.errors != "ignore" and not torch.cuda.is_current_stream_capturing():
            self._enqueue_check(i)
        return buf

    def capture_begin(self):
        """Before an outside CUDA-graph capture of steps: nothing outstanding,
        no waits on events recorded outside the capture."""
        self.check_errors()
        torch.cuda.synchronize(self.opt.device)
        self._free = [None] * self.STAT_SLOTS
        self.stats_event = None

    def capture_end(self):
        """After the capture (whose last step joined the side stream with
        wait_stats()): events recorded inside it are not waited on outside."""
        self._free = [None] * self.STAT_SLOTS
        self.stats_event = None

    def wait_stats(self) -> torch.Tensor:
        """The last step's reduced statistics, ordered on the current stream."""
        if getattr(self, "stats_event", None) is not None:
            torch.cuda.current_stream(self.opt.device).wait_event(self.stats_event)
        return self.stats

    # ----------------------------------------------------------------- errors
    def _enqueue_check(self, i: int):
        if len(self._pending) >= self.STAT_SLOTS:
            self._poll(block=True, limit=1)
        opt = self.opt
        st_host, ab_host = self._host[i]
        s = self._side if self._free[i] is not None else torch.cuda.current_stream(opt.device)
        with torch.cuda.stream(s):
            st_host.copy_(self._bufs[i], non_blocking=True)
        strict = opt.check == "strict"
        cur = torch.cuda.current_stream(opt.device)
        if strict:  # the abort flag was max-reduced before the step
            ab_host.copy_(opt.engine.abort, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s)
        if s is not cur:
            ev2 = torch.cuda.Event()
            ev2.record(cur)
        else:
            ev2 = None
        self._pending.append((ev, ev2, st_host, ab_host if strict else None, opt._last_ctx))
        if self.errors == "raise":
            self._poll(block=True)

    def _poll(self, block: bool, limit: int | None = None):
        n = 0
        while self._pending and (limit is None or n < limit):
            ev, ev2 = self._pending[0][:2]
            if not block and not (ev.query() and (ev2 is None or ev2.query())):
                return
            _, _, st_host, ab_host, ctx = self._pending.popleft()
            ev.synchronize()
            if ev2 is not None:
                ev2.synchronize()
            n += 1
            self._raise_for(_stats_dict(st_host.tolist()),
                            int(ab_host.item()) if ab_host is not None else 0, ctx)

    def _raise_for(self, st: dict, flag: int, ctx):
        """Every rank sees the same reduced statistics and flag, so every
        rank takes this branch together; the ids are gathered globally."""
        opt = self.opt
        if self.n_global:  # the kernel-choice hints (global view)
            opt._vis_frac = st["n_visible"] / self.n_global
            if st.get("n_runs", 0) > 0:
                opt._vis_run = st["n_visible"] / st["n_runs"]
        if flag and opt.mode == "coupled-adam":
            opt.state.global_t -= 1  # aborted everywhere before any mutation
        bad_g = st["n_bad_grad"] > 0 or (flag & 1)
        bad_d = st["n_bad_domain"] > 0 or (flag & 2)
        if not (bad_g or bad_d):
            return
        self._pending.clear()
        b, rows, count, lo, ls, mode, vis = ctx
        if mode == "coupled-adam":
            rows, count = opt.engine.all_rows()
        elif rows is None:  # the fused step made no index list
            rows, count = opt.engine.compact(vis)
        g_ids, d_ids = opt.engine.bad_rows(b, rows, count, lo, ls)
        mine = (np.asarray(g_ids, np.int64) + self.lo, np.asarray(d_ids, np.int64) + self.lo)
        allv = [None] * self.world
        dist.all_gather_object(allv, mine, group=self.group)
        g_all = np.concatenate([a[0] for a in allv])
        d_all = np.concatenate([a[1] for a in allv])
        if bad_g:
            raise GradientError(g_all)
        raise DomainError("tau must be finite / log-scale above 80.0 would overflow", d_all)

    def check_errors(self):
        """Wait for the outstanding steps; raise a deferred error (all ranks)."""
        self._poll(block=True)

    # ------------------------------------------------------------- state ops
    def global_rows(self) -> torch.Tensor:
        """This shard's visible rows in global numbering (after a step)."""
        eng = self.opt.engine
        ctx = self.opt._last_ctx
        if ctx is not None and ctx[1] is None and ctx[-1] is not None:
            eng.compact(ctx[-1])  # the fused step made no index list
        c = int(eng.count.item())
        return eng.idx[:c].to(torch.int64) + self.lo

    def rsr_apply(self, global_indices, alpha1: float, alpha2: float):
        """RSR on the shared global sample (stss_sample on every rank), sliced."""
        local = shard_rows(np.asarray(global_indices, dtype=np.int64), self.lo, self.hi)
        self.opt.rsr_apply(local, alpha1, alpha2)

    def reset_rows(self, global_indices):
        local = shard_rows(np.asarray(global_indices, dtype=np.int64), self.lo, self.hi)
        self.opt.reset_rows(local)

    def aiu_apply(self, visibility_local: torch.Tensor, aiu, rng, iteration: int,
                  alive_local: torch.Tensor | None = None):
        """Sharded AIU (optimizer.py:425-450), picks bit-identical to one process.

        One all-gather of the per-rank invisible counts; every rank draws the
        global Bernoulli vector from the same stream and keeps its slice
        (sampling.aiu_shard_select). Returns this shard's picks in global
        numbering."""
        from .sampling import device_bernoulli

        def draw(n_local, prob):
            dev = self.opt.device if not _host_collective(self.group) else "cpu"
            mine = torch.tensor([n_local], dtype=torch.int64, device=dev)
            allc = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(allc, mine, group=self.group)
            counts = [int(c.item()) for c in allc]
            # this shard's slice of the global draw, on the device
            # (sampling.aiu_shard_select restated there)
            return device_bernoulli(rng, sum(counts), prob, sum(counts[:self.rank]), n_local,
                                    self.opt.device)

        picked = self.opt.aiu_apply(visibility_local, aiu, rng, iteration, alive_local, draw=draw)
        return np.asarray(picked, np.int64) + self.lo

    def capture(self, visibility_local: torch.Tensor, n_pixels=None, **kw) -> "ShardStepGraph":
        """Capture one shard step — compaction, the fused step, the statistics
        all-reduce (NCCL, on the side stream in the decoupled modes) — as a
        CUDA graph over static buffers (see AdamWGS.capture)."""
        if self.opt.mode == "coupled-adam":
            raise ConfigError("coupled-adam advances a host-side global clock; capture the "
                              "sparse modes")
        if _host_collective(self.group):
            raise ConfigError("graph capture of the sharded step needs the NCCL backend")
        return ShardStepGraph(self, visibility_local, n_pixels, kw)


class ShardStepGraph:
    """A captured ShardedAdamWGS.step (see ShardedAdamWGS.capture)."""

    def __init__(self, sh: ShardedAdamWGS, visibility, n_pixels, step_kwargs):
        self.sh = sh
        opt = sh.opt
        dev = opt.device
        opt.engine.group_array(opt._bindings(step_kwargs.get("grads"),
                                             step_kwargs.get("mu_lr_scale", 1.0)))
        cap = torch.cuda.Stream(dev)
        # the communicator must exist before capture (NCCL initialises lazily
        # on the first collective, which cannot happen inside a graph)
        dist.all_reduce(torch.zeros(1, dtype=torch.float64, device=dev), group=sh.group)
        sh.capture_begin()
        self.slot = sh._slot
        self.graph = torch.cuda.CUDAGraph()
        launches = opt.engine.launches
        opt._capturing = True
        try:
            with torch.cuda.stream(cap):
                with torch.cuda.graph(self.graph, stream=cap):
                    opt.step(visibility, n_pixels, **step_kwargs)
                    buf = sh._reduce_stats()
                    if sh.stats_event is not None:  # join the side stream inside the graph
                        torch.cuda.current_stream(dev).wait_event(sh.stats_event)
        finally:
            opt._capturing = False
        torch.cuda.current_stream(dev).wait_stream(cap)
        sh.capture_end()  # replays join the side stream inside the graph
        self.stats = buf
        self.launches_per_replay = opt.engine.launches - launches
        opt.engine.launches = launches

    def replay(self) -> torch.Tensor:
        sh = self.sh
        sh._poll(block=sh.errors == "raise")
        self.graph.replay()
        sh.opt.engine.launches += self.launches_per_replay
        sh.stats = self.stats
        if sh.errors != "ignore":
            sh._enqueue_check(self.slot)
        return self.stats
