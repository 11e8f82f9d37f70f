"""AdamW-GS optimizer: the reference's optimizer API over CUDA tensors.

Drop-in for the reference step family (/root/reference/pkg/src/splatlab/
optimizer.py) on the 3DGS parameter groups ``xyz / f_dc / f_rest / opacity /
scaling / rotation`` (or the reference's own ``mu / kappa / rot / tau /
color``).  Construction takes torch-style param groups, ``step()`` takes the
per-view visibility mask (or the rasterizer's int32 radii), and the state is
the reference's ``MomentState`` layout: per-group ``m`` and ``v`` shaped like
the parameters plus the per-primitive step clock.

All arithmetic runs in the sm_100a kernels behind ``include/adamw_gs.h``;
this module is host plumbing.  There is no CPU path.
"""

from __future__ import annotations

import collections
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import records as _records
from .records import base_grad_view
from .sampling import device_bernoulli
from .engine import (ConfigError, DomainError, GradientError, GroupBinding, StepEngine,
                     _stream_handle, round_pixel_count, row_stride)

MODES = ("coupled-adam", "sparse-adam", "adamw-const", "adamw-const-clip", "adamw-gs")
CHECKS = ("fused", "strict")
ERRORS = ("raise", "defer", "ignore")

# group name -> role (optimizer.py:217,259-263 key on mu / tau / kappa)
ROLE_BY_NAME = {
    "xyz": L.ROLE_POSITION, "mu": L.ROLE_POSITION, "means": L.ROLE_POSITION,
    "opacity": L.ROLE_OPACITY, "tau": L.ROLE_OPACITY, "opacities": L.ROLE_OPACITY,
    "scaling": L.ROLE_SCALE, "kappa": L.ROLE_SCALE, "scales": L.ROLE_SCALE,
}
ROLE_NAMES = {"plain": L.ROLE_PLAIN, "position": L.ROLE_POSITION, "opacity": L.ROLE_OPACITY,
              "scale": L.ROLE_SCALE}
# reference attribute <-> 3DGS group
SH3_ALIASES = {"xyz": "mu", "f_dc": "color", "opacity": "tau", "scaling": "kappa",
               "rotation": "rot"}


def role_of(name: str, role=None) -> int:
    if role is None:
        return ROLE_BY_NAME.get(name, L.ROLE_PLAIN)
    if isinstance(role, str):
        return ROLE_NAMES[role]
    return int(role)


@dataclass
class OptimizerConfig:
    """optimizer.py:70-100, plus learning rates for groups the reference lacks."""

    mode: str = "coupled-adam"
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    lr_mu: float = 0.029
    lr_tau: float = 0.05
    lr_kappa: float = 5e-3
    lr_rot: float = 1e-3
    lr_color: float = 2.5e-3
    lambda_o: float = 0.0
    lambda_s: float = 0.0
    ct_opacity: float = 10.0
    ct_scale: float = 10.0
    round_n_pixels: bool = True
    lr_extra: dict = field(default_factory=dict)

    def __post_init__(self):
        validate_hyper(self.mode, self.beta1, self.beta2, self.eps, self.ct_opacity, self.ct_scale)

    def lr(self, attr: str) -> float:
        if attr in self.lr_extra:
            return float(self.lr_extra[attr])
        name = SH3_ALIASES.get(attr, attr)
        if hasattr(self, f"lr_{name}"):
            return float(getattr(self, f"lr_{name}"))
        raise ConfigError(f"no learning rate for attribute group {attr!r}")


def validate_hyper(mode, beta1, beta2, eps, ct_opacity, ct_scale):
    if mode not in MODES:
        raise ConfigError(f"unknown mode {mode!r}; expected one of {MODES}")
    for name, b in (("beta1", beta1), ("beta2", beta2)):
        if not (0.0 <= b < 1.0):
            raise ConfigError(f"{name} must lie in [0, 1)")
    if not (eps > 0.0):
        raise ConfigError("eps must be positive")
    if not (ct_opacity > 0.0 and ct_scale > 0.0):
        raise ConfigError("clip bounds C_t must be positive")


def _tail_strides(tail: tuple) -> tuple:
    out, acc = [], 1
    for d in reversed(tail):
        out.append(acc)
        acc *= d
    return tuple(reversed(out))


class MomentState:
    """optimizer.py:103-156 — m, v per group (param-shaped) + the step clock.

    The reference keeps one int64 clock per group; every code path moves them
    together, so one int32 clock per primitive is stored
    and ``t[group]`` returns that shared tensor.

    Two storage layouts, same interface:

    ``"rows"`` (default) — one fp32 record per primitive holding the (m, v)
        pairs of all its elements in group order followed by the int32 clock
        (``record`` [N, >= 2*(P+1)], rows padded to ``row_align`` floats);
        ``m[g]``, ``v[g]`` and ``clock`` are strided views into it.  A visible
        primitive's whole optimizer state is one contiguous 8*(P+1)-byte span
        (480 B for SH-3, in a 512-B granule-aligned row by default), which is
        what the fused B200 step streams.
    ``"groups"`` — contiguous per-group ``m`` / ``v`` tensors and a separate
        int32 clock (the reference's own layout).
    """

    def __init__(self, m: dict, v: dict, clock: torch.Tensor, global_t: int = 0,
                 record: torch.Tensor | None = None, spec: tuple | None = None):
        self.m, self.v, self.clock = m, v, clock
        self.global_t = int(global_t)
        self.record = record
        self.spec = spec

    @property
    def layout(self) -> str:
        return "rows" if self.record is not None else "groups"

    @property
    def t(self) -> dict:
        return {k: self.clock for k in self.m}

    def __len__(self) -> int:
        return int(self.clock.numel())

    @staticmethod
    def _views(record: torch.Tensor, spec: tuple):
        n, stride, base = record.shape[0], record.stride(0), record.storage_offset()
        m, v = {}, {}
        for name, off, tail in spec:
            st = (stride,) + tuple(2 * x for x in _tail_strides(tail))
            m[name] = record.as_strided((n,) + tail, st, base + 2 * off)
            v[name] = record.as_strided((n,) + tail, st, base + 2 * off + 1)
        p = sum(int(np.prod(t)) for _, _, t in spec)
        clock = record.view(torch.int32).as_strided((n,), (stride,), base + 2 * p)
        return m, v, clock

    @staticmethod
    def from_record(record: torch.Tensor, spec: tuple, global_t: int = 0) -> "MomentState":
        m, v, clock = MomentState._views(record, spec)
        return MomentState(m, v, clock, global_t, record, spec)

    @staticmethod
    def zeros_like(params: dict, layout: str = "rows", row_align: int = 16) -> "MomentState":
        first = next(iter(params.values()))
        n = first.shape[0]
        if layout == "groups":
            return MomentState(
                m={k: torch.zeros(p.shape, dtype=torch.float32, device=p.device)
                   for k, p in params.items()},
                v={k: torch.zeros(p.shape, dtype=torch.float32, device=p.device)
                   for k, p in params.items()},
                clock=torch.zeros(n, dtype=torch.int32, device=first.device))
        if layout != "rows":
            raise ConfigError(f"unknown state layout {layout!r}")
        spec, off = [], 0
        for k, p in params.items():
            tail = tuple(p.shape[1:])
            spec.append((k, off, tail))
            off += int(np.prod(tail)) if tail else 1
        w = 2 * (off + 1)
        # rows padded to a multiple of row_align floats; 16 = whole 64-byte
        # DRAM granules (SH-3: 120 -> 128 floats, 512 B)
        a = max(2, int(row_align))
        w = (w + a - 1) // a * a
        record = torch.zeros((n, w), dtype=torch.float32, device=first.device)
        return MomentState.from_record(record, tuple(spec))

    def copy(self) -> "MomentState":
        if self.record is not None:
            return MomentState.from_record(self.record.clone(), self.spec, self.global_t)
        return MomentState({k: t.clone() for k, t in self.m.items()},
                           {k: t.clone() for k, t in self.v.items()}, self.clock.clone(),
                           self.global_t)

    def select(self, index) -> "MomentState":
        """Rows ``index`` (prune/clone bookkeeping, optimizer.py:141-147)."""
        if self.record is not None:
            return MomentState.from_record(self.record[index].contiguous(), self.spec,
                                           self.global_t)
        return MomentState({k: t[index].contiguous() for k, t in self.m.items()},
                           {k: t[index].contiguous() for k, t in self.v.items()},
                           self.clock[index].contiguous(), self.global_t)

    @staticmethod
    def concatenate(a: "MomentState", b: "MomentState") -> "MomentState":
        """optimizer.py:149-156."""
        if a.record is not None and b.record is not None:
            return MomentState.from_record(torch.cat([a.record, b.record]), a.spec, a.global_t)
        return MomentState({k: torch.cat([a.m[k], b.m[k]]) for k in a.m},
                           {k: torch.cat([a.v[k], b.v[k]]) for k in a.v},
                           torch.cat([a.clock, b.clock]), a.global_t)


def _stats_dict(arr) -> dict:
    vals = [float(x) for x in arr]
    out = {}
    for k, x in zip(L.STAT_FIELDS, vals):
        out[k] = x if k.startswith("sum_") else int(x)
    return out


class AdamWGS:
    """Fused sparse Adam + DAR + RSR optimizer over 3DGS parameter groups.

    ``params``: list of dicts ``{"params": [tensor], "lr": float, "name": str}``
    (optionally ``"role"``: plain / position / opacity / scale), one tensor per
    group, all with the same leading row count N, fp32, on one CUDA device;
    each row dense, either contiguous per attribute or attribute views of
    one row-interleaved record (records.py, the faster HBM layout).
    Gradients are read from ``tensor.grad``, from the record's ``.grad``
    for record views, or from the ``grads`` mapping passed to :meth:`step`.
    """

    ERROR_SLOTS = 4  # steps whose error check may be outstanding (errors="defer")

    def __init__(self, params, *, mode: str = "adamw-gs", betas=(0.9, 0.999), eps: float = 1e-8,
                 lambda_o: float = 0.0, lambda_s: float = 0.0, ct_opacity: float = 10.0,
                 ct_scale: float = 10.0, round_n_pixels: bool = True, check: str = "fused",
                 errors: str = "defer", state_layout: str = "rows",
                 state_row_align: int = 16, adopt="auto", fused_compaction: bool = True):
        validate_hyper(mode, betas[0], betas[1], eps, ct_opacity, ct_scale)
        if check not in CHECKS:
            raise ConfigError(f"check must be one of {CHECKS}")
        if errors not in ERRORS:
            raise ConfigError(f"errors must be one of {ERRORS}")
        self.mode = mode
        self.beta1, self.beta2 = float(betas[0]), float(betas[1])
        self.eps = float(eps)
        self.lambda_o, self.lambda_s = float(lambda_o), float(lambda_s)
        self.ct_opacity, self.ct_scale = float(ct_opacity), float(ct_scale)
        self.round_n_pixels = bool(round_n_pixels)
        self.check, self.errors = check, errors
        self.fused_compaction = bool(fused_compaction)

        self.param_groups = []
        for i, g in enumerate(params):
            ps = g["params"]
            ps = [ps] if isinstance(ps, torch.Tensor) else list(ps)
            if len(ps) != 1:
                raise ConfigError("each attribute group holds exactly one tensor")
            name = g.get("name", f"group{i}")
            self.param_groups.append({"params": ps, "lr": float(g["lr"]), "name": name,
                                      "role": role_of(name, g.get("role"))})
        if not self.param_groups:
            raise ConfigError("no parameter groups")
        first = self.param_groups[0]["params"][0]
        self.device = first.device
        self.n_rows = int(first.shape[0])
        for g in self.param_groups:
            p = g["params"][0]
            if p.device != self.device or p.shape[0] != self.n_rows:
                raise ConfigError(f"group {g['name']}: all groups must share device and row count")
            if p.dtype != torch.float32:
                raise ConfigError(f"group {g['name']}: parameters must be fp32")
            w = max(1, int(np.prod(p.shape[1:]))) if p.dim() > 1 else 1
            row_stride(f"group {g['name']}", p, self.n_rows, w)
        self.param_record = self.grad_record = None
        self._maybe_adopt(adopt)
        self.state_row_align = int(state_row_align)
        self.state = MomentState.zeros_like({g["name"]: g["params"][0] for g in self.param_groups},
                                            state_layout, self.state_row_align)
        self.engine = StepEngine(self.n_rows, self.device, self.beta1, self.beta2)
        # pinned slots for the asynchronous error check: a step copies its
        # statistics (and strict abort flag) into a slot and records an
        # event; the host inspects completed slots at the next step
        self._slots = [(torch.zeros(L.GS_STEP_STATS, dtype=torch.float64, pin_memory=True),
                        torch.zeros(1, dtype=torch.int32, pin_memory=True))
                       for _ in range(self.ERROR_SLOTS)]
        self._slot = 0
        self._slot_events = [torch.cuda.Event() for _ in range(self.ERROR_SLOTS)]
        self._dev_index = self.device.index if self.device.index is not None else \
            torch.cuda.current_device()
        self._pending = collections.deque()
        self._capturing = False
        self._last_ctx = None
        self._densify = None  # (accum, count, group index) when enabled
        # index-sharded hooks (sharded.ShardedAdamWGS): the global N_v from
        # the local count, and the all-shard abort flag of the strict check
        self._nv_reduce = None
        self._abort_reduce = None
        self._clock_bound = 0  # upper bound of every clock (and global_t): sizes the bias LUT
        self._vis_frac = None  # visible fraction of the last step whose statistics were read
        self._vis_run = None   # its mean run of consecutive visible rows (n_visible / n_runs)

    def _maybe_adopt(self, adopt):
        """Per-attribute leaf parameters -> one parameter record and one
        gradient record (records.adopt), see the class docstring."""
        if adopt is False or adopt is None:
            return
        if adopt not in (True, "auto"):
            raise ConfigError("adopt must be 'auto', True or False")
        ps = {g["name"]: g["params"][0] for g in self.param_groups}
        if len(ps) < 2 or _records.record_of(ps) is not None:
            return  # already views of one record
        if not all(p.is_leaf and p.is_contiguous() and p.device.type == "cuda" for p in ps.values()):
            if adopt is True:
                raise ConfigError("adopt=True needs contiguous leaf CUDA tensors")
            return
        if adopt == "auto" and not all(p.requires_grad for p in ps.values()):
            return
        self.param_record, self.grad_record = _records.adopt(ps)

    # ------------------------------------------------------------------ helpers
    def _bindings(self, grads=None, mu_lr_scale: float = 1.0) -> list[GroupBinding]:
        out = []
        for g in self.param_groups:
            p = g["params"][0]
            name = g["name"]
            gr = None
            if grads is not None:
                gr = grads[name]
            elif p.is_leaf and p.grad is not None:
                gr = p.grad
            else:  # attribute view of a leaf parameter record (records.py)
                gr = base_grad_view(p)
            lr = g["lr"] * (mu_lr_scale if g["role"] == L.ROLE_POSITION else 1.0)
            rows = self.state.record is not None
            out.append(GroupBinding(name, g["role"], lr, p, gr,  # kernels see pointers only
                                    None if rows else self.state.m[name],
                                    None if rows else self.state.v[name]))
        return out

    def _state_bindings(self) -> list[GroupBinding]:
        rows = self.state.record is not None
        return [GroupBinding(g["name"], g["role"], g["lr"], g["params"][0].data, None,
                             None if rows else self.state.m[g["name"]],
                             None if rows else self.state.v[g["name"]])
                for g in self.param_groups]

    # --------------------------------------------------------------------- step
    @torch.no_grad()
    def step(self, visibility: torch.Tensor | None = None, n_pixels: int | None = None, *,
             mu_lr_scale: float = 1.0, lambda_o: float | None = None,
             lambda_s: float | None = None, clip: float | None = None, grads=None,
             n_visible: torch.Tensor | None = None, densify_scale: float | None = None):
        """One optimizer step over the visible primitives.

        adamw-gs            dar_step (optimizer.py:269-298): ``n_pixels`` = N_I,
                            ``lambda_o`` / ``lambda_s`` override the configured
                            lambdas (the pipeline's DAR gating, pipeline.py:316-320).
        adamw-const[-clip]  adamw_const_step (optimizer.py:301-324); the clip
                            defaults to C_t(opacity) as the pipeline passes it.
        sparse-adam         sparse_adam_step with the pipeline's coupled
                            L1 gradients lambda*R'(theta)/N_v folded in
                            (pipeline.py:311-315); lambda 0 is plain Sparse Adam.
        coupled-adam        adam_step_sync over every row, coupled terms on
                            every row (pipeline.py:305-310).
        ``grads``: name -> gradient tensor, on the device or in pinned host
        memory; pinned host gradients are gathered zero-copy by the step
        kernel, so only the visible rows cross PCIe.
        ``n_visible``: device int32 [1] global N_v (index-sharded multi-GPU).
        ``densify_scale``: with :meth:`enable_densify_stats`, accumulate
        ||grad_position|| * densify_scale and a count per stepped row, fused
        into the step (DensifyStats.observe, pipeline.py:67-91).
        """
        # deferred checks of earlier steps: only those already complete,
        # except that a strict coupled-adam abort must roll back the clock
        # before the next step advances it
        self._poll(block=self.errors == "raise" or
                   (self.mode == "coupled-adam" and self.check == "strict"))
        mode = self.mode
        b = self._bindings(grads, mu_lr_scale)
        eng = self.engine
        self._clock_bound += 1
        eng.ensure_lut(self._clock_bound + 1)
        lo = self.lambda_o if lambda_o is None else float(lambda_o)
        ls = self.lambda_s if lambda_s is None else float(lambda_s)
        kw = dict(eps=self.eps, check=self.check, record=self.state.record)
        if densify_scale is not None:
            if self._densify is None:
                raise ConfigError("call enable_densify_stats() first")
            acc, cnt, gidx = self._densify
            kw["densify"] = (acc, cnt, float(densify_scale), gidx)
        if mode == "coupled-adam":
            self.state.global_t += 1
            nv = None
            listed = None
            regular = lo != 0.0 or ls != 0.0
            if (regular and n_visible is None) or "densify" in kw:
                if visibility is None:
                    raise ConfigError("coupled-adam regularization and densification statistics "
                                      "need the visibility mask")
                vrows, vcount = eng.compact(visibility)
                if "densify" in kw:
                    listed = (vrows, vcount)  # observe the visible rows only (pipeline.py:338-339)
                if regular:
                    nv = vcount if self._nv_reduce is None else self._nv_reduce(vcount)
            if regular and n_visible is not None:
                nv = n_visible
            stats = eng.step(b, mode, self.state.clock, rows=None, count=None,
                             lambda_opacity=lo, lambda_scale=ls, global_t=self.state.global_t,
                             n_visible_dev=nv, abort_hook=self._abort_reduce, densify_rows=listed,
                             **kw)
            rows = count = None
        else:
            if visibility is None:
                raise ConfigError(f"{mode} needs the visibility mask")
            stats = self._step_fused(b, mode, visibility, n_pixels, lo, ls, clip, kw, n_visible)
            if stats is not None:
                self._last_ctx = (b, None, None, lo, ls, mode, visibility)
                self._after_step(stats)
                return
            rows, count = eng.compact(visibility)
            kw["abort_hook"] = self._abort_reduce
            if mode == "adamw-gs":
                if n_pixels is None:
                    raise ConfigError("adamw-gs needs n_pixels (N_I)")
                n_i = round_pixel_count(int(n_pixels), self.round_n_pixels)
                stats = eng.step(b, mode, self.state.clock, rows=rows, count=count,
                                 lambda_opacity=lo, lambda_scale=ls, clip_opacity=self.ct_opacity,
                                 clip_scale=self.ct_scale, n_pixels_rounded=n_i, **kw)
            elif mode in ("adamw-const", "adamw-const-clip"):
                lo, ls = self.lambda_o, self.lambda_s
                c = clip if clip is not None else (self.ct_opacity if mode == "adamw-const-clip"
                                                   else None)
                m = "adamw-const-clip" if c is not None else "adamw-const"
                cv = float(c) if c is not None else 0.0
                stats = eng.step(b, m, self.state.clock, rows=rows, count=count,
                                 lambda_opacity=lo, lambda_scale=ls, clip_opacity=cv,
                                 clip_scale=cv, **kw)
            else:  # sparse-adam (+ coupled)
                nv = n_visible
                if nv is None:
                    nv = count if (self._nv_reduce is None or (lo == 0.0 and ls == 0.0)) \
                        else self._nv_reduce(count)
                stats = eng.step(b, mode, self.state.clock, rows=rows, count=count,
                                 lambda_opacity=lo, lambda_scale=ls, n_visible_dev=nv, **kw)
        self._last_ctx = (b, rows, count, lo, ls, mode, visibility)
        self._after_step(stats)

    def _fused_eligible(self, vis: torch.Tensor) -> bool:
        """Whether gs_step_rows_masked would take this mask (the check the
        library makes that the host can see: 16-byte alignment)."""
        return vis.data_ptr() % 16 == 0 and vis.is_contiguous()

    def _fused_small(self, vis: torch.Tensor) -> bool:
        """Clouds under 16 one-KB mask tiles per CTA slot (gs_step_sh3.cu):
        the library balances coherent masks there and counts a coupled
        sparse-adam step's N_v itself (the two-phase kernel)."""
        tile_rows = 256 if vis.dtype == torch.int32 else 1024
        return -(-self.n_rows // tile_rows) < 16 * 2 * L.load().gs_device_sm_count()

    def _step_fused(self, b, mode, visibility, n_pixels, lo, ls, clip, kw, n_visible=None):
        """K1 fused into K2 (engine.step_masked) where it applies; None otherwise."""
        if not self.fused_compaction or self.check != "fused" or self.state.record is None:
            return None
        eng = self.engine
        nv = None
        if not self._fused_eligible(visibility):
            return None
        small = self._fused_small(visibility)
        if mode == "sparse-adam" and (lo != 0.0 or ls != 0.0):
            # the coupled normaliser N_v (loss.py:190) before the step: the
            # caller's / all ranks' count, or the count pass; on small clouds
            # the two-phase kernel counts the mask itself
            nv = n_visible
            if nv is None and (self._nv_reduce is not None or not small):
                nv = eng.count_visible(visibility)
                if self._nv_reduce is not None:
                    nv = self._nv_reduce(nv)
        # the last known step (the deferred statistics; no synchronisation)
        # steers the choice: index-coherent visible rows (long runs) keep the
        # global index order of K1 + K2 on big clouds, which streams DRAM
        # better there (c3, 64-row blocks: 0.52 against 0.58 ms), and take
        # the balanced two-phase kernel on small ones (c1: 0.032 against
        # 0.039 ms streaming); sparse masks take the fused kernel's
        # bias-warp shape (c5 at 1%: 0.19 against 0.22 ms)
        coherent = self._vis_run is not None and self._vis_run >= 4.0
        if coherent and not small:
            return None
        low = self._vis_frac is not None and self._vis_frac < 0.05
        # masks >= 2 % visible: the last mask tiles are claimed dynamically
        # (c5 at 30%: 4.22 against 4.34 ms; at 1% the claims cost more)
        balance = self._vis_frac is not None and self._vis_frac >= 0.02
        kwm = dict(eps=self.eps, record=self.state.record, densify=kw.get("densify"),
                   low_visibility=low, coherent=coherent, balance_tail=balance)
        if mode == "adamw-gs":
            if n_pixels is None:
                raise ConfigError("adamw-gs needs n_pixels (N_I)")
            n_i = round_pixel_count(int(n_pixels), self.round_n_pixels)
            return eng.step_masked(b, mode, visibility, lambda_opacity=lo, lambda_scale=ls,
                                   clip_opacity=self.ct_opacity, clip_scale=self.ct_scale,
                                   n_pixels_rounded=n_i, **kwm)
        if mode in ("adamw-const", "adamw-const-clip"):
            c = clip if clip is not None else (self.ct_opacity if mode == "adamw-const-clip"
                                               else None)
            m = "adamw-const-clip" if c is not None else "adamw-const"
            cv = float(c) if c is not None else 0.0
            return eng.step_masked(b, m, visibility, lambda_opacity=self.lambda_o,
                                   lambda_scale=self.lambda_s, clip_opacity=cv, clip_scale=cv,
                                   **kwm)
        return eng.step_masked(b, mode, visibility, lambda_opacity=lo, lambda_scale=ls,
                               n_visible_dev=nv, **kwm)  # sparse Adam (+ coupled L1)

    # ---------------------------------------------------------------- errors
    def _after_step(self, stats: torch.Tensor):
        if self.errors == "ignore" or self._capturing:
            return  # (StepGraph.replay() enqueues the check after each replay)
        self._enqueue_check()

    def _enqueue_check(self):
        """Copy this step's statistics (and strict abort flag) into a pinned
        slot and record an event; no host synchronisation unless every slot
        is still outstanding (the host is ERROR_SLOTS steps ahead)."""
        if len(self._pending) >= self.ERROR_SLOTS:
            self._poll(block=True, limit=1)
        st_host, ab_host = self._slots[self._slot]
        # the slot's event is free: at most ERROR_SLOTS checks are pending
        ev = self._slot_events[self._slot]
        self._slot = (self._slot + 1) % self.ERROR_SLOTS
        strict = self.check == "strict"
        eng = self.engine
        # one small kernel stores the statistics (and the abort flag) into the
        # pinned slot through its mapped pointer (no copy-engine transfer)
        L.check(eng.lib.gs_mirror_to_host(eng.stats.data_ptr(), st_host.data_ptr(),
                                          eng.stats.numel() * 8,
                                          eng.abort.data_ptr() if strict else None,
                                          ab_host.data_ptr() if strict else None,
                                          4 if strict else 0, _stream_handle(self.device)),
                "gs_mirror_to_host")
        # the engine launched on the current stream of the optimizer's device
        if torch.cuda.current_device() == self._dev_index:
            ev.record()
        else:
            ev.record(torch.cuda.current_stream(self._dev_index))
        self._pending.append((ev, st_host, ab_host if strict else None, self._last_ctx))
        if self.errors == "raise":
            self._poll(block=True)

    def _poll(self, block: bool, limit: int | None = None):
        """Inspect the outstanding step checks in order; raise the first
        error.  ``block=False`` stops at the first step still running."""
        n = 0
        while self._pending and (limit is None or n < limit):
            ev = self._pending[0][0]
            if not block and not ev.query():
                return
            _, st_host, ab_host, ctx = self._pending.popleft()
            ev.synchronize()
            n += 1
            vals = st_host.tolist()
            flag = int(ab_host.item()) if ab_host is not None else 0
            if flag == 0 and vals[2] == 0.0 and vals[3] == 0.0:
                # no bad rows: only the layout hints (the common case, cheap)
                if self.n_rows:
                    self._vis_frac = vals[0] / self.n_rows
                if vals[10] > 0:
                    self._vis_run = vals[0] / vals[10]
                continue
            self._raise_for(_stats_dict(vals), flag, ctx)

    def _raise_pending(self):
        self._poll(block=True)

    # ------------------------------------------------------ structural ops
    def rebind(self, params: dict, state: "MomentState | None" = None):
        """Point the optimizer at new parameter tensors after a structural
        change (densification, pruning, a loaded checkpoint): ``params`` maps
        every group name to its new tensor, ``state`` holds their moments
        (fresh zeros when None).  The row count may change; the
        densification statistics, if enabled, restart from zero."""
        self._raise_pending()
        names = [g["name"] for g in self.param_groups]
        if set(params) != set(names):
            raise ConfigError(f"rebind needs exactly the groups {names}")
        n = int(params[names[0]].shape[0])
        for name in names:
            p = params[name]
            if p.device != self.device or p.dtype != torch.float32 or p.shape[0] != n:
                raise ConfigError(f"group {name}: fp32 on {self.device} with {n} rows expected")
            w = max(1, int(np.prod(p.shape[1:]))) if p.dim() > 1 else 1
            row_stride(f"group {name}", p, n, w)
        if state is None:
            layout = "rows" if self.state.record is not None else "groups"
            state = MomentState.zeros_like({k: params[k] for k in names}, layout,
                                           self.state_row_align)
        if len(state) != n:
            raise ConfigError(f"state has {len(state)} rows, parameters {n}")
        for g in self.param_groups:
            g["params"] = [params[g["name"]]]
        self.state = state
        if n:
            self._clock_bound = max(self._clock_bound, int(state.clock.max().item()),
                                    state.global_t)
        if n != self.n_rows:
            self.n_rows = n
            self.engine = StepEngine(n, self.device, self.beta1, self.beta2)
        self._last_ctx = None
        if self._densify is not None:
            self.enable_densify_stats(names[self._densify[2]])


    def relocate_rows(self, plan) -> None:
        """Apply a relocation plan (structural.RelocationPlan): respawn rows
        take their target's attributes, target and respawn share the planned
        opacity logit, respawn state is reset (pipeline.py:221-228)."""
        if plan.count == 0:
            return
        opac = [i for i, g in enumerate(self.param_groups) if g["role"] == L.ROLE_OPACITY]
        if len(opac) != 1:
            raise ConfigError("relocation needs exactly one opacity group")
        dev = self.device
        dead = torch.from_numpy(plan.dead.astype(np.int32)).to(dev)
        targets = torch.from_numpy(plan.targets.astype(np.int32)).to(dev)
        tau_new = torch.from_numpy(plan.tau_new.astype(np.float32)).to(dev)
        groups = self._state_bindings()
        if self.state.record is not None:
            self.engine.relocate(groups, self.state.record, opac[0], dead, targets, tau_new)
            return
        # per-group state layout: the row copies as device gathers, then K3 reset
        with torch.no_grad():
            for i, g in enumerate(self.param_groups):
                p = g["params"][0]
                if i == opac[0]:
                    col = p.reshape(p.shape[0], -1)[:, 0]
                    col[dead.long()] = tau_new
                    col[targets.long()] = tau_new
                else:
                    p[dead.long()] = p[targets.long()]
        self.reset_rows(dead)

    def densify_adc(self, cfg, rng: np.random.Generator, alive=None, iteration: int = 0):
        """densify_adc (pipeline.py:116-185) from the fused densification
        statistics; see structural.densify_adc.  Rebinds the optimizer to
        the new rows and returns the DensifyResult (new parameter tensors,
        alive mask, source row per output row, the reference's events)."""
        from .structural import densify_adc
        acc, cnt = self.densify_stats()
        return densify_adc(self, acc, cnt, cfg, rng, alive, iteration)

    def mcmc_relocate(self, rng: np.random.Generator, alive=None):
        """mcmc_relocate (pipeline.py:197-233): plan on the host with the
        caller's Generator (targets identical to the reference's), move rows
        on the GPU. Returns the RelocationPlan (``count``, ``ids_hash()``
        match the reference's relocate event)."""
        from .structural import mcmc_plan
        opac = [g for g in self.param_groups if g["role"] == L.ROLE_OPACITY]
        if len(opac) != 1:
            raise ConfigError("relocation needs exactly one opacity group")
        tau = opac[0]["params"][0].detach().reshape(-1).cpu().numpy()
        if alive is not None and isinstance(alive, torch.Tensor):
            alive = alive.detach().cpu().numpy()
        plan = mcmc_plan(tau, alive, rng)
        self.relocate_rows(plan)
        return plan

    # ------------------------------------------------------------ CUDA graphs
    def capture(self, visibility: torch.Tensor, n_pixels: int | None = None, *,
                grads=None, **step_kwargs) -> "StepGraph":
        """Capture one :meth:`step` (compaction + fused step, statistics copy)
        as a CUDA graph over static buffers, for clouds small enough that host
        launch latency rivals the GPU work.  Refill ``visibility`` and the
        gradient tensors in place, then call ``StepGraph.replay()``; scalars
        (n_pixels, lambdas, clip, lr scale) are fixed at capture — capture
        again when they change.  Errors surface after each replay as
        configured (``errors="raise"`` synchronises, ``"defer"`` raises at
        the next step / :meth:`check_errors`).  The dense coupled-adam mode
        keeps a host-side global clock and is not capturable."""
        if self.mode == "coupled-adam":
            raise ConfigError("coupled-adam advances a host-side global clock; capture the "
                              "sparse modes")
        # replays advance the clocks without the host: the captured bias
        # table must be exact for every clock
        self.engine.ensure_lut(self.engine.lut_exact_len)
        return StepGraph(self, visibility, n_pixels, grads, step_kwargs)

    def _note_layout(self, st: dict):
        """Remember the visible fraction and run length of a finished step."""
        if self.n_rows:
            self._vis_frac = st["n_visible"] / self.n_rows
        if st.get("n_runs", 0) > 0:
            self._vis_run = st["n_visible"] / st["n_runs"]

    def _raise_for(self, st: dict, flag: int, ctx):
        self._note_layout(st)
        if flag and self.mode == "coupled-adam":
            # the strict check aborted the step before any mutation: the
            # reference checks before advancing the clock (optimizer.py:225-226)
            self.state.global_t -= 1
        bad_g = st["n_bad_grad"] > 0 or (flag & 1)
        bad_d = st["n_bad_domain"] > 0 or (flag & 2)
        if not (bad_g or bad_d):
            return
        self._pending.clear()  # later steps' checks are superseded by this error
        b, rows, count, lo, ls, mode, vis = ctx
        if mode == "coupled-adam":
            rows, count = self.engine.all_rows()
        elif rows is None:  # the fused step made no index list
            rows, count = self.engine.compact(vis)
        # ids from the failing step's gradient bindings (deferred: the caller
        # keeps those buffers until the error surfaces, or uses errors="raise")
        g_ids, d_ids = self.engine.bad_rows(b, rows, count, lo, ls)
        if bad_g:
            raise GradientError(g_ids)
        raise DomainError("tau must be finite / log-scale above 80.0 would overflow", d_ids)

    def check_errors(self):
        """Wait for the outstanding steps and raise a deferred GradientError /
        DomainError, if any."""
        self._poll(block=True)

    def last_stats(self) -> dict:
        """Per-step statistics of the last step (host sync)."""
        st = _stats_dict(self.engine.stats.tolist())
        if self.engine.launches:  # zeros before the first step are no layout hint
            self._note_layout(st)
        return st

    # ----------------------------------------------- densification statistics
    def enable_densify_stats(self, group: str | None = None):
        """Allocate the per-row gradient-norm accumulator and count
        (DensifyStats, pipeline.py:67-91) for the position group (or ``group``)."""
        names = [g["name"] for g in self.param_groups]
        if group is None:
            pos = [g["name"] for g in self.param_groups if g["role"] == L.ROLE_POSITION]
            if not pos:
                raise ConfigError("no position group; pass group=")
            group = pos[0]
        gidx = names.index(group)
        acc = torch.zeros(self.n_rows, dtype=torch.float32, device=self.device)
        cnt = torch.zeros(self.n_rows, dtype=torch.int32, device=self.device)
        self._densify = (acc, cnt, gidx)

    def densify_stats(self):
        """(accum, count) device tensors; mean = accum / max(count, 1)."""
        if self._densify is None:
            raise ConfigError("densification statistics are not enabled")
        return self._densify[0], self._densify[1]

    def reset_densify_stats(self):
        if self._densify is not None:
            self._densify[0].zero_()
            self._densify[1].zero_()

    # ----------------------------------------------------------- state ops
    @torch.no_grad()
    def rsr_apply(self, indices, alpha1: float, alpha2: float):
        """Re-State Regularization (optimizer.py:327-340): m*=a1, v*=a2, clock kept."""
        self.engine.rsr_apply(self._state_bindings(), indices, alpha1, alpha2,
                              record=self.state.record)

    @torch.no_grad()
    def reset_rows(self, indices):
        """Fresh state on the rows (optimizer.py:159-165): m = v = 0, t = 0."""
        self.engine.reset_rows(self._state_bindings(), self.state.clock, indices,
                               record=self.state.record)

    @torch.no_grad()
    def aiu_apply(self, visibility: torch.Tensor, aiu, rng: np.random.Generator, iteration: int,
                  alive: torch.Tensor | None = None, draw=None) -> np.ndarray:
        """Artificial implicit updates (optimizer.py:425-450).

        The invisible alive rows are compacted on the GPU; the Bernoulli picks
        ``rng.random(invisible.size) < prob`` are drawn on the GPU from the
        reference's Philox stream, bit for bit, and ``rng`` advances as the
        host draw would (sampling.device_bernoulli), so the picked set is
        bit-identical; the frozen-moment update runs on the GPU.  Returns the
        picked rows (int64, ascending).  ``draw(n_invisible, prob)`` replaces
        the local draw (the index-sharded wrapper's global-stream slice).
        """
        empty = np.empty(0, dtype=np.int64)
        if not aiu.active(iteration):
            return empty
        if self.state.record is None:
            raise ConfigError("aiu_apply needs the row-record state layout")
        prob, eta = aiu.prob_at(iteration), aiu.eta_at(iteration)
        eng = self.engine
        vis = visibility if visibility.dtype in (torch.bool, torch.uint8) else visibility > 0
        inv_idx, inv_cnt = eng.compact_select(vis, alive, invert=True)
        n_inv = int(inv_cnt.item())
        if draw is not None:  # collective draw: every shard takes part, even an empty one
            if prob <= 0.0 or eta == 0.0:
                return empty
            jmask = draw(n_inv, prob)
        else:
            if n_inv == 0 or prob <= 0.0 or eta == 0.0:
                return empty
            # rng.random(n_inv) < prob, drawn on the device bit for bit
            # (sampling.device_bernoulli: the reference's Philox stream)
            jmask = device_bernoulli(rng, n_inv, prob, 0, n_inv, self.device)
        if not isinstance(jmask, torch.Tensor):
            jmask = torch.from_numpy(np.asarray(jmask, bool).view(np.uint8)).to(self.device)
        if n_inv == 0:
            return empty
        # positions of the picks inside the invisible list (bit-exact order)
        jlist, jcnt = eng.compact_positions(jmask)
        k = int(jcnt.item())
        if k == 0:
            return empty
        picked = eng.aiu(self._state_bindings(), self.state.record, inv_idx, jlist, jcnt, k, eta,
                         self.eps)
        return picked.cpu().numpy().astype(np.int64)

    @torch.no_grad()
    def noise_perturb(self, lr_position: float, cfg, seed: int, iteration: int,
                      alive: torch.Tensor | None = None, add: bool = True) -> torch.Tensor:
        """Opacity-gated position noise (optimizer.py:453-486) over the
        position / scale / rotation / opacity groups; added in place by default
        (pipeline.py:334-336)."""
        from .noise import noise_perturb
        by_role = {g["role"]: g["params"][0] for g in self.param_groups}
        rot = [g["params"][0] for g in self.param_groups if g["name"] in ("rotation", "rot")]
        if L.ROLE_POSITION not in by_role or L.ROLE_SCALE not in by_role or \
                L.ROLE_OPACITY not in by_role or not rot:
            raise ConfigError("noise needs position, scaling, rotation and opacity groups")
        return noise_perturb(by_role[L.ROLE_POSITION].data, by_role[L.ROLE_SCALE].data,
                             rot[0].data, by_role[L.ROLE_OPACITY].data, lr_position, cfg, seed,
                             iteration, alive=alive, add=add)

    @torch.no_grad()
    def moment_stats(self, alive: torch.Tensor | None = None) -> dict:
        """optimizer.py:489-506 over alive rows."""
        return _moment_stats(self.engine, self._state_bindings(), alive, self.state.record)

    @torch.no_grad()
    def classify_active(self, alive: torch.Tensor | None = None) -> tuple[int, int]:
        """(N_a, N_d) of primitives.py:228-238 (opacity group)."""
        out = self.engine.stats_all(self._state_bindings(), alive, self.state.record).tolist()
        return int(out[1]), int(out[0]) - int(out[1])

    def moment_state(self) -> MomentState:
        return self.state

    def zero_grad(self, set_to_none: bool = True):
        """Gradients that are views of a gradient record (``records.adopt``)
        are zeroed in place even with ``set_to_none``: dropping them would
        detach the parameters from the record layout."""
        bases = set()
        for g in self.param_groups:
            p = g["params"][0]
            if p.grad is not None:
                base = p.grad._base
                if base is not None and p.grad.dim() >= 1 and p.grad.stride(0) > math.prod(p.shape[1:]):
                    if id(base) not in bases:
                        bases.add(id(base))
                        base.zero_()
                elif set_to_none:
                    p.grad = None
                else:
                    p.grad.zero_()

    def state_dict(self) -> dict:
        """Optimizer-state checkpoint (the reference persists none)."""
        return {"format": "adamw-gs-b200/1", "mode": self.mode, "global_t": self.state.global_t,
                "clock": self.state.clock.detach().cpu(),
                "m": {k: t.detach().cpu() for k, t in self.state.m.items()},
                "v": {k: t.detach().cpu() for k, t in self.state.v.items()},
                "hyper": {"betas": (self.beta1, self.beta2), "eps": self.eps,
                          "lambda_o": self.lambda_o, "lambda_s": self.lambda_s,
                          "ct_opacity": self.ct_opacity, "ct_scale": self.ct_scale,
                          "lr": {g["name"]: g["lr"] for g in self.param_groups}}}

    def load_state_dict(self, sd: dict):
        if sd.get("format") != "adamw-gs-b200/1":
            raise ConfigError("unknown optimizer-state format")
        with torch.no_grad():
            self.state.clock.copy_(sd["clock"])
            for k in self.state.m:
                self.state.m[k].copy_(sd["m"][k])
                self.state.v[k].copy_(sd["v"][k])
        # (views into the row record are written in place)
        self.state.global_t = int(sd["global_t"])
        clock = sd["clock"]
        self._clock_bound = max(int(clock.max()) if clock.numel() else 0, self.state.global_t)


def _moment_stats(engine: StepEngine, bindings, alive, record=None) -> dict:
    out = engine.stats_all(bindings, alive, record).tolist()
    n_alive = out[0]
    res = {}
    for i, b in enumerate(bindings):
        s_sq, m_sq, n_pos, s_rt, m_rt = out[2 + 5 * i: 7 + 5 * i]
        cnt = n_alive * b.width
        res[b.name] = {
            "mean_sqrt_v": s_sq / cnt if cnt else 0.0,
            "max_sqrt_v": m_sq if cnt else 0.0,
            "mean_abs_m_over_sqrt_v": s_rt / n_pos if n_pos else 0.0,
            "max_abs_m_over_sqrt_v": m_rt if n_pos else 0.0,
        }
    return res


class StepGraph:
    """A captured :meth:`AdamWGS.step` (see :meth:`AdamWGS.capture`)."""

    def __init__(self, opt: AdamWGS, visibility: torch.Tensor, n_pixels, grads, step_kwargs):
        self.opt = opt
        self.visibility = visibility
        self.grads = grads
        opt._raise_pending()
        dev = opt.device
        # host-side caches (ctypes group array, lazily allocated scratch) are
        # built outside the capture: one binding pass, no kernel launches
        opt.engine.group_array(opt._bindings(grads, step_kwargs.get("mu_lr_scale", 1.0)))
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        launches = opt.engine.launches
        opt._capturing = True
        try:
            with torch.cuda.stream(side):
                with torch.cuda.graph(self.graph, stream=side):
                    opt.step(visibility, n_pixels, grads=grads, **step_kwargs)
        finally:
            opt._capturing = False
        torch.cuda.current_stream(dev).wait_stream(side)
        self.launches_per_replay = opt.engine.launches - launches
        opt.engine.launches = launches

    def replay(self):
        """One optimizer step on the current contents of the static buffers."""
        opt = self.opt
        opt._poll(block=opt.errors == "raise")
        self.graph.replay()
        opt.engine.launches += self.launches_per_replay
        if opt.errors != "ignore":
            opt._enqueue_check()

