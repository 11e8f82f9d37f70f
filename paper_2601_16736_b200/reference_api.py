"""Reference-signature entry points over CUDA tensors.

Same names, arguments, return values and error behaviour as the reference
functions in /root/reference/pkg/src/splatlab/optimizer.py, so a
``run_training``-style loop (pipeline.py:300-370) or the reference's own
tests drive the B200 path unchanged:

    dar_step(state, pset, grads, vis, cfg, n_pixels, mu_lr_scale=1.0,
             lambda_o=None, lambda_s=None) -> (pset, state)          # :269-298
    sparse_adam_step(state, pset, grads, vis, cfg, mu_lr_scale=1.0)  # :231-238
    adamw_const_step(state, pset, grads, vis, cfg, clip=None,
                     mu_lr_scale=1.0)                                 # :301-324
    adam_step_sync(state, pset, grads, cfg, mu_lr_scale=1.0)          # :222-228
    rsr_apply(state, indices, alpha1, alpha2) -> state                # :327-340
    reset_rows(state, indices) -> state                               # :159-165
    moment_stats(state, alive) -> dict                                # :489-506
    classify_active(pset, threshold=1/255) -> (n_active, n_dead, None) # primitives.py:228-238

``state`` is a :class:`MomentState` (m, v dicts of CUDA tensors + one
clock); ``pset`` any object with one CUDA tensor attribute per group;
``grads`` a mapping / object with the same groups; the attribute groups are
the keys of ``state.m`` in order.  Errors raise immediately as in the
reference: ``GradientError`` aborts before any mutation (strict check) and
``DomainError`` for tau / kappa outside the activation domain.

Extension over the reference signatures: ``sparse_adam_step`` and
``adam_step_sync`` accept ``coupled=(lambda_o, lambda_s)`` to fold the
pipeline's ``coupled_reg_grad`` (loss.py:177-198) into the same kernel.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .engine import (ConfigError, DomainError, GradientError, GroupBinding, StepEngine,
                     round_pixel_count)
from .optimizer import MomentState, OptimizerConfig, _moment_stats, role_of
from .noise import NoiseConfig, seed_from_generator
from .noise import noise_perturb as _noise_perturb
from .sampling import AiuConfig, RsrConfig, StSSchedule, stss_sample

__all__ = ["noise_perturb", "aiu_apply", "NoiseConfig", "AiuConfig", "MODES", "ConfigError", "GradientError", "DomainError", "OptimizerConfig",
           "MomentState", "StSSchedule", "RsrConfig", "round_pixel_count", "adam_step_sync",
           "sparse_adam_step", "dar_step", "adamw_const_step", "rsr_apply", "stss_sample",
           "reset_rows", "moment_stats", "classify_active"]

MODES = ("coupled-adam", "sparse-adam", "adamw-const", "adamw-const-clip", "adamw-gs")

_ENGINES: dict = {}


def _engine(n_rows: int, device, beta1: float, beta2: float) -> StepEngine:
    key = (str(device), int(n_rows), float(beta1), float(beta2))
    eng = _ENGINES.get(key)
    if eng is None:
        if len(_ENGINES) >= 8:
            _ENGINES.pop(next(iter(_ENGINES)))
        eng = StepEngine(n_rows, device, beta1, beta2)
        _ENGINES[key] = eng
    return eng


def _cover_clocks(eng: StepEngine, state: MomentState, ahead: int) -> None:
    """Size the engine's bias LUT for the state's clocks (this shim is
    synchronous anyway; the caller owns the state and may edit it)."""
    t = int(state.clock.max().item()) if len(state) else 0
    eng.ensure_lut(max(t, state.global_t) + ahead + 1)


def _get(obj, name):
    return obj[name] if isinstance(obj, dict) else getattr(obj, name)


def _bindings(state: MomentState, pset, grads, cfg: OptimizerConfig, mu_lr_scale: float):
    out = []
    rows = state.record is not None
    for name in state.m:
        role = role_of(name)
        lr = cfg.lr(name) * (mu_lr_scale if role == L.ROLE_POSITION else 1.0)
        p = _get(pset, name)
        g = None if grads is None else _get(grads, name)
        out.append(GroupBinding(name, role, lr, p, g, None if rows else state.m[name],
                                None if rows else state.v[name]))
    return out


def _as_mask(vis, n: int, device) -> torch.Tensor:
    if isinstance(vis, torch.Tensor):
        v = vis.to(device)
    else:
        v = torch.from_numpy(np.ascontiguousarray(np.asarray(vis, dtype=bool))).to(device)
    if v.dtype not in (torch.bool, torch.uint8, torch.int32):
        v = v.to(torch.bool)
    return v.contiguous()


def _run(mode, state, pset, grads, vis, cfg, *, mu_lr_scale=1.0, lam_o=0.0, lam_s=0.0,
         clip_o=10.0, clip_s=10.0, n_i=0.0, coupled=False):
    n = len(state)
    dev = state.clock.device
    eng = _engine(n, dev, cfg.beta1, cfg.beta2)
    b = _bindings(state, pset, grads, cfg, mu_lr_scale)
    _cover_clocks(eng, state, 1)
    if mode == "coupled-adam":
        rows = count = None
        nv = None
        if coupled and (lam_o != 0.0 or lam_s != 0.0):
            _, nv = eng.compact(_as_mask(vis, n, dev))
        state.global_t += 1
        stats = eng.step(b, mode, state.clock, rows=None, count=None, eps=cfg.eps,
                         lambda_opacity=lam_o, lambda_scale=lam_s, global_t=state.global_t,
                         n_visible_dev=nv, check="strict", record=state.record)
        drows, dcount = eng.all_rows()
    else:
        rows, count = eng.compact(_as_mask(vis, n, dev))
        stats = eng.step(b, mode, state.clock, rows=rows, count=count, eps=cfg.eps,
                         lambda_opacity=lam_o, lambda_scale=lam_s, clip_opacity=clip_o,
                         clip_scale=clip_s, n_pixels_rounded=n_i,
                         n_visible_dev=count if coupled else None, check="strict",
                         record=state.record)
        drows, dcount = rows, count
    flag = int(eng.abort.item())                      # reference semantics: raise now
    if flag:
        if mode == "coupled-adam":
            state.global_t -= 1                       # aborted before mutation
        g_ids, d_ids = eng.bad_rows(b, drows, dcount, lam_o, lam_s)
        if flag & 1:
            raise GradientError(g_ids)
        raise DomainError("tau must be finite / log-scale above 80.0 would overflow", d_ids)
    return stats


def adam_step_sync(state, pset, grads, cfg, mu_lr_scale=1.0, *, vis=None, coupled=None):
    """optimizer.py:222-228 (dense; ``coupled`` folds loss.py:177-198 with apply_to_all)."""
    lo, ls = coupled if coupled is not None else (0.0, 0.0)
    _run("coupled-adam", state, pset, grads, vis, cfg, mu_lr_scale=mu_lr_scale, lam_o=lo,
         lam_s=ls, coupled=coupled is not None)
    return pset, state


def sparse_adam_step(state, pset, grads, vis, cfg, mu_lr_scale=1.0, *, coupled=None):
    """optimizer.py:231-238."""
    lo, ls = coupled if coupled is not None else (0.0, 0.0)
    _run("sparse-adam", state, pset, grads, vis, cfg, mu_lr_scale=mu_lr_scale, lam_o=lo,
         lam_s=ls, coupled=coupled is not None)
    return pset, state


def dar_step(state, pset, grads, vis, cfg, n_pixels, mu_lr_scale=1.0, lambda_o=None,
             lambda_s=None):
    """optimizer.py:269-298."""
    lo = cfg.lambda_o if lambda_o is None else lambda_o
    ls = cfg.lambda_s if lambda_s is None else lambda_s
    if cfg.ct_opacity <= 0.0 or cfg.ct_scale <= 0.0:
        raise ConfigError("clip bounds C_t must be positive")
    n_i = round_pixel_count(n_pixels, cfg.round_n_pixels)
    _run("adamw-gs", state, pset, grads, vis, cfg, mu_lr_scale=mu_lr_scale, lam_o=lo, lam_s=ls,
         clip_o=cfg.ct_opacity, clip_s=cfg.ct_scale, n_i=n_i)
    return pset, state


def adamw_const_step(state, pset, grads, vis, cfg, clip=None, mu_lr_scale=1.0):
    """optimizer.py:301-324."""
    mode = "adamw-const" if clip is None else "adamw-const-clip"
    c = 0.0 if clip is None else float(clip)
    _run(mode, state, pset, grads, vis, cfg, mu_lr_scale=mu_lr_scale, lam_o=cfg.lambda_o,
         lam_s=cfg.lambda_s, clip_o=c, clip_s=c)
    return pset, state


def _state_bindings(state: MomentState, pset=None):
    rows = state.record is not None
    out = []
    for k in state.m:
        p = None
        if pset is not None:
            p = _get(pset, k)
        w = max(1, int(np.prod(state.m[k].shape[1:]))) if state.m[k].dim() > 1 else 1
        out.append(GroupBinding(k, role_of(k), 0.0, p, None, None if rows else state.m[k],
                                None if rows else state.v[k], w))
    return out


def rsr_apply(state: MomentState, indices, alpha1: float, alpha2: float) -> MomentState:
    """optimizer.py:327-340."""
    if not (0.0 <= alpha1 < 1.0 and 0.0 <= alpha2 < 1.0):
        raise ConfigError("RSR factors must lie in [0, 1)")
    eng = _engine(len(state), state.clock.device, 0.9, 0.999)
    eng.rsr_apply(_state_bindings(state), indices, alpha1, alpha2, record=state.record)
    return state


def reset_rows(state: MomentState, indices) -> MomentState:
    """optimizer.py:159-165."""
    eng = _engine(len(state), state.clock.device, 0.9, 0.999)
    eng.reset_rows(_state_bindings(state), state.clock, indices, record=state.record)
    return state


def moment_stats(state: MomentState, alive=None) -> dict:
    """optimizer.py:489-506."""
    eng = _engine(len(state), state.clock.device, 0.9, 0.999)
    if alive is not None and not isinstance(alive, torch.Tensor):
        alive = torch.from_numpy(np.asarray(alive, dtype=bool)).to(state.clock.device)
    return _moment_stats(eng, _state_bindings(state), alive, state.record)


def classify_active(pset, threshold: float = 1.0 / 255.0, alive=None):
    """primitives.py:228-238 — counts only (the mask is not materialised)."""
    if threshold != 1.0 / 255.0:
        raise ConfigError("only the reference threshold 1/255 is compiled in")
    tau = _get(pset, "tau") if hasattr(pset, "tau") or isinstance(pset, dict) and "tau" in pset \
        else _get(pset, "opacity")
    tau = tau.reshape(-1, 1).contiguous()
    n = tau.shape[0]
    eng = _engine(n, tau.device, 0.9, 0.999)
    # counts only: the per-group moment sums computed alongside are ignored
    b = [GroupBinding("tau", L.ROLE_OPACITY, 0.0, tau, None, tau, tau)]
    if alive is None:
        alive = getattr(pset, "alive", None)
    if alive is not None and not isinstance(alive, torch.Tensor):
        alive = torch.from_numpy(np.asarray(alive, dtype=bool)).to(tau.device)
    out = eng.stats_all(b, alive).tolist()
    return int(out[1]), int(out[0]) - int(out[1]), None


def noise_perturb(pset, state, lr_position: float, cfg, rng) -> torch.Tensor:
    """optimizer.py:463-486 — the additive position perturbation of every alive
    row (the caller adds it, pipeline.py:335).  ``pset`` holds ``mu``, ``kappa``,
    ``rot`` (2-D) or ``xyz``, ``scaling``, ``rotation`` (3DGS) and the opacity
    logit ``tau`` / ``opacity``; ``rng`` seeds the on-device Philox stream."""
    def pick(*names):
        for nm in names:
            if (isinstance(pset, dict) and nm in pset) or hasattr(pset, nm):
                return _get(pset, nm)
        raise ConfigError(f"primitive set lacks {names}")
    pos = pick("mu", "xyz")
    alive = pset.get("alive") if isinstance(pset, dict) else getattr(pset, "alive", None)
    if alive is not None and not isinstance(alive, torch.Tensor):
        alive = torch.from_numpy(np.asarray(alive, dtype=bool)).to(pos.device)
    return _noise_perturb(pos, pick("kappa", "scaling"), pick("rot", "rotation"),
                          pick("tau", "opacity"), lr_position, cfg, seed_from_generator(rng), 0,
                          alive=alive)


def aiu_apply(state, pset, vis, cfg, aiu, rng, iteration: int, alive=None) -> np.ndarray:
    """optimizer.py:425-450 over a row-record MomentState (picked rows bit-exact)."""
    from .optimizer import AdamWGS  # noqa: F401  (engine plumbing below)
    if state.record is None:
        raise ConfigError("aiu_apply needs the row-record state layout")
    if not aiu.active(iteration):
        return np.empty(0, dtype=np.int64)
    n = len(state)
    eng = _engine(n, state.clock.device, cfg.beta1, cfg.beta2)
    vis_t = _as_mask(vis, n, state.clock.device)
    if vis_t.dtype == torch.int32:
        vis_t = vis_t > 0
    if alive is None:
        alive = getattr(pset, "alive", None) if not isinstance(pset, dict) else pset.get("alive")
    if alive is not None and not isinstance(alive, torch.Tensor):
        alive = torch.from_numpy(np.asarray(alive, dtype=bool)).to(state.clock.device)
    prob, eta = aiu.prob_at(iteration), aiu.eta_at(iteration)
    _cover_clocks(eng, state, 0)
    inv_idx, inv_cnt = eng.compact_select(vis_t, alive, invert=True)
    n_inv = int(inv_cnt.item())
    if n_inv == 0 or prob <= 0.0 or eta == 0.0:
        return np.empty(0, dtype=np.int64)
    from .sampling import device_bernoulli
    sel = device_bernoulli(rng, n_inv, prob, 0, n_inv, inv_idx.device)  # rng.random(n) < prob
    jlist, jcnt = eng.compact_positions(sel)
    k = int(jcnt.item())
    if k == 0:
        return np.empty(0, dtype=np.int64)
    groups = [GroupBinding(k_, role_of(k_), cfg.lr(k_), _get(pset, k_), None, None, None)
              for k_ in state.m]
    picked = eng.aiu(groups, state.record, inv_idx, jlist, jcnt, k, eta, cfg.eps)
    return picked.cpu().numpy().astype(np.int64)
