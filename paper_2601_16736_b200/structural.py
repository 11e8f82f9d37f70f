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

Transcription note: ``_ids_hash`` / ``_event`` (pipeline.py:94-102) and the
split-child sampling (pipeline.py:153-162) follow the reference line for
line: identical rng draw order and event hashes are what make the
densification and relocation results bit-exact against reference runs.
The device side (record gathers, gs_relocate_rows) and the 3-D split are new.
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


# --------------------------------------------------------------------------
# Adaptive density control (vanilla 3DGS densification), pipeline.py:116-185
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class DensifyConfig:
    """The densify_adc fields of DensifyConfig (config.py:60-77)."""

    grad_threshold: float = 0.012
    prune_opacity: float = 0.005
    split_scale_px: float = 3.0  # clone at or below, split above
    split_shrink: float = 1.6
    max_primitives: int = 2000


@dataclass
class DensifyResult:
    params: dict            # name -> new parameter tensor (the optimizer is rebound to them)
    alive: np.ndarray       # bool per output row
    src: np.ndarray         # int64 source row of each output row (children -> parent)
    events: list            # the reference's event dicts (kind, count, affected_ids_hash)


def _ids_hash(ids) -> str:
    data = np.sort(np.asarray(ids, dtype=np.int64)).tobytes()
    return hashlib.blake2b(data, digest_size=8).hexdigest()


def _event(iteration: int, kind: str, ids) -> dict:
    ids = np.asarray(ids)
    return {"iter": int(iteration), "kind": kind, "count": int(ids.size),
            "affected_ids_hash": _ids_hash(ids)}


def _logit_checked(o: np.ndarray) -> np.ndarray:
    if np.any(o <= 0.0) or np.any(o >= 1.0):
        raise DomainError("opacity must lie strictly inside (0, 1)")
    return np.log(o / (1.0 - o))


def quat_rotation(q: np.ndarray) -> np.ndarray:
    """[k, 3, 3] rotation matrices of (w, x, y, z) quaternions, normalised
    (the 3DGS convention, as gs_noise.cu builds them)."""
    q = np.asarray(q, np.float64)
    q = q / np.maximum(np.linalg.norm(q, axis=1, keepdims=True), 1e-12)
    w, x, y, z = q.T
    r = np.empty((q.shape[0], 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - w * z)
    r[:, 0, 2] = 2 * (x * z + w * y)
    r[:, 1, 0] = 2 * (x * y + w * z)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - w * x)
    r[:, 2, 0] = 2 * (x * z - w * y)
    r[:, 2, 1] = 2 * (y * z + w * x)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def densify_adc(opt, accum, count, cfg: DensifyConfig, rng: np.random.Generator, alive=None,
                iteration: int = 0) -> DensifyResult:
    """Clone, split, then prune (pipeline.py:116-185) for the reference's 2-D
    layout (position 2, log scale 2, rotation angle 1, opacity 1, plain
    groups) and for the 3DGS SH-3 layout (xyz 3, log scaling 3, rotation
    quaternion 4, opacity 1, f_dc / f_rest carried along): a split child is
    sampled in the parent's 3-D footprint, R(q) (exp(scaling) * gamma) with
    gamma ~ N(0, I_3) clipped at norm 2.5 (oracle densify_adc_sh3_f64).

    The decisions and the few new attribute values are computed on the host in
    float64 with the reference's formulas and ``rng`` draws:
    * hot rows: mean gradient norm over the threshold (``accum`` / ``count``,
      the fused densification statistics);
    * clone/split by the largest scale;
    * blend-preserving clone opacity;
    * split children sampled inside the parent footprint;
    * prune at low opacity.
    The new rows are built on the GPU as one gather of the parameter rows
    (one record gather for record views) and of the moment record, plus small
    patches. The optimizer is rebound to the new rows: children start with
    zero moments and clock, and the densification statistics restart from
    zero, as ``stats.reset`` does.
    """
    import torch

    from . import _lib as L
    from .records import record_of, views_like

    roles = {g["role"]: g for g in opt.param_groups}
    need = (L.ROLE_POSITION, L.ROLE_SCALE, L.ROLE_OPACITY)
    if any(r not in roles for r in need):
        raise ConfigError("densify_adc needs position, scale and opacity groups")
    pos_g, sc_g, op_g = (roles[r] for r in need)
    rot_g = next((g for g in opt.param_groups if g["name"] in ("rot", "rotation")), None)
    pos_t, sc_t, op_t = (g["params"][0] for g in (pos_g, sc_g, op_g))
    n = opt.n_rows
    dims = pos_t.reshape(n, -1).shape[1]
    rot_w = None if rot_g is None else rot_g["params"][0].reshape(n, -1).shape[1]
    if (dims, sc_t.reshape(n, -1).shape[1], rot_w) not in ((2, 2, 1), (3, 3, 4)):
        raise ConfigError("densify_adc splits the reference's 2-D layout (mu 2, kappa 2, rot "
                          "angle 1) or the 3DGS layout (xyz 3, scaling 3, rotation quaternion 4)")
    host = lambda t: t.detach().reshape(n, -1).cpu().numpy().astype(np.float64)  # noqa: E731
    tau = host(op_t)[:, 0]
    kappa = host(sc_t)
    acc = np.asarray(accum.detach().cpu().numpy() if hasattr(accum, "detach") else accum,
                     np.float64).reshape(-1)
    cnt = np.asarray(count.detach().cpu().numpy() if hasattr(count, "detach") else count,
                     np.int64).reshape(-1)
    alive = (np.ones(n, bool) if alive is None else
             np.asarray(alive.detach().cpu().numpy() if hasattr(alive, "detach") else alive,
                        bool).reshape(-1))
    events = []
    mean_grad = acc / np.maximum(cnt, 1)
    scale_max = np.exp(kappa).max(axis=1)
    hot = alive & (mean_grad > cfg.grad_threshold) & (cnt > 0)
    clone_rows = np.flatnonzero(hot & (scale_max <= cfg.split_scale_px))
    split_rows = np.flatnonzero(hot & (scale_max > cfg.split_scale_px))
    n_new = clone_rows.size + 2 * split_rows.size
    if n_new and n + n_new - split_rows.size > cfg.max_primitives:
        events.append(_event(iteration, "densify_skip", np.concatenate([clone_rows, split_rows])))
        clone_rows = split_rows = np.empty(0, dtype=np.int64)

    patches = {}  # name -> list of (merged rows, float64 values [k, w])
    tau_m = [tau.copy()]
    if clone_rows.size:
        o = opacity_f64(tau[clone_rows])
        tau_c = _logit_checked(1.0 - np.power(1.0 - o, 1.0 / 2.0))   # _clone_opacity, k = 2
        tau_m[0][clone_rows] = tau_c
        tau_m.append(tau_c)
        patches.setdefault(op_g["name"], []).append((clone_rows, tau_c[:, None]))
        patches[op_g["name"]].append((n + np.arange(clone_rows.size), tau_c[:, None]))
        events.append(_event(iteration, "clone", clone_rows))
    if split_rows.size:
        mu = host(pos_t)[split_rows]
        rot = host(rot_g["params"][0])[split_rows]
        rot = rot[:, 0] if dims == 2 else rot
        ks = kappa[split_rows]
        base = n + clone_rows.size
        for c in range(2):
            # pipeline.py:153-162; in 3-D gamma ~ N(0, I_3) and the offset is
            # rotated by the quaternion (the 2-D rule, one dimension up)
            gamma = rng.standard_normal((split_rows.size, dims))
            norms = np.linalg.norm(gamma, axis=1)
            gamma *= (np.minimum(norms, 2.5) / np.maximum(norms, 1e-12))[:, None]
            s = np.exp(ks)
            local = s * gamma
            cmu = mu.copy()
            if dims == 2:
                cs, sn = np.cos(rot), np.sin(rot)
                cmu[:, 0] += cs * local[:, 0] - sn * local[:, 1]
                cmu[:, 1] += sn * local[:, 0] + cs * local[:, 1]
            else:
                cmu += np.einsum("kij,kj->ki", quat_rotation(rot), local)
            rows = base + c * split_rows.size + np.arange(split_rows.size)
            patches.setdefault(pos_g["name"], []).append((rows, cmu))
            patches.setdefault(sc_g["name"], []).append((rows, ks - np.log(cfg.split_shrink)))
            tau_m.append(tau[split_rows])
        events.append(_event(iteration, "split", split_rows))
    src_m = np.concatenate([np.arange(n), clone_rows, split_rows, split_rows]).astype(np.int64)
    tau_all = np.concatenate(tau_m) if len(tau_m) > 1 else tau_m[0]
    alive_m = alive[src_m]
    keep = np.ones(src_m.size, bool)
    keep[split_rows] = False
    prune = alive_m & (opacity_f64(tau_all) <= cfg.prune_opacity)
    pruned_ids = np.flatnonzero(prune & keep)
    keep &= ~prune
    if pruned_ids.size:
        events.append(_event(iteration, "prune", pruned_ids))
    final_src = src_m[keep]
    final_pos = np.cumsum(keep) - 1          # merged row -> output row (where kept)

    # ---- device: one gather of the parameter rows + patches; state rows ----
    dev = opt.device
    idx = torch.from_numpy(final_src).to(dev)
    old = {g["name"]: g["params"][0] for g in opt.param_groups}
    rec = record_of(old)   # packed or adopted parameter record
    if rec is not None:
        new_params = views_like(rec.detach().index_select(0, idx), old)
    else:
        new_params = {k: t.detach().index_select(0, idx).contiguous() for k, t in old.items()}
    with torch.no_grad():
        for name, plist in patches.items():
            t2 = new_params[name].reshape(final_src.size, -1)
            for rows, vals in plist:
                sel = keep[rows]
                if not sel.any():
                    continue
                r = torch.from_numpy(final_pos[rows[sel]]).to(dev)
                t2[r] = torch.from_numpy(np.asarray(vals[sel], np.float32)).to(dev)
    new_state = opt.state.select(idx)
    children = np.flatnonzero(np.flatnonzero(keep) >= n)   # output rows that are new
    opt.rebind(new_params, new_state)
    if children.size:
        opt.reset_rows(children)
    return DensifyResult(new_params, alive_m[keep], final_src, events)
