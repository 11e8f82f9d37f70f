"""CPU oracle for the AdamW-GS optimizer step — TEST INFRASTRUCTURE ONLY.

Not part of the product: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU legs may import this module (see ``oracle/__init__.py``).

Two restatements of the reference step, both over an arbitrary ordered
group layout (the reference's 2D ``mu/kappa/rot/tau/color`` testbed or the
3DGS SH-3 ``xyz/f_dc/f_rest/opacity/scaling/rotation`` layout):

``*_f64``
    The reference algorithm of ``/root/reference/pkg/src/splatlab/optimizer.py``
    restated in NumPy float64 with the reference's own association order, so
    that it reproduces the reference bit for bit.  Pinned against golden
    vectors written by the UNMODIFIED reference (``tests/golden/make_golden.py``
    imports ``splatlab`` and drives it through the SH-3 adapter of SURVEY §8(c)).

``step_fp32``
    The exact fp32 operation order of the CUDA kernels
    (``paper_2601_16736_b200/csrc/gs_common.cuh::update_element``): every
    operation one correctly rounded fp32 op, no FMA contraction, the
    activation derivatives through the kernel's own deterministic ``gs_expf``,
    bias-correction factors from the same float64-derived LUT.  The GPU path
    must agree with it bit for bit.

Every function cites the reference file:line it follows.  Rows are 2-D
``(N, W)`` arrays for every group (width-1 groups are ``(N, 1)``).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

F32 = np.float32
F64 = np.float64

MODES = ("coupled-adam", "sparse-adam", "adamw-const", "adamw-const-clip", "adamw-gs")
ACTIVE_OPACITY_THRESHOLD = 1.0 / 255.0          # primitives.py:33
MAX_LOG_SCALE = 80.0                            # primitives.py:37


class OracleDomainError(ValueError):
    """primitives.py:40 DomainError."""


class OracleGradientError(RuntimeError):
    """optimizer.py:62-67 GradientError (carries ``ids``)."""

    def __init__(self, ids):
        self.ids = np.asarray(ids)
        super().__init__(f"non-finite gradient on primitives {self.ids.tolist()[:16]}")


class OracleConfigError(ValueError):
    """optimizer.py:58 ConfigError."""


@dataclass(frozen=True)
class Group:
    """One attribute group: name, row width and role.

    ``role`` is ``"position"`` (takes ``mu_lr_scale``, optimizer.py:217,263),
    ``"opacity"`` (tau DAR, optimizer.py:259-260), ``"scale"`` (kappa DAR,
    optimizer.py:261-262) or ``"plain"``.
    """

    name: str
    width: int
    role: str = "plain"


LAYOUT_REF2D = (Group("mu", 2, "position"), Group("kappa", 2, "scale"), Group("rot", 1),
                Group("tau", 1, "opacity"), Group("color", 3))          # gradients.py:15
LAYOUT_SH3 = (Group("xyz", 3, "position"), Group("f_dc", 3), Group("f_rest", 45),
              Group("opacity", 1, "opacity"), Group("scaling", 3, "scale"), Group("rotation", 4))


@dataclass
class Hyper:
    """The OptimizerConfig fields the step reads (optimizer.py:70-100)."""

    lr: dict
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    lambda_o: float = 0.0
    lambda_s: float = 0.0
    ct_opacity: float = 10.0
    ct_scale: float = 10.0
    round_n_pixels: bool = True


# --------------------------------------------------------------------------
# scalar helpers
# --------------------------------------------------------------------------

def round_pixel_count(n_pixels: int, enabled: bool = True) -> float:
    """optimizer.py:168-178 — keep the leading digit of N_I, divide by ten."""
    if n_pixels <= 0:
        raise OracleConfigError("pixel count must be positive")
    if not enabled:
        return float(n_pixels)
    p = 10 ** math.floor(math.log10(n_pixels))
    return (n_pixels // p) * p / 10.0


def _finite_or_raise(name, x):
    a = np.asarray(x, dtype=F64)
    if not np.all(np.isfinite(a)):
        raise OracleDomainError(f"{name} must be finite")
    return a


def sigmoid_f64(tau):
    """primitives.py:51-59 — stable two-branch sigmoid in float64."""
    t = _finite_or_raise("tau", tau)
    out = np.empty_like(t)
    pos = t >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-t[pos]))
    e = np.exp(t[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def opacity_derivative_f64(tau):
    """primitives.py:62-66 — sigma * (1 - sigma)."""
    o = sigmoid_f64(tau)
    return o * (1.0 - o)


def activate_scale_f64(kappa):
    """primitives.py:78-84 — exp with the kappa > 80 guard."""
    k = _finite_or_raise("kappa", kappa)
    if np.any(k > MAX_LOG_SCALE):
        raise OracleDomainError(f"log-scale above {MAX_LOG_SCALE} would overflow")
    return np.exp(k)


def active_logit_threshold_f32() -> np.float32:
    """Largest fp32 tau with sigmoid_f64(tau) <= 1/255.

    ``classify_active`` (primitives.py:228-238) tests ``sigmoid(tau) > 1/255``
    in float64; on fp32 inputs that is exactly ``tau > T`` for this T because
    the float64 sigmoid is monotone at fp32 spacing near the threshold.
    """
    t = F32(math.log(ACTIVE_OPACITY_THRESHOLD / (1.0 - ACTIVE_OPACITY_THRESHOLD)))
    for _ in range(64):
        if sigmoid_f64(np.array([t], F64))[0] > ACTIVE_OPACITY_THRESHOLD:
            t = np.nextafter(t, F32(-np.inf))
        else:
            break
    while sigmoid_f64(np.array([np.nextafter(t, F32(np.inf))], F64))[0] <= ACTIVE_OPACITY_THRESHOLD:
        t = np.nextafter(t, F32(np.inf))
    return F32(t)


def bias_lut_f32(beta1: float, beta2: float, t_max: int) -> np.ndarray:
    """fp32 bias-correction factors 1/(1-beta^t), t in [0, t_max], from float64.

    The denominators are the reference's ``1 - np.power(beta, t)``
    (optimizer.py:202-203); entry 0 is unused (set to 1).
    """
    t = np.arange(t_max + 1, dtype=F64)
    with np.errstate(divide="ignore"):
        c1 = 1.0 / (1.0 - np.power(beta1, t))
        c2 = 1.0 / (1.0 - np.power(beta2, t))
    c1[0] = c2[0] = 1.0
    return np.stack([c1.astype(F32), c2.astype(F32)], axis=1)


# --------------------------------------------------------------------------
# float64 restatement of the reference (bit-exact with splatlab)
# --------------------------------------------------------------------------

def finite_check_f64(layout, grads):
    """gradients.py:50-58 — ids of rows with any non-finite gradient, or None."""
    n = grads[layout[0].name].shape[0]
    bad = np.zeros(n, dtype=bool)
    for g in layout:
        bad |= ~np.isfinite(grads[g.name]).all(axis=1)
    ids = np.flatnonzero(bad)
    return ids if ids.size else None


def _corrected_f64(m, v, t_rows, beta1, beta2, global_t=None):
    """optimizer.py:187-204 — bias correction with per-row (async) or global clock."""
    if global_t is not None:
        t = float(global_t)
    else:
        t = t_rows.astype(F64)[:, None]
    return m / (1.0 - np.power(beta1, t)), v / (1.0 - np.power(beta2, t))


def _lr_of(g: Group, hp: Hyper, mu_lr_scale: float) -> float:
    """optimizer.py:217,263 — per-group lr, position group scaled."""
    return hp.lr[g.name] * (mu_lr_scale if g.role == "position" else 1.0)


def _update_rows_f64(layout, params, grads, m, v, t, rows, hp, mu_lr_scale, global_t=None):
    """optimizer.py:207-219 — plain Adam on selected rows (association lr*m_hat/(...))."""
    t[rows] += 1                       # one clock for all groups
    for g in layout:
        gr = grads[g.name][rows]
        m[g.name][rows] = hp.beta1 * m[g.name][rows] + (1.0 - hp.beta1) * gr
        v[g.name][rows] = hp.beta2 * v[g.name][rows] + (1.0 - hp.beta2) * (gr * gr)
        mh, vh = _corrected_f64(m[g.name][rows], v[g.name][rows], t[rows], hp.beta1, hp.beta2,
                                global_t)
        lr = _lr_of(g, hp, mu_lr_scale)
        params[g.name][rows] = params[g.name][rows] - lr * mh / (np.sqrt(vh) + hp.eps)


def adam_step_sync_f64(layout, params, grads, m, v, t, state_global_t, hp, mu_lr_scale=1.0):
    """optimizer.py:222-228.  Returns the new global_t."""
    ids = finite_check_f64(layout, grads)
    if ids is not None:
        raise OracleGradientError(ids)
    gt = state_global_t + 1
    _update_rows_f64(layout, params, grads, m, v, t, slice(None), hp, mu_lr_scale, gt)
    return gt


def sparse_adam_step_f64(layout, params, grads, m, v, t, vis, hp, mu_lr_scale=1.0):
    """optimizer.py:231-238."""
    ids = finite_check_f64(layout, grads)
    if ids is not None:
        raise OracleGradientError(ids)
    rows = np.flatnonzero(np.asarray(vis, dtype=bool))
    if rows.size:
        _update_rows_f64(layout, params, grads, m, v, t, rows, hp, mu_lr_scale)


def _decoupled_reg_step_f64(layout, params, grads, m, v, t, vis, hp, mu_lr_scale,
                            extra_opacity, extra_scale):
    """optimizer.py:241-266 (association lr*(m_hat/(...) + extra))."""
    ids = finite_check_f64(layout, grads)
    if ids is not None:
        raise OracleGradientError(ids)
    rows = np.flatnonzero(np.asarray(vis, dtype=bool))
    if rows.size == 0:
        return
    t[rows] += 1
    for g in layout:
        gr = grads[g.name][rows]
        m[g.name][rows] = hp.beta1 * m[g.name][rows] + (1.0 - hp.beta1) * gr
        v[g.name][rows] = hp.beta2 * v[g.name][rows] + (1.0 - hp.beta2) * (gr * gr)
        mh, vh = _corrected_f64(m[g.name][rows], v[g.name][rows], t[rows], hp.beta1, hp.beta2)
        step = mh / (np.sqrt(vh) + hp.eps)
        if g.role == "opacity" and extra_opacity is not None:
            step = step + extra_opacity(params[g.name][rows], vh)
        elif g.role == "scale" and extra_scale is not None:
            step = step + extra_scale(params[g.name][rows], vh)
        lr = _lr_of(g, hp, mu_lr_scale)
        params[g.name][rows] = params[g.name][rows] - lr * step


def dar_step_f64(layout, params, grads, m, v, t, vis, hp, n_pixels, mu_lr_scale=1.0,
                 lambda_o=None, lambda_s=None):
    """optimizer.py:269-298 — DAR: min(lambda*(R'/N_I')/(sqrt(v_hat)+eps), C_t)."""
    lo = hp.lambda_o if lambda_o is None else lambda_o
    ls = hp.lambda_s if lambda_s is None else lambda_s
    if hp.ct_opacity <= 0.0 or hp.ct_scale <= 0.0:
        raise OracleConfigError("clip bounds C_t must be positive")
    n_i = round_pixel_count(n_pixels, hp.round_n_pixels)

    def extra_tau(tau, vh):
        if lo == 0.0:
            return 0.0
        reg = opacity_derivative_f64(tau) / n_i
        return np.minimum(lo * reg / (np.sqrt(vh) + hp.eps), hp.ct_opacity)

    def extra_kappa(kappa, vh):
        if ls == 0.0:
            return 0.0
        reg = activate_scale_f64(kappa) / n_i
        return np.minimum(ls * reg / (np.sqrt(vh) + hp.eps), hp.ct_scale)

    _decoupled_reg_step_f64(layout, params, grads, m, v, t, vis, hp, mu_lr_scale,
                            extra_tau, extra_kappa)


def adamw_const_step_f64(layout, params, grads, m, v, t, vis, hp, clip=None, mu_lr_scale=1.0):
    """optimizer.py:301-324 — constant penalty lambda*R'(theta), optional clamp."""

    def extra_tau(tau, vh):
        if hp.lambda_o == 0.0:
            return 0.0
        term = hp.lambda_o * opacity_derivative_f64(tau)
        return np.minimum(term, clip) if clip is not None else term

    def extra_kappa(kappa, vh):
        if hp.lambda_s == 0.0:
            return 0.0
        term = hp.lambda_s * activate_scale_f64(kappa)
        return np.minimum(term, clip) if clip is not None else term

    _decoupled_reg_step_f64(layout, params, grads, m, v, t, vis, hp, mu_lr_scale,
                            extra_tau, extra_kappa)


def coupled_reg_grad_f64(layout, params, vis, lambda_o, lambda_s, alive=None, apply_to_all=False):
    """loss.py:177-198 — coupled L1 gradients lambda*R'(theta)/N_v.

    Returns ``{group_name: grad}`` for the opacity and scale groups.
    """
    n = params[layout[0].name].shape[0]
    out = {g.name: np.zeros((n, g.width)) for g in layout if g.role in ("opacity", "scale")}
    n_vis = int(np.asarray(vis).sum())
    if n_vis == 0 or (lambda_o == 0.0 and lambda_s == 0.0):
        return out
    if apply_to_all:
        rows = np.ones(n, bool) if alive is None else np.asarray(alive, bool)
    else:
        rows = np.asarray(vis, dtype=bool)
    for g in layout:
        if g.role == "opacity" and lambda_o != 0.0:
            out[g.name][rows] = lambda_o * opacity_derivative_f64(params[g.name][rows]) / n_vis
        elif g.role == "scale" and lambda_s != 0.0:
            out[g.name][rows] = lambda_s * activate_scale_f64(params[g.name][rows]) / n_vis
    return out


def rsr_apply_f64(layout, m, v, indices, alpha1, alpha2):
    """optimizer.py:327-340 — m *= alpha1, v *= alpha2 on the rows; clock untouched."""
    if not (0.0 <= alpha1 < 1.0 and 0.0 <= alpha2 < 1.0):
        raise OracleConfigError("RSR factors must lie in [0, 1)")
    for g in layout:
        m[g.name][indices] *= alpha1
        v[g.name][indices] *= alpha2


def reset_rows_f64(layout, m, v, t, indices):
    """optimizer.py:159-165 — m = v = 0, t = 0 on the rows."""
    for g in layout:
        m[g.name][indices] = 0.0
        v[g.name][indices] = 0.0
    t[indices] = 0


def classify_active_f64(tau, alive=None, threshold=ACTIVE_OPACITY_THRESHOLD):
    """primitives.py:228-238 — (n_active, n_dead) over alive rows."""
    tau = np.asarray(tau, F64).reshape(-1)
    alive = np.ones(tau.shape[0], bool) if alive is None else np.asarray(alive, bool)
    active = alive & (sigmoid_f64(tau) > threshold)
    n_active = int(active.sum())
    return n_active, int(alive.sum()) - n_active


def moment_stats_f64(layout, m, v, alive=None):
    """optimizer.py:489-506 — per-group mean/max sqrt(v) and |m|/sqrt(v) over alive rows."""
    out = {}
    for g in layout:
        n = m[g.name].shape[0]
        al = np.ones(n, bool) if alive is None else np.asarray(alive, bool)
        vv = np.asarray(v[g.name], F64)[al].reshape(-1)
        mm = np.asarray(m[g.name], F64)[al].reshape(-1)
        sq = np.sqrt(vv)
        pos = sq > 0.0
        ratio = np.abs(mm[pos]) / sq[pos]
        out[g.name] = {
            "mean_sqrt_v": float(sq.mean()) if sq.size else 0.0,
            "max_sqrt_v": float(sq.max()) if sq.size else 0.0,
            "mean_abs_m_over_sqrt_v": float(ratio.mean()) if ratio.size else 0.0,
            "max_abs_m_over_sqrt_v": float(ratio.max()) if ratio.size else 0.0,
        }
    return out


def flatnonzero(mask) -> np.ndarray:
    """optimizer.py:235,249 — the visibility compaction, ascending indices."""
    return np.flatnonzero(np.asarray(mask, dtype=bool))


# --------------------------------------------------------------------------
# host RNG restatement for the RSR sample (rng.py:17-30, optimizer.py:379-386)
# --------------------------------------------------------------------------

def rng_stream(seed: int, label: str, *indices: int) -> np.random.Generator:
    """rng.py:17-30 — Philox keyed by (seed, blake2b-4(label), indices)."""
    key = (int.from_bytes(hashlib.blake2b(label.encode("utf-8"), digest_size=4).digest(), "little"),
           *(int(i) & 0xFFFFFFFF for i in indices))
    ss = np.random.SeedSequence(entropy=int(seed), spawn_key=key)
    return np.random.Generator(np.random.Philox(ss))


def stss_sample(milestones, iteration: int, n_p: int, rng: np.random.Generator) -> np.ndarray:
    """optimizer.py:359-364,379-386 — floor(ratio*N) sorted distinct rows."""
    ratio = 0.0
    for it, r in milestones:
        if iteration >= it:
            ratio = r
    k = int(math.floor(ratio * n_p))
    if k <= 0:
        return np.empty(0, dtype=np.int64)
    return np.sort(rng.choice(n_p, size=k, replace=False).astype(np.int64))


# --------------------------------------------------------------------------
# fp32 restatement in the CUDA kernel's exact op order
# --------------------------------------------------------------------------

STAT_FIELDS = ("n_visible", "n_stepped", "n_bad_grad", "n_bad_domain", "n_active_pre",
               "n_active_post", "n_clip_opacity", "n_clip_scale", "sum_extra_opacity",
               "sum_extra_scale")


_EXP_C = tuple(F32(c) for c in (1.0 / 5040, 1.0 / 720, 1.0 / 120, 1.0 / 24, 1.0 / 6, 0.5, 1.0,
                                  1.0))


def gs_expf(x):
    """The kernel's deterministic fp32 exp (csrc/gs_common.cuh::gs_expf).

    Cody-Waite reduction x = n*ln2 + r, degree-7 Taylor polynomial in Horner
    form, exact power-of-two scaling; every operation one rounded fp32 op.
    Inputs below -86 return 0.
    """
    x = np.asarray(x, F32)
    n = np.rint(x * F32(1.442695))
    r = x - n * F32(0.693145751953125)
    r = r - n * F32(1.4286068e-06)
    p = _EXP_C[0] * np.ones_like(r)
    for c in _EXP_C[1:]:
        p = p * r + c
    with np.errstate(over="ignore", invalid="ignore"):
        scale = np.ldexp(np.ones_like(p), np.clip(n, -126, 127).astype(np.int32)).astype(F32)
    out = (p * scale).astype(F32)
    return np.where(x < F32(-86.0), F32(0.0), out).astype(F32)


def _reg_deriv_f32(role, theta32):
    """R'(theta) in fp32 (gs_common.cuh::reg_deriv): sigma' = e/(1+e)^2 with
    e = exp(-|tau|) for opacity (primitives.py:51-66), exp(kappa) for scale."""
    th = np.asarray(theta32, F32)
    if role == "opacity":
        e = gs_expf(-np.abs(th))
        d = F32(1.0) + e
        return (e / (d * d)).astype(F32)
    return gs_expf(th)


def _domain_bad(role, theta32):
    th = theta32.astype(F64)
    bad = ~np.isfinite(th)
    if role == "scale":
        bad |= th > MAX_LOG_SCALE
    return bad.any(axis=1)


def step_fp32(mode, layout, params, grads, m, v, clock, rows, hp, *, n_pixels=None,
              mu_lr_scale=1.0, lambda_o=None, lambda_s=None, clip=None, n_visible_norm=None,
              global_t=None, lut=None, alive=None, skip_bad_rows=True):
    """One fused step in the kernel's fp32 op order; mutates the fp32 arrays in place.

    ``rows`` is the ascending visible index list (dense ``coupled-adam`` passes
    all rows).  ``n_visible_norm`` is N_v for the coupled regularization
    (``sparse-adam`` / ``coupled-adam`` with lambda != 0).  Returns the
    per-step statistics dict (STAT_FIELDS).  Bad rows (non-finite gradient,
    or tau/kappa out of the activation domain where a penalty is active) are
    skipped and counted, as the kernel does in fused-check mode.
    """
    assert mode in MODES
    rows = np.asarray(rows, dtype=np.int64)
    dense = mode == "coupled-adam"
    coupled = mode in ("sparse-adam", "coupled-adam")
    if coupled:
        # the pipeline's coupled composite (pipeline.py:305-315): lambdas are
        # explicit, absent means plain sparse / sync Adam
        lo = 0.0 if lambda_o is None else lambda_o
        ls = 0.0 if lambda_s is None else lambda_s
    elif mode == "adamw-gs":
        lo = hp.lambda_o if lambda_o is None else lambda_o        # optimizer.py:279-280
        ls = hp.lambda_s if lambda_s is None else lambda_s
    else:
        lo, ls = hp.lambda_o, hp.lambda_s                         # optimizer.py:312,318
    n_i = round_pixel_count(n_pixels, hp.round_n_pixels) if mode == "adamw-gs" else None
    a1 = F32(1.0 - hp.beta1)
    a2 = F32(1.0 - hp.beta2)
    eps = F32(hp.eps)
    if lut is None:
        tmax = int(clock.max(initial=0)) + 2 if not dense else int(global_t) + 1
        lut = bias_lut_f32(hp.beta1, hp.beta2, max(tmax, 2))
    thr = active_logit_threshold_f32()

    stats = {k: 0 for k in STAT_FIELDS}
    stats["sum_extra_opacity"] = 0.0
    stats["sum_extra_scale"] = 0.0
    stats["n_visible"] = int(rows.size)
    if rows.size == 0:
        return stats
    if coupled and (n_visible_norm is None or n_visible_norm == 0):
        lo_c = ls_c = 0.0
    else:
        lo_c, ls_c = lo, ls

    # ---- pass A: per-row validity --------------------------------------
    bad_grad = np.zeros(rows.size, bool)
    bad_dom = np.zeros(rows.size, bool)
    for g in layout:
        bad_grad |= ~np.isfinite(grads[g.name][rows]).all(axis=1)
        lam = lo if g.role == "opacity" else ls if g.role == "scale" else 0.0
        if coupled:
            lam = lo_c if g.role == "opacity" else ls_c if g.role == "scale" else 0.0
        if g.role in ("opacity", "scale") and lam != 0.0:
            bad_dom |= _domain_bad(g.role, params[g.name][rows])
    if coupled:
        # coupled reg is added to the gradient first; a domain error makes it
        # non-computable, a non-finite sum is a gradient error
        pass
    bad_dom &= ~bad_grad
    ok = ~(bad_grad | bad_dom) if skip_bad_rows else np.ones(rows.size, bool)
    stats["n_bad_grad"] = int(bad_grad.sum())
    stats["n_bad_domain"] = int(bad_dom.sum())
    r = rows[ok]
    stats["n_stepped"] = int(r.size)
    if r.size == 0:
        return stats

    # ---- clocks and bias correction --------------------------------------
    clock[r] += 1
    tb = np.full(r.size, int(global_t)) if dense else clock[r].astype(np.int64)
    inside = tb < lut.shape[0]
    c1 = np.empty(r.size, F32)
    c2 = np.empty(r.size, F32)
    c1[inside] = lut[tb[inside], 0]
    c2[inside] = lut[tb[inside], 1]
    tf = tb[~inside].astype(F64)          # past the table: float64 formula, rounded once
    c1[~inside] = (1.0 / (1.0 - np.power(hp.beta1, tf))).astype(F32)
    c2[~inside] = (1.0 / (1.0 - np.power(hp.beta2, tf))).astype(F32)
    c1 = c1[:, None]
    c2 = c2[:, None]

    lam32 = {"opacity": F32(lo), "scale": F32(ls)}
    cap32 = {"opacity": F32(hp.ct_opacity), "scale": F32(hp.ct_scale)}
    if mode in ("adamw-const", "adamw-const-clip") and (clip is not None or
                                                        mode == "adamw-const-clip"):
        c = clip if clip is not None else hp.ct_opacity          # pipeline.py:323-325
        cap32 = {"opacity": F32(c), "scale": F32(c)}
    inv_ni = F32(1.0 / n_i) if n_i else F32(0.0)
    inv_nv = (F32(1.0) / F32(n_visible_norm)) if (coupled and n_visible_norm) else F32(0.0)
    for g in layout:
        th = params[g.name][r]
        gr = grads[g.name][r]
        mm = m[g.name][r]
        vv = v[g.name][r]
        lam = lam32.get(g.role, F32(0.0)) if g.role in ("opacity", "scale") else F32(0.0)
        if coupled and g.role in ("opacity", "scale") and lam != 0.0 and (lo_c or ls_c):
            # loss.py:177-198 folded in: g += (lambda * R') * (1/N_v)
            gr = gr + (lam * _reg_deriv_f32(g.role, th)) * inv_nv
        d = gr - mm
        m_new = mm + a1 * d
        g2 = gr * gr
        e = g2 - vv
        v_new = vv + a2 * e
        mh = m_new * c1
        vh = v_new * c2
        den = np.sqrt(vh) + eps
        step = mh / den
        if g.role in ("opacity", "scale") and not coupled and lam != 0.0:
            deriv = _reg_deriv_f32(g.role, th)
            cap = cap32[g.role]
            if mode == "adamw-gs":
                # min(lambda * (R' / N_I') / (sqrt(v^) + eps), C_t), optimizer.py:285-295
                x = ((lam * deriv) * inv_ni) / den
                clipped = x >= cap
                ex = np.where(clipped, cap, x).astype(F32)
            elif mode == "adamw-const-clip" or clip is not None:
                x = lam * deriv                                   # optimizer.py:314-315
                clipped = x >= cap
                ex = np.where(clipped, cap, x).astype(F32)
            else:
                ex = (lam * deriv).astype(F32)
                clipped = np.zeros(ex.shape, bool)
            step = step + ex
            key = "opacity" if g.role == "opacity" else "scale"
            stats["n_clip_" + key] += int(clipped.sum())
            stats["sum_extra_" + key] += float(ex.astype(F64).sum())
        lr = F32(hp.lr[g.name] * (mu_lr_scale if g.role == "position" else 1.0))
        th_new = th - lr * step
        if g.role == "opacity":
            stats["n_active_pre"] += int((th[:, 0] > thr).sum())
            stats["n_active_post"] += int((th_new[:, 0] > thr).sum())
        params[g.name][r] = th_new
        m[g.name][r] = m_new
        v[g.name][r] = v_new
    return stats


def densify_observe_fp32(grad_pos, rows, accum, count, scale):
    """DensifyStats.observe (pipeline.py:77-82) in the kernels' fp32 order:
    accum[r] += sqrt(sum_c g_c^2) * scale (sequential fp32 sum), count[r] += 1."""
    g = np.asarray(grad_pos, F32)[rows]
    s2 = np.zeros(g.shape[0], F32)
    for c in range(g.shape[1]):
        s2 = s2 + g[:, c] * g[:, c]
    accum[rows] = accum[rows] + np.sqrt(s2) * F32(scale)
    count[rows] += 1


def densify_observe_f64(grad_pos, vis, accum, count, view_scale):
    """pipeline.py:77-82 restated (float64): the reference's DensifyStats.observe."""
    rows = np.flatnonzero(vis)
    if rows.size:
        norms = np.linalg.norm(np.asarray(grad_pos, F64)[rows], axis=1) * view_scale
        accum[rows] += norms
        count[rows] += 1


def aiu_apply_f64(layout, params, m, v, t, vis, alive, lr, beta1, beta2, eps, prob, eta, rng):
    """optimizer.py:425-450 restated: extra steps on sampled invisible rows with
    frozen moments and clocks; returns the picked rows (int64)."""
    invisible = np.flatnonzero(np.asarray(alive, bool) & ~np.asarray(vis, bool))
    if invisible.size == 0 or prob <= 0.0 or eta == 0.0:
        return np.empty(0, dtype=np.int64)
    picked = invisible[rng.random(invisible.size) < prob]
    if picked.size == 0:
        return picked
    for g in layout:
        started = picked[t[picked] > 0]
        if started.size == 0:
            continue
        mh, vh = _corrected_f64(m[g.name][started], v[g.name][started], t[started], beta1, beta2)
        params[g.name][started] = params[g.name][started] - lr[g.name] * eta * mh / (
            np.sqrt(vh) + eps)
    return picked


def aiu_apply_fp32(layout, params, m, v, t, picked, lr, eta, eps, lut):
    """The AIU kernel's fp32 order (gs_state.cu::aiu_rows_kernel):
    theta -= (fl32(lr*eta) * m^) / (sqrt(v^) + eps), rows with clock 0 skipped."""
    rows = np.asarray(picked, np.int64)
    rows = rows[t[rows] > 0]
    tb = np.minimum(t[rows], lut.shape[0] - 1)
    c1 = lut[tb, 0][:, None]
    c2 = lut[tb, 1][:, None]
    for g in layout:
        mh = m[g.name][rows] * c1
        vh = v[g.name][rows] * c2
        den = np.sqrt(vh) + F32(eps)
        params[g.name][rows] = params[g.name][rows] - (F32(lr[g.name] * eta) * mh) / den


def _sigmoid_ref_f64(tau):
    """activate_opacity (primitives.py:51-59), float64, branch-stable."""
    t = np.asarray(tau, np.float64)
    out = np.empty_like(t)
    pos = t >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-t[pos]))
    e = np.exp(t[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def mcmc_relocate_f64(layout, params, m, v, t, alive, rng, opacity="tau"):
    """mcmc_relocate (pipeline.py:197-233) on host arrays, float64: dead rows
    (alive, o <= 1/255) take the attributes of opacity-weighted live targets
    drawn with ``rng.choice``; target and respawns share the blend-preserving
    opacity 1 - (1 - o)^(1/(k+1)) (_clone_opacity, pipeline.py:110-113); the
    respawns' moments and clocks are reset (optimizer.py:159-165).  Returns
    the dead rows."""
    o = _sigmoid_ref_f64(params[opacity].reshape(-1))
    alive = np.ones(o.size, bool) if alive is None else np.asarray(alive, bool)
    dead = np.flatnonzero(alive & (o <= 1.0 / 255.0))
    live = np.flatnonzero(alive & (o > 1.0 / 255.0))
    if live.size == 0:
        raise RuntimeError("no alive primitives to relocate onto")
    if dead.size == 0:
        return dead
    probs = o[live] / o[live].sum()
    targets = live[rng.choice(live.size, size=dead.size, p=probs)]
    uniq, inverse, counts = np.unique(targets, return_inverse=True, return_counts=True)
    k = np.asarray(counts + 1.0, np.float64)
    o_new = 1.0 - np.power(1.0 - o[uniq], 1.0 / k)
    tau_new = np.log(o_new / (1.0 - o_new))
    for g in layout:
        if g.name != opacity:
            params[g.name][dead] = params[g.name][targets]
    params[opacity].reshape(-1)[dead] = tau_new[inverse]
    params[opacity].reshape(-1)[uniq] = tau_new
    for g in layout:
        m[g.name][dead] = 0.0
        v[g.name][dead] = 0.0
    t[dead] = 0
    return dead


def densify_adc_f64(params, m, v, t, alive, accum, count, cfg, rng):
    """densify_adc (pipeline.py:116-185) on the 2-D layout's host arrays,
    float64: clone (blend-preserving opacity), split (children sampled in the
    parent footprint with ``rng``, scales shrunk), prune; children get zero
    moments and clocks.  Returns (params, m, v, t, alive, src, event counts)."""
    n = params["tau"].shape[0]
    tau = params["tau"].reshape(-1).astype(np.float64).copy()
    kappa = params["kappa"].astype(np.float64)
    mean = accum / np.maximum(count, 1)
    hot = alive & (mean > cfg["grad_threshold"]) & (count > 0)
    smax = np.exp(kappa).max(axis=1)
    clone = np.flatnonzero(hot & (smax <= cfg["split_scale_px"]))
    split = np.flatnonzero(hot & (smax > cfg["split_scale_px"]))
    if clone.size + 2 * split.size and n + clone.size + split.size > cfg["max_primitives"]:
        clone = split = np.empty(0, np.int64)
    pieces = {k: [a.astype(np.float64).reshape(n, -1)] for k, a in params.items()}
    if clone.size:
        o = _sigmoid_ref_f64(tau[clone])
        o2 = 1.0 - np.power(1.0 - o, 1.0 / 2.0)
        tc = np.log(o2 / (1.0 - o2))
        for k in params:
            pieces[k].append(pieces[k][0][clone].copy())
        pieces["tau"][-1][:, 0] = tc
        pieces["tau"][0][clone, 0] = tc
    for _ in range(2 if split.size else 0):
        child = {k: pieces[k][0][split].copy() for k in params}
        gamma = rng.standard_normal((split.size, 2))
        norms = np.linalg.norm(gamma, axis=1)
        gamma *= (np.minimum(norms, 2.5) / np.maximum(norms, 1e-12))[:, None]
        s = np.exp(child["kappa"])
        c, sn = np.cos(child["rot"][:, 0]), np.sin(child["rot"][:, 0])
        local = s * gamma
        child["mu"][:, 0] += c * local[:, 0] - sn * local[:, 1]
        child["mu"][:, 1] += sn * local[:, 0] + c * local[:, 1]
        child["kappa"] -= np.log(cfg["split_shrink"])
        for k in params:
            pieces[k].append(child[k])
    merged = {k: np.concatenate(p) for k, p in pieces.items()}
    src = np.concatenate([np.arange(n), clone, split, split]).astype(np.int64)
    nm = src.size
    am = alive[src]
    keep = np.ones(nm, bool)
    keep[split] = False
    prune = am & (_sigmoid_ref_f64(merged["tau"][:, 0]) <= cfg["prune_opacity"])
    n_pruned = int((prune & keep).sum())
    keep &= ~prune
    fresh = np.arange(nm) >= n
    out_m = {k: np.where(fresh[:, None], 0.0, x.reshape(n, -1)[src])[keep] for k, x in m.items()}
    out_v = {k: np.where(fresh[:, None], 0.0, x.reshape(n, -1)[src])[keep] for k, x in v.items()}
    out_t = np.where(fresh, 0, t[src])[keep]
    return ({k: x[keep] for k, x in merged.items()}, out_m, out_v, out_t, am[keep], src[keep],
            (int(clone.size), int(split.size), n_pruned))


def quat_rotation_f64(q):
    """Rotation matrices [k, 3, 3] of (w, x, y, z) quaternions, normalised
    (the 3DGS convention; the same matrix gs_noise.cu builds)."""
    q = np.asarray(q, F64)
    q = q / np.maximum(np.linalg.norm(q, axis=1, keepdims=True), 1e-12)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], 1)


def densify_adc_sh3_f64(params, m, v, t, alive, accum, count, cfg, rng):
    """densify_adc (pipeline.py:116-185) generalised to the 3DGS SH-3 layout
    (xyz 3, f_dc 3, f_rest 45, opacity 1, log scaling 3, rotation quaternion
    4), float64.  Decisions, clone opacity, prune and the rng draw order are
    the reference's; a split child is sampled inside the parent's 3-D
    footprint: gamma ~ N(0, I_3) (one rng.standard_normal((k, 3)) per child,
    where the 2-D reference draws (k, 2)), its norm clipped at 2.5 as in
    pipeline.py:155-157, offset R(q) (exp(scaling) * gamma), and the log
    scales shrink by log(split_shrink).  Returns like densify_adc_f64."""
    n = params["opacity"].shape[0]
    tau = params["opacity"].reshape(-1).astype(np.float64).copy()
    kappa = params["scaling"].astype(np.float64)
    mean = accum / np.maximum(count, 1)
    hot = alive & (mean > cfg["grad_threshold"]) & (count > 0)
    smax = np.exp(kappa).max(axis=1)
    clone = np.flatnonzero(hot & (smax <= cfg["split_scale_px"]))
    split = np.flatnonzero(hot & (smax > cfg["split_scale_px"]))
    if clone.size + 2 * split.size and n + clone.size + split.size > cfg["max_primitives"]:
        clone = split = np.empty(0, np.int64)
    pieces = {k: [a.astype(np.float64).reshape(n, -1)] for k, a in params.items()}
    if clone.size:
        o = _sigmoid_ref_f64(tau[clone])
        o2 = 1.0 - np.power(1.0 - o, 1.0 / 2.0)
        tc = np.log(o2 / (1.0 - o2))
        for k in params:
            pieces[k].append(pieces[k][0][clone].copy())
        pieces["opacity"][-1][:, 0] = tc
        pieces["opacity"][0][clone, 0] = tc
    for _ in range(2 if split.size else 0):
        child = {k: pieces[k][0][split].copy() for k in params}
        gamma = rng.standard_normal((split.size, 3))
        norms = np.linalg.norm(gamma, axis=1)
        gamma *= (np.minimum(norms, 2.5) / np.maximum(norms, 1e-12))[:, None]
        local = np.exp(child["scaling"]) * gamma
        child["xyz"] += np.einsum("kij,kj->ki", quat_rotation_f64(child["rotation"]), local)
        child["scaling"] -= np.log(cfg["split_shrink"])
        for k in params:
            pieces[k].append(child[k])
    merged = {k: np.concatenate(p) for k, p in pieces.items()}
    src = np.concatenate([np.arange(n), clone, split, split]).astype(np.int64)
    nm = src.size
    am = alive[src]
    keep = np.ones(nm, bool)
    keep[split] = False
    prune = am & (_sigmoid_ref_f64(merged["opacity"][:, 0]) <= cfg["prune_opacity"])
    n_pruned = int((prune & keep).sum())
    keep &= ~prune
    fresh = np.arange(nm) >= n
    out_m = {k: np.where(fresh[:, None], 0.0, x.reshape(n, -1)[src])[keep] for k, x in m.items()}
    out_v = {k: np.where(fresh[:, None], 0.0, x.reshape(n, -1)[src])[keep] for k, x in v.items()}
    out_t = np.where(fresh, 0, t[src])[keep]
    return ({k: x[keep] for k, x in merged.items()}, out_m, out_v, out_t, am[keep], src[keep],
            (int(clone.size), int(split.size), n_pruned))


# --------------------------------------------------------------------------
# NumPy's Philox4x64-10 (the reference's rng.stream bit generator,
# rng.py:17-30) and Generator.random, restated: pins the GPU Bernoulli draw
# (gs_philox_bernoulli) that replaces the host draw of aiu_apply
# (optimizer.py:437-440).  Third-party algorithm: numpy.random.Philox
# (numpy/random/src/philox/philox.h, Random123 philox4x64 with 10 rounds);
# numpy 2.3 in this image.
# --------------------------------------------------------------------------
_M64 = (1 << 64) - 1
PHILOX_M0, PHILOX_M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
PHILOX_W0, PHILOX_W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B


def philox4x64_block(ctr, key):
    """Random123 philox4x64_R(10, ctr, key): four uint64 outputs."""
    c = [int(x) & _M64 for x in ctr]
    k0, k1 = int(key[0]) & _M64, int(key[1]) & _M64
    for r in range(10):
        if r:
            k0 = (k0 + PHILOX_W0) & _M64
            k1 = (k1 + PHILOX_W1) & _M64
        p0 = PHILOX_M0 * c[0]
        p1 = PHILOX_M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & _M64, (p0 >> 64) ^ c[3] ^ k1, p0 & _M64]
    return c


def philox_uniforms(state: dict, n: int) -> np.ndarray:
    """Generator(Philox).random(n) from a bit_generator.state dict: the
    buffered outputs first, then one block per counter increment
    (philox_next), each uint64 -> (x >> 11) * 2^-53 (next_double)."""
    st = state["state"]
    ctr = [int(x) for x in st["counter"]]
    key = [int(x) for x in st["key"]]
    buf = [int(x) for x in state["buffer"]]
    pos = int(state["buffer_pos"])
    out = np.empty(n, F64)
    for i in range(n):
        if pos >= 4:
            v = (ctr[0] + (ctr[1] << 64) + (ctr[2] << 128) + (ctr[3] << 192) + 1) % (1 << 256)
            ctr = [(v >> (64 * j)) & _M64 for j in range(4)]
            buf = philox4x64_block(ctr, key)
            pos = 0
        out[i] = (buf[pos] >> 11) * (1.0 / 9007199254740992.0)
        pos += 1
    return out
