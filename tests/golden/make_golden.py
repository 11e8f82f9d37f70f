"""Generate golden vectors from the UNMODIFIED reference optimizer.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports ``splatlab`` from ``/root/reference/pkg/src`` and drives the
reference's own step functions — ``dar_step``, ``sparse_adam_step``,
``adamw_const_step``, ``adam_step_sync``, ``coupled_reg_grad``,
``rsr_apply``, ``stss_sample``, ``classify_active``, ``moment_stats``,
``round_pixel_count`` — on seeded fp32-representable inputs, and writes the
results as ``tests/golden/*.npz``.  The SH-3 layout is driven through the
adapter of SURVEY §8(c): a duck-typed primitive set, a hand-built
``MomentState``, ``ATTR_GROUPS`` patched in ``splatlab.optimizer`` and
``splatlab.gradients``, and ``cfg.lr_f_rest`` added.  Nothing in the
reference is modified on disk.

The GPU box never runs this script; it only reads the committed ``.npz``.
"""

from __future__ import annotations

import json
import math
import sys
import types
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

# reference name  <->  3DGS SH-3 name
SH3_MAP = (("mu", "xyz", 3), ("color", "f_dc", 3), ("f_rest", "f_rest", 45),
           ("tau", "opacity", 1), ("kappa", "scaling", 3), ("rot", "rotation", 4))
REF2D = (("mu", 2), ("kappa", 2), ("rot", 1), ("tau", 1), ("color", 3))

LR_SH3 = {"xyz": 1.6e-4 * 5.0, "f_dc": 2.5e-3, "f_rest": 2.5e-3 / 20.0, "opacity": 0.05,
          "scaling": 5e-3, "rotation": 1e-3}


def _import_reference():
    sys.path.insert(0, str(REF_SRC))
    import splatlab.gradients as gradients
    import splatlab.loss as loss
    import splatlab.optimizer as optimizer
    import splatlab.primitives as primitives
    return gradients, optimizer, primitives, loss


def f32(x):
    return np.asarray(x, dtype=np.float32)


def sh3_params(rng, n):
    """SURVEY §8(d) distributions, rounded to fp32."""
    return {
        "xyz": f32(rng.normal(0.0, 5.0, (n, 3))),
        "f_dc": f32(rng.normal(0.0, 0.5, (n, 3))),
        "f_rest": f32(rng.normal(0.0, 0.05, (n, 45))),
        "opacity": f32(rng.normal(-1.0, 2.0, (n, 1))),
        "scaling": f32(rng.uniform(math.log(1e-3), math.log(0.5), (n, 3))),
        "rotation": f32(rng.normal(0.0, 1.0, (n, 4))),
    }


def grads_for(rng, widths, vis, zero_rows=()):
    """g = z * s, s ~ logU(1e-7, 1e-2); invisible rows exactly 0 (renderer.py:222)."""
    out = {}
    for name, w in widths:
        n = vis.shape[0]
        s = np.exp(rng.uniform(math.log(1e-7), math.log(1e-2), (n, w)))
        g = f32(rng.standard_normal((n, w)) * s)
        g[~vis] = 0.0
        for r in zero_rows:
            g[r] = 0.0
        out[name] = g
    return out


def save(name, meta, arrays):
    arrays = dict(arrays)
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", name, {k: v.shape for k, v in arrays.items() if k != "meta"})


class _PSet(types.SimpleNamespace):
    def __len__(self):
        return len(self.tau)


def run_sh3_case(name, mode, n=32, steps=16, seed=0, p_vis=0.5, lambda_o=1e-3, lambda_s=1e-5,
                 n_pixels=1_000_000, clip=None, mu_lr_scale=1.0, ct=10.0):
    gradients, optimizer, primitives, loss = _import_reference()
    groups = tuple(r for r, _, _ in SH3_MAP)
    saved = (optimizer.ATTR_GROUPS, gradients.ATTR_GROUPS)
    optimizer.ATTR_GROUPS = gradients.ATTR_GROUPS = groups
    try:
        rng = np.random.default_rng(seed)
        p0 = sh3_params(rng, n)
        widths = [(s, w) for _, s, w in SH3_MAP]
        vis_seq = rng.random((steps, n)) < p_vis
        vis_seq[:, 0] = True                       # row 0 always visible
        vis_seq[:, 1] = False                      # row 1 never visible (frozen)
        grads_seq = [grads_for(rng, widths, vis_seq[s], zero_rows=(2,)) for s in range(steps)]

        def to_ref(arr, w):
            a = np.asarray(arr, dtype=np.float64)
            return a[:, 0].copy() if w == 1 and a.ndim == 2 else a.copy()

        ps = _PSet(**{r: to_ref(p0[s], w) for r, s, w in SH3_MAP})
        ps.alive = np.ones(n, bool)
        st = optimizer.MomentState(
            m={r: np.zeros((n,) if w == 1 else (n, w)) for r, _, w in SH3_MAP},
            v={r: np.zeros((n,) if w == 1 else (n, w)) for r, _, w in SH3_MAP},
            t={r: np.zeros(n, dtype=np.int64) for r, _, _ in SH3_MAP})
        cfg = optimizer.OptimizerConfig(
            mode=mode, lr_mu=LR_SH3["xyz"], lr_color=LR_SH3["f_dc"], lr_tau=LR_SH3["opacity"],
            lr_kappa=LR_SH3["scaling"], lr_rot=LR_SH3["rotation"], lambda_o=lambda_o,
            lambda_s=lambda_s, ct_opacity=ct, ct_scale=ct)
        cfg.lr_f_rest = LR_SH3["f_rest"]
        first = None
        for s in range(steps):
            g = gradients.ParamGrads(mu=None, kappa=None, rot=None, tau=None, color=None)
            for r, sh, w in SH3_MAP:
                setattr(g, r, to_ref(grads_seq[s][sh], w))
            if mode == "adamw-gs":
                optimizer.dar_step(st, ps, g, vis_seq[s], cfg, n_pixels, mu_lr_scale)
            elif mode == "sparse-adam":
                optimizer.sparse_adam_step(st, ps, g, vis_seq[s], cfg, mu_lr_scale)
            elif mode in ("adamw-const", "adamw-const-clip"):
                optimizer.adamw_const_step(st, ps, g, vis_seq[s], cfg, clip=clip,
                                           mu_lr_scale=mu_lr_scale)
            else:
                raise ValueError(mode)
            if s == 0:
                first = {sh: np.asarray(getattr(ps, r), np.float64).reshape(n, w).copy()
                         for r, sh, w in SH3_MAP}
        arrays = {}
        for r, sh, w in SH3_MAP:
            arrays[f"init_{sh}"] = p0[sh]
            arrays[f"grads_{sh}"] = np.stack([grads_seq[s][sh] for s in range(steps)])
            arrays[f"out_{sh}"] = np.asarray(getattr(ps, r), np.float64).reshape(n, w)
            arrays[f"first_{sh}"] = first[sh]
            arrays[f"m_{sh}"] = np.asarray(st.m[r], np.float64).reshape(n, w)
            arrays[f"v_{sh}"] = np.asarray(st.v[r], np.float64).reshape(n, w)
        for r, _, _ in SH3_MAP:
            assert np.array_equal(st.t[r], st.t["tau"])      # one clock
        arrays["t"] = st.t["tau"].copy()
        arrays["vis"] = vis_seq
        meta = dict(layout="sh3", mode=mode, n=n, steps=steps, seed=seed, lambda_o=lambda_o,
                    lambda_s=lambda_s, n_pixels=n_pixels, clip=clip, mu_lr_scale=mu_lr_scale,
                    ct_opacity=ct, ct_scale=ct, lr=LR_SH3, beta1=0.9, beta2=0.999, eps=1e-8)
        save(name, meta, arrays)
    finally:
        optimizer.ATTR_GROUPS, gradients.ATTR_GROUPS = saved


def run_ref2d_coupled(name, mode, n=24, steps=16, seed=5, p_vis=0.6, lambda_o=0.01,
                      lambda_s=0.01, mu_lr_scale=0.9):
    """Reference-native 2-D layout through the pipeline's coupled composite
    (pipeline.py:305-315): grads += coupled_reg_grad(...); then the step."""
    gradients, optimizer, primitives, loss = _import_reference()
    rng = np.random.default_rng(seed)
    p0 = {"mu": f32(rng.normal(0, 5, (n, 2))),
          "kappa": f32(rng.uniform(math.log(1e-3), math.log(0.5), (n, 2))),
          "rot": f32(rng.normal(0, 1, (n, 1))), "tau": f32(rng.normal(-1, 2, (n, 1))),
          "color": f32(rng.normal(0, 0.5, (n, 3)))}
    ps = primitives.PrimitiveSet(mu=p0["mu"], kappa=p0["kappa"], rot=p0["rot"][:, 0],
                                 tau=p0["tau"][:, 0], color=p0["color"], depth=np.zeros(n))
    st = optimizer.MomentState.zeros_like(ps)
    lr = {"mu": 0.029, "kappa": 5e-3, "rot": 1e-3, "tau": 0.05, "color": 2.5e-3}
    cfg = optimizer.OptimizerConfig(mode=mode, lr_mu=lr["mu"], lr_kappa=lr["kappa"],
                                    lr_rot=lr["rot"], lr_tau=lr["tau"], lr_color=lr["color"],
                                    lambda_o=lambda_o, lambda_s=lambda_s)
    vis_seq = rng.random((steps, n)) < p_vis
    vis_seq[:, 0] = True
    if mode == "sparse-adam":
        vis_seq[:, 1] = False
    grads_seq = [grads_for(rng, REF2D, vis_seq[s]) for s in range(steps)]
    for s in range(steps):
        g = gradients.ParamGrads(
            mu=grads_seq[s]["mu"].astype(np.float64), kappa=grads_seq[s]["kappa"].astype(np.float64),
            rot=grads_seq[s]["rot"][:, 0].astype(np.float64),
            tau=grads_seq[s]["tau"][:, 0].astype(np.float64),
            color=grads_seq[s]["color"].astype(np.float64))
        if mode == "sparse-adam":
            g_tau, g_kappa = loss.coupled_reg_grad(ps, vis_seq[s], lambda_o, lambda_s)
            g.tau += g_tau
            g.kappa += g_kappa
            optimizer.sparse_adam_step(st, ps, g, vis_seq[s], cfg, mu_lr_scale)
        elif mode == "coupled-adam":
            g_tau, g_kappa = loss.coupled_reg_grad(ps, vis_seq[s], lambda_o, lambda_s,
                                                   apply_to_all=True)
            g.tau += g_tau
            g.kappa += g_kappa
            optimizer.adam_step_sync(st, ps, g, cfg, mu_lr_scale)
        else:
            raise ValueError(mode)
    arrays = {"vis": vis_seq}
    for a, w in REF2D:
        arrays[f"init_{a}"] = p0[a]
        arrays[f"grads_{a}"] = np.stack([grads_seq[s][a] for s in range(steps)])
        arrays[f"out_{a}"] = np.asarray(getattr(ps, a), np.float64).reshape(n, w)
        arrays[f"m_{a}"] = np.asarray(st.m[a], np.float64).reshape(n, w)
        arrays[f"v_{a}"] = np.asarray(st.v[a], np.float64).reshape(n, w)
    arrays["t"] = st.t["tau"].copy()
    meta = dict(layout="ref2d", mode=mode, n=n, steps=steps, seed=seed, lambda_o=lambda_o,
                lambda_s=lambda_s, mu_lr_scale=mu_lr_scale, lr=lr, beta1=0.9, beta2=0.999,
                eps=1e-8, global_t=int(st.global_t))
    save(name, meta, arrays)


def run_rsr_stats(name="rsr_stats", n=64, seed=11):
    gradients, optimizer, primitives, loss = _import_reference()
    import splatlab.rng as ref_rng
    arrays, meta = {}, {"stss": []}
    # stss_sample index lists (bit-exact host RNG contract)
    cases = [(0, 10, 1000, 0.1), (7, 100, 6000, 0.25), (3, 770, 4096, 0.05), (0, 20, 64, 1.0),
             (123, 2500, 100_000, 0.25)]
    for i, (seed_, boundary, n_p, ratio) in enumerate(cases):
        sched = optimizer.StSSchedule(milestones=((0, ratio),), interval=10)
        idx = optimizer.stss_sample(sched, boundary, n_p, ref_rng.stream(seed_, "stss", boundary))
        arrays[f"stss_{i}"] = idx
        meta["stss"].append([seed_, boundary, n_p, ratio])
    # rsr_apply on a random REF2D state
    rng = np.random.default_rng(seed)
    st = optimizer.MomentState.zeros(n)
    for a in gradients.ATTR_GROUPS:
        st.m[a][:] = f32(rng.standard_normal(st.m[a].shape))
        st.v[a][:] = f32(rng.random(st.v[a].shape))
        st.t[a][:] = 9
    for a, w in REF2D:
        arrays[f"rsr_m0_{a}"] = f32(st.m[a]).reshape(n, w)
        arrays[f"rsr_v0_{a}"] = f32(st.v[a]).reshape(n, w)
    picked = np.sort(rng.choice(n, 20, replace=False))
    optimizer.rsr_apply(st, picked, 0.2, 0.04)
    arrays["rsr_idx"] = picked
    for a, w in REF2D:
        arrays[f"rsr_m1_{a}"] = np.asarray(st.m[a]).reshape(n, w)
        arrays[f"rsr_v1_{a}"] = np.asarray(st.v[a]).reshape(n, w)
    # moment_stats / classify_active on a random state with some zero-v rows
    st2 = optimizer.MomentState.zeros(n)
    for a in gradients.ATTR_GROUPS:
        st2.m[a][:] = f32(rng.standard_normal(st2.m[a].shape) * 1e-3)
        st2.v[a][:] = f32(rng.random(st2.v[a].shape) * 1e-6)
        st2.v[a][:5] = 0.0
    alive = rng.random(n) < 0.8
    ms = optimizer.moment_stats(st2, alive)
    for a, w in REF2D:
        arrays[f"ms_m_{a}"] = f32(st2.m[a]).reshape(n, w)
        arrays[f"ms_v_{a}"] = f32(st2.v[a]).reshape(n, w)
    arrays["ms_alive"] = alive
    meta["moment_stats"] = ms
    tau = f32(rng.normal(-5.5, 1.0, 4096))
    # pin fp32 neighbours of the threshold too
    thr = np.float32(math.log(1 / 254))
    near = [thr]
    for _ in range(8):
        near.append(np.nextafter(near[-1], np.float32(np.inf)))
    x = thr
    for _ in range(8):
        x = np.nextafter(x, np.float32(-np.inf))
        near.append(x)
    tau = np.concatenate([tau, np.array(near, np.float32)])
    ps = primitives.PrimitiveSet(mu=np.zeros((tau.size, 2)), kappa=np.zeros((tau.size, 2)),
                                 rot=np.zeros(tau.size), tau=tau.astype(np.float64),
                                 color=np.zeros((tau.size, 3)), depth=np.zeros(tau.size),
                                 alive=rng.random(tau.size) < 0.9)
    n_a, n_d, act = primitives.classify_active(ps)
    arrays["ca_tau"] = tau
    arrays["ca_alive"] = ps.alive
    arrays["ca_active"] = act
    meta["classify_active"] = [int(n_a), int(n_d)]
    meta["round_pixel_count"] = [[k, optimizer.round_pixel_count(k)]
                                 for k in (1024, 4096, 256, 999, 1, 9, 10, 1_000_000, 2_073_600,
                                           1_440_000, 65536)]
    save(name, meta, arrays)


def run_aiu(name="aiu", n=200, seed=21):
    """aiu_apply (optimizer.py:425-450) on the native 2-D layout."""
    gradients, optimizer, primitives, loss = _import_reference()
    rng = np.random.default_rng(seed)
    p0 = {"mu": f32(rng.normal(0, 5, (n, 2))),
          "kappa": f32(rng.uniform(math.log(1e-3), math.log(0.5), (n, 2))),
          "rot": f32(rng.normal(0, 1, (n, 1))), "tau": f32(rng.normal(-1, 2, (n, 1))),
          "color": f32(rng.normal(0, 0.5, (n, 3)))}
    alive = rng.random(n) < 0.9
    ps = primitives.PrimitiveSet(mu=p0["mu"], kappa=p0["kappa"], rot=p0["rot"][:, 0],
                                 tau=p0["tau"][:, 0], color=p0["color"], depth=np.zeros(n),
                                 alive=alive)
    st = optimizer.MomentState.zeros_like(ps)
    t = rng.integers(0, 40, n)                  # some rows never stepped (t = 0)
    m0, v0 = {}, {}
    for a, w in REF2D:
        m0[a] = f32(rng.standard_normal((n, w)) * 1e-3)
        v0[a] = f32(rng.random((n, w)) * 1e-6)
        st.m[a][:] = m0[a].reshape(st.m[a].shape)
        st.v[a][:] = v0[a].reshape(st.v[a].shape)
        st.t[a][:] = t
    vis = rng.random(n) < 0.4
    cfg = optimizer.OptimizerConfig()
    aiu = optimizer.AiuConfig(start=0, end=100, prob_schedule=((0, 0.3),),
                              eta_schedule=((0, 0.1),), enabled=True)
    draw_seed = 777
    picked = optimizer.aiu_apply(st, ps, vis, cfg, aiu, np.random.default_rng(draw_seed), 10)
    arrays = {"vis": vis, "alive": alive, "t": t.astype(np.int64), "picked": picked}
    for a, w in REF2D:
        arrays[f"init_{a}"] = p0[a]
        arrays[f"m_{a}"] = m0[a]
        arrays[f"v_{a}"] = v0[a]
        arrays[f"out_{a}"] = np.asarray(getattr(ps, a), np.float64).reshape(n, w)
    meta = dict(layout="ref2d", n=n, seed=seed, draw_seed=draw_seed, prob=0.3, eta=0.1,
                iteration=10, lr={"mu": cfg.lr_mu, "kappa": cfg.lr_kappa, "rot": cfg.lr_rot,
                                  "tau": cfg.lr_tau, "color": cfg.lr_color},
                beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps)
    save(name, meta, arrays)


def run_relocate(name="relocate", n=300, seed=41):
    """mcmc_relocate (pipeline.py:197-233) on the native 2-D layout: the
    reference draws the targets and rewrites the set; recorded before/after."""
    gradients, optimizer, primitives, loss = _import_reference()
    import splatlab.pipeline as pipeline
    rng = np.random.default_rng(seed)
    p0 = {"mu": f32(rng.normal(0, 5, (n, 2))),
          "kappa": f32(rng.uniform(math.log(1e-3), math.log(0.5), (n, 2))),
          "rot": f32(rng.normal(0, 1, (n, 1))), "tau": f32(rng.normal(0.0, 2.0, (n, 1))),
          "color": f32(rng.normal(0, 0.5, (n, 3)))}
    dead = rng.random(n) < 0.25                 # well below 1/255
    p0["tau"][dead, 0] = f32(rng.uniform(-12.0, -6.0, int(dead.sum())))
    alive = rng.random(n) < 0.95
    ps = primitives.PrimitiveSet(mu=p0["mu"].astype(np.float64),
                                 kappa=p0["kappa"].astype(np.float64),
                                 rot=p0["rot"][:, 0].astype(np.float64),
                                 tau=p0["tau"][:, 0].astype(np.float64),
                                 color=p0["color"].astype(np.float64), depth=np.zeros(n),
                                 alive=alive)
    st = optimizer.MomentState.zeros_like(ps)
    t = rng.integers(1, 40, n)
    m0, v0 = {}, {}
    for a, w in REF2D:
        m0[a] = f32(rng.standard_normal((n, w)) * 1e-3)
        v0[a] = f32(rng.random((n, w)) * 1e-6)
        st.m[a][:] = m0[a].reshape(st.m[a].shape)
        st.v[a][:] = v0[a].reshape(st.v[a].shape)
        st.t[a][:] = t
    draw_seed = 99
    out, out_st, events = pipeline.mcmc_relocate(ps, st, np.random.default_rng(draw_seed), 7)
    arrays = {"alive": alive, "t": t.astype(np.int64),
              "out_t": np.asarray(out_st.t["tau"], np.int64)}
    for a, w in REF2D:
        arrays[f"init_{a}"] = p0[a]
        arrays[f"m_{a}"] = m0[a]
        arrays[f"v_{a}"] = v0[a]
        arrays[f"out_{a}"] = np.asarray(getattr(out, a), np.float64).reshape(n, w)
        arrays[f"out_m_{a}"] = np.asarray(out_st.m[a], np.float64).reshape(n, w)
        arrays[f"out_v_{a}"] = np.asarray(out_st.v[a], np.float64).reshape(n, w)
    meta = dict(layout="ref2d", n=n, seed=seed, draw_seed=draw_seed,
                event_count=int(events[0]["count"]) if events else 0,
                event_hash=events[0]["affected_ids_hash"] if events else None)
    save(name, meta, arrays)


def run_densify(name="densify", n=240, seed=51):
    """densify_adc (pipeline.py:116-185) on the native 2-D layout: clone,
    split (with the reference's rng draws), prune; recorded before/after."""
    gradients, optimizer, primitives, loss = _import_reference()
    import splatlab.config as config
    import splatlab.pipeline as pipeline
    rng = np.random.default_rng(seed)
    p0 = {"mu": f32(rng.normal(0, 5, (n, 2))),
          "kappa": f32(rng.uniform(math.log(0.3), math.log(8.0), (n, 2))),
          "rot": f32(rng.normal(0, 1, (n, 1))), "tau": f32(rng.normal(0.0, 3.0, (n, 1))),
          "color": f32(rng.normal(0, 0.5, (n, 3)))}
    alive = rng.random(n) < 0.95
    depth = np.arange(n, dtype=np.float64)            # row identity through the transform
    ps = primitives.PrimitiveSet(mu=p0["mu"].astype(np.float64),
                                 kappa=p0["kappa"].astype(np.float64),
                                 rot=p0["rot"][:, 0].astype(np.float64),
                                 tau=p0["tau"][:, 0].astype(np.float64),
                                 color=p0["color"].astype(np.float64), depth=depth, alive=alive)
    st = optimizer.MomentState.zeros_like(ps)
    t = rng.integers(1, 40, n)
    m0, v0 = {}, {}
    for a, w in REF2D:
        m0[a] = f32(rng.standard_normal((n, w)) * 1e-3)
        v0[a] = f32(rng.random((n, w)) * 1e-6)
        st.m[a][:] = m0[a].reshape(st.m[a].shape)
        st.v[a][:] = v0[a].reshape(st.v[a].shape)
        st.t[a][:] = t
    accum = f32(rng.random(n) * 0.05).astype(np.float64)
    count = rng.integers(0, 4, n)
    stats = pipeline.DensifyStats(accum=accum.copy(), count=count.copy())
    cfg = config.DensifyConfig(grad_threshold=0.012, prune_opacity=0.005, split_scale_px=3.0,
                               split_shrink=1.6, max_primitives=2000)
    draw_seed = 1234
    out, out_st, events = pipeline.densify_adc(ps, st, stats, cfg, np.random.default_rng(draw_seed),
                                               iteration=5)
    arrays = {"alive": alive, "t": t.astype(np.int64), "accum": accum, "count": count,
              "out_alive": out.alive, "out_src": out.depth.astype(np.int64),
              "out_t": np.asarray(out_st.t["tau"], np.int64)}
    for a, w in REF2D:
        arrays[f"init_{a}"] = p0[a]
        arrays[f"m_{a}"] = m0[a]
        arrays[f"v_{a}"] = v0[a]
        arrays[f"out_{a}"] = np.asarray(getattr(out, a), np.float64).reshape(len(out), w)
        arrays[f"out_m_{a}"] = np.asarray(out_st.m[a], np.float64).reshape(len(out), w)
        arrays[f"out_v_{a}"] = np.asarray(out_st.v[a], np.float64).reshape(len(out), w)
    meta = dict(layout="ref2d", n=n, seed=seed, draw_seed=draw_seed, n_out=len(out),
                cfg=dict(grad_threshold=0.012, prune_opacity=0.005, split_scale_px=3.0,
                         split_shrink=1.6, max_primitives=2000),
                events=[{k: e[k] for k in ("kind", "count", "affected_ids_hash")} for e in events])
    save(name, meta, arrays)


if __name__ == "__main__":
    run_sh3_case("sh3_dar", "adamw-gs")
    run_sh3_case("sh3_dar_clip", "adamw-gs", seed=1, lambda_o=0.1, lambda_s=0.05, n_pixels=1024,
                 mu_lr_scale=0.7)
    run_sh3_case("sh3_sparse", "sparse-adam", seed=2)
    run_sh3_case("sh3_const", "adamw-const", seed=3, lambda_o=0.01, lambda_s=0.001)
    run_sh3_case("sh3_const_clip", "adamw-const-clip", seed=4, lambda_o=100.0, lambda_s=0.5,
                 clip=10.0)
    run_ref2d_coupled("ref2d_sparse_coupled", "sparse-adam")
    run_ref2d_coupled("ref2d_sync_coupled", "coupled-adam", seed=6, p_vis=0.7)
    run_rsr_stats()
    run_aiu()
    run_relocate()
    run_densify()
