"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The float64 restatement must reproduce the unmodified reference bit for
bit; the fp32 kernel-order restatement must stay within the north-star
tolerance (normwise 1e-6) of it.
"""

import math

import numpy as np
import pytest

from _golden import STEP_CASES, Case, normwise
from oracle import adamw_gs_oracle as O


def run_f64(case: Case):
    hp = case.hyper()
    p = case.init()
    m = {g.name: np.zeros((case.n, g.width)) for g in case.layout}
    v = {g.name: np.zeros((case.n, g.width)) for g in case.layout}
    t = np.zeros(case.n, np.int64)
    gt = 0
    meta = case.meta
    for s in range(case.steps):
        g = case.grads(s)
        vis = case.vis[s]
        mode = case.mode
        if mode == "adamw-gs":
            O.dar_step_f64(case.layout, p, g, m, v, t, vis, hp, meta["n_pixels"],
                           meta["mu_lr_scale"])
        elif mode == "sparse-adam":
            if case.layout is O.LAYOUT_REF2D:
                reg = O.coupled_reg_grad_f64(case.layout, p, vis, hp.lambda_o, hp.lambda_s)
                for k, r in reg.items():
                    g[k] = g[k] + r
            O.sparse_adam_step_f64(case.layout, p, g, m, v, t, vis, hp, meta["mu_lr_scale"])
        elif mode in ("adamw-const", "adamw-const-clip"):
            O.adamw_const_step_f64(case.layout, p, g, m, v, t, vis, hp, clip=meta["clip"],
                                   mu_lr_scale=meta["mu_lr_scale"])
        elif mode == "coupled-adam":
            reg = O.coupled_reg_grad_f64(case.layout, p, vis, hp.lambda_o, hp.lambda_s,
                                         apply_to_all=True)
            for k, r in reg.items():
                g[k] = g[k] + r
            gt = O.adam_step_sync_f64(case.layout, p, g, m, v, t, gt, hp, meta["mu_lr_scale"])
    return p, m, v, t


def coupled_lambdas(case: Case):
    """The coupled-regularization lambdas of the pipeline composite, if any."""
    if case.layout is O.LAYOUT_REF2D and case.mode in ("sparse-adam", "coupled-adam"):
        return {"lambda_o": case.meta["lambda_o"], "lambda_s": case.meta["lambda_s"]}
    return {}


def run_fp32(case: Case):
    hp = case.hyper()
    p = case.init(np.float32)
    m = {g.name: np.zeros((case.n, g.width), np.float32) for g in case.layout}
    v = {g.name: np.zeros((case.n, g.width), np.float32) for g in case.layout}
    clock = np.zeros(case.n, np.int32)
    meta = case.meta
    lut = O.bias_lut_f32(hp.beta1, hp.beta2, case.steps + 2)
    for s in range(case.steps):
        g = case.grads(s, np.float32)
        vis = case.vis[s]
        rows = np.flatnonzero(vis) if case.mode != "coupled-adam" else np.arange(case.n)
        O.step_fp32(case.mode, case.layout, p, g, m, v, clock, rows, hp,
                    n_pixels=meta.get("n_pixels"), mu_lr_scale=meta["mu_lr_scale"],
                    clip=meta.get("clip"), n_visible_norm=int(vis.sum()), global_t=s + 1,
                    lut=lut, **coupled_lambdas(case))
    return p, m, v, clock


@pytest.mark.parametrize("name", STEP_CASES)
def test_f64_restatement_is_bitwise_reference(name):
    case = Case(name)
    p, m, v, t = run_f64(case)
    out, em, ev, et = case.expected()
    for g in case.layout:
        assert np.array_equal(p[g.name], out[g.name]), g.name
        assert np.array_equal(m[g.name], em[g.name]), g.name
        assert np.array_equal(v[g.name], ev[g.name]), g.name
    assert np.array_equal(t, et)


@pytest.mark.parametrize("name", STEP_CASES)
def test_fp32_restatement_within_tolerance(name):
    """Tier (i) of SURVEY §7.3(1): normwise <= 1e-6 vs the f64 reference."""
    case = Case(name)
    p, m, v, clock = run_fp32(case)
    out, em, ev, et = case.expected()
    for g in case.layout:
        assert normwise(p[g.name], out[g.name]) <= 1e-6, g.name
        assert normwise(m[g.name], em[g.name]) <= 1e-6, g.name
        assert normwise(v[g.name], ev[g.name]) <= 1e-6, g.name
    assert np.array_equal(clock, et)


def test_stss_restatement_bit_exact():
    case = np.load(Case.__init__.__globals__["GOLDEN"] / "rsr_stats.npz")
    import json
    meta = json.loads(str(case["meta"]))
    for i, (seed, boundary, n_p, ratio) in enumerate(meta["stss"]):
        idx = O.stss_sample(((0, ratio),), boundary, n_p, O.rng_stream(seed, "stss", boundary))
        assert np.array_equal(idx, case[f"stss_{i}"])


def test_rsr_moment_stats_classify_round():
    import json
    z = np.load(Case.__init__.__globals__["GOLDEN"] / "rsr_stats.npz")
    meta = json.loads(str(z["meta"]))
    lay = O.LAYOUT_REF2D
    m = {g.name: z[f"rsr_m0_{g.name}"].astype(np.float64) for g in lay}
    v = {g.name: z[f"rsr_v0_{g.name}"].astype(np.float64) for g in lay}
    O.rsr_apply_f64(lay, m, v, z["rsr_idx"], 0.2, 0.04)
    for g in lay:
        assert np.array_equal(m[g.name], z[f"rsr_m1_{g.name}"])
        assert np.array_equal(v[g.name], z[f"rsr_v1_{g.name}"])
    ms = O.moment_stats_f64(lay, {g.name: z[f"ms_m_{g.name}"] for g in lay},
                            {g.name: z[f"ms_v_{g.name}"] for g in lay}, z["ms_alive"])
    for g in lay:
        for k, val in meta["moment_stats"][g.name].items():
            assert ms[g.name][k] == pytest.approx(val, rel=1e-15, abs=0), (g.name, k)
    n_a, n_d = O.classify_active_f64(z["ca_tau"], z["ca_alive"])
    assert [n_a, n_d] == meta["classify_active"]
    thr = O.active_logit_threshold_f32()
    act = z["ca_alive"] & (z["ca_tau"].astype(np.float32) > thr)
    assert np.array_equal(act, z["ca_active"])
    for k, want in meta["round_pixel_count"]:
        assert O.round_pixel_count(k) == want


def test_reference_known_answers_on_oracle():
    """Known answers of R/pkg/tests/test_optimizer.py restated on the oracle."""
    assert O.round_pixel_count(1024) == 100.0          # :69-74
    assert O.round_pixel_count(4096) == 400.0
    assert O.round_pixel_count(256) == 20.0
    assert O.round_pixel_count(999) == 90.0
    assert O.round_pixel_count(1024, enabled=False) == 1024.0
    term = min(0.001 * (0.25 / O.round_pixel_count(1024)) / (1e-4 + 1e-8), 10.0)   # :214-217
    assert term == pytest.approx(0.025, rel=1e-3)
    # clip engages at v_hat = 0 (:203-212), single tau row, fp32 kernel order
    lay = (O.Group("tau", 1, "opacity"),)
    hp = O.Hyper(lr={"tau": 1.0}, lambda_o=10.0, ct_opacity=10.0)
    p = {"tau": np.zeros((2, 1), np.float32)}
    z = {"tau": np.zeros((2, 1), np.float32)}
    m = {"tau": np.zeros((2, 1), np.float32)}
    v = {"tau": np.zeros((2, 1), np.float32)}
    st = O.step_fp32("adamw-gs", lay, p, z, m, v, np.zeros(2, np.int32), np.arange(2), hp,
                     n_pixels=100)
    assert np.allclose(-p["tau"], 10.0, rtol=1e-7)
    assert st["n_clip_opacity"] == 2


def test_sigmoid_threshold_is_exact_boundary():
    thr = O.active_logit_threshold_f32()
    s = O.sigmoid_f64(np.array([thr, np.nextafter(thr, np.float32(1))], np.float64))
    assert s[0] <= O.ACTIVE_OPACITY_THRESHOLD < s[1]
    assert abs(float(thr) - math.log(1 / 254)) < 1e-6


def test_aiu_f64_restatement_is_bitwise_reference():
    import json
    z = np.load(Case.__init__.__globals__["GOLDEN"] / "aiu.npz")
    meta = json.loads(str(z["meta"]))
    lay = O.LAYOUT_REF2D
    p = {g.name: z[f"init_{g.name}"].astype(np.float64) for g in lay}
    m = {g.name: z[f"m_{g.name}"].astype(np.float64) for g in lay}
    v = {g.name: z[f"v_{g.name}"].astype(np.float64) for g in lay}
    picked = O.aiu_apply_f64(lay, p, m, v, z["t"], z["vis"], z["alive"], meta["lr"],
                             meta["beta1"], meta["beta2"], meta["eps"], meta["prob"],
                             meta["eta"], np.random.default_rng(meta["draw_seed"]))
    assert np.array_equal(picked, z["picked"])
    for g in lay:
        assert np.array_equal(p[g.name], z[f"out_{g.name}"]), g.name


def test_relocate_f64_restatement_is_bitwise_reference():
    """mcmc_relocate (pipeline.py:197-233): the oracle restatement and the
    product's host plan (structural.mcmc_plan) against the reference run."""
    import json

    from paper_2601_16736_b200.structural import mcmc_plan
    z = np.load(Case.__init__.__globals__["GOLDEN"] / "relocate.npz")
    meta = json.loads(str(z["meta"]))
    lay = O.LAYOUT_REF2D
    p = {g.name: z[f"init_{g.name}"].astype(np.float64) for g in lay}
    m = {g.name: z[f"m_{g.name}"].astype(np.float64) for g in lay}
    v = {g.name: z[f"v_{g.name}"].astype(np.float64) for g in lay}
    t = z["t"].copy()
    dead = O.mcmc_relocate_f64(lay, p, m, v, t, z["alive"],
                               np.random.default_rng(meta["draw_seed"]))
    assert dead.size == meta["event_count"]
    for g in lay:
        assert np.array_equal(p[g.name], z[f"out_{g.name}"]), g.name
        assert np.array_equal(m[g.name], z[f"out_m_{g.name}"]), g.name
        assert np.array_equal(v[g.name], z[f"out_v_{g.name}"]), g.name
    assert np.array_equal(t, z["out_t"])
    plan = mcmc_plan(z["init_tau"], z["alive"], np.random.default_rng(meta["draw_seed"]))
    assert plan.count == meta["event_count"] and plan.ids_hash() == meta["event_hash"]
    assert np.array_equal(plan.dead, dead)
    assert np.array_equal(plan.tau_new, z["out_tau"][plan.dead, 0])


def test_densify_adc_f64_restatement_is_bitwise_reference():
    import json
    z = np.load(Case.__init__.__globals__["GOLDEN"] / "densify.npz")
    meta = json.loads(str(z["meta"]))
    lay = O.LAYOUT_REF2D
    p = {g.name: z[f"init_{g.name}"].astype(np.float64) for g in lay}
    m = {g.name: z[f"m_{g.name}"].astype(np.float64) for g in lay}
    v = {g.name: z[f"v_{g.name}"].astype(np.float64) for g in lay}
    out, om, ov, ot, alive, src, counts = O.densify_adc_f64(
        p, m, v, z["t"], z["alive"], z["accum"], z["count"], meta["cfg"],
        np.random.default_rng(meta["draw_seed"]))
    assert list(counts) == [e["count"] for e in meta["events"]]
    assert np.array_equal(src, z["out_src"]) and np.array_equal(alive, z["out_alive"])
    for g in lay:
        assert np.array_equal(out[g.name], z[f"out_{g.name}"]), g.name
        assert np.array_equal(om[g.name], z[f"out_m_{g.name}"]), g.name
        assert np.array_equal(ov[g.name], z[f"out_v_{g.name}"]), g.name
    assert np.array_equal(ot, z["out_t"])


@pytest.mark.parametrize("skip", [0, 1, 2, 3, 4, 9])
def test_philox_restatement_is_numpy_generator_random(skip):
    """oracle.philox_uniforms (NumPy's Philox4x64-10 + next_double, the
    reference's rng.stream, rng.py:17-30) reproduces Generator.random bit
    for bit from any buffer position: it pins the GPU AIU draw."""
    from paper_2601_16736_b200.sampling import stream
    rng = stream(3, "aiu", 17)
    rng.random(skip)
    st = rng.bit_generator.state
    want = rng.random(41)
    assert np.array_equal(O.philox_uniforms(st, 41), want)
