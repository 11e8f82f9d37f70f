"""The reference's own optimizer tests (R/pkg/tests/test_optimizer.py), run on
the B200 path through the reference-signature API, plus error semantics,
state ops and kernel-variant equivalence (marked gpu).

Each test cites the reference test it restates.  Tolerances widen from the
reference's float64 ones (1e-12..1e-15) to the fp32 contract of the north
star (1e-6 relative) where values are floating point; clocks, counts and
indices stay exact.
"""

import json

import numpy as np
import pytest
import torch

from _golden import GOLDEN
from oracle import adamw_gs_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
REF2D = (("mu", 2), ("kappa", 2), ("rot", 1), ("tau", 1), ("color", 3))


def small_set(rng, n=5, layout="rows"):
    """R/pkg/tests/conftest.py:18-33 restated on CUDA fp32 tensors."""
    from paper_2601_16736_b200.optimizer import MomentState
    span, inset = 16.0, 3.0
    o = rng.uniform(0.25, 0.7, size=n)
    p = {
        "mu": rng.uniform(inset, span - inset, size=(n, 2)),
        "kappa": np.log(rng.uniform(1.0, 3.0, size=(n, 2))),
        "rot": rng.uniform(0.0, np.pi, size=(n, 1)),
        "tau": np.log(o / (1 - o)).reshape(n, 1),
        "color": rng.uniform(0.1, 0.9, size=(n, 3)),
    }
    ps = {k: torch.tensor(v, dtype=torch.float32, device=DEV) for k, v in p.items()}
    st = MomentState.zeros_like(ps, layout)
    return ps, st


def make_grads(rng, n, scale=1.0):
    return {k: torch.tensor(rng.standard_normal((n, w)) * scale, dtype=torch.float32, device=DEV)
            for k, w in REF2D}


def zero_grads(n):
    return {k: torch.zeros((n, w), dtype=torch.float32, device=DEV) for k, w in REF2D}


def vis_t(mask):
    return torch.tensor(np.asarray(mask, bool), device=DEV)


LAYOUTS = ["rows", "groups"]


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


@pytest.mark.parametrize("layout", LAYOUTS)
class TestSyncAdam:
    def test_implicit_update_rescales_and_moves(self, rng, layout):   # :78-89
        from paper_2601_16736_b200.reference_api import OptimizerConfig, adam_step_sync
        ps, st = small_set(rng, 4, layout)
        st.m["tau"][:] = 0.5
        st.v["tau"][:] = 0.01
        st.clock[:] = 5
        st.global_t = 5
        tau0 = ps["tau"].clone()
        adam_step_sync(st, ps, zero_grads(4), OptimizerConfig())
        m = st.m["tau"].cpu().numpy()
        v = st.v["tau"].cpu().numpy()
        assert np.allclose(m, 0.9 * 0.5, rtol=1e-6)
        assert np.allclose(v, 0.999 * 0.01, rtol=1e-6)
        assert torch.all(ps["tau"] != tau0)

    def test_first_step_is_signlike(self, rng, layout):                # :91-99
        from paper_2601_16736_b200.reference_api import OptimizerConfig, adam_step_sync
        ps, st = small_set(rng, 3, layout)
        g = make_grads(rng, 3, scale=10.0)
        tau0 = ps["tau"].clone()
        adam_step_sync(st, ps, g, OptimizerConfig(lr_tau=0.1))
        got = (ps["tau"] - tau0).cpu().numpy()
        assert np.allclose(got, -0.1 * np.sign(g["tau"].cpu().numpy()), rtol=1e-6)

    def test_scalar_oracle_trace(self, rng, layout):                   # :101-112
        from paper_2601_16736_b200.reference_api import OptimizerConfig, adam_step_sync
        ps, st = small_set(rng, 1, layout)
        cfg = OptimizerConfig(lr_tau=0.1)
        theta0 = float(ps["tau"][0, 0])
        for gv in [1.0, -1.0, 1.0]:
            g = zero_grads(1)
            g["tau"][:] = gv
            adam_step_sync(st, ps, g, cfg)
        ref = theta0
        m = v = 0.0
        for t, gv in enumerate([1.0, -1.0, 1.0], 1):          # oracles.py:17-30
            m = 0.9 * m + 0.1 * gv
            v = 0.999 * v + 0.001 * gv * gv
            ref -= 0.1 * (m / (1 - 0.9 ** t)) / (np.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
        assert float(ps["tau"][0, 0]) == pytest.approx(ref, rel=1e-6)

    def test_nonfinite_gradient_aborts_with_ids(self, rng, layout):    # :114-121
        from paper_2601_16736_b200.reference_api import (GradientError, OptimizerConfig,
                                                         adam_step_sync)
        ps, st = small_set(rng, 4, layout)
        g = make_grads(rng, 4)
        g["kappa"][2, 1] = float("nan")
        before = {k: t.clone() for k, t in ps.items()}
        with pytest.raises(GradientError) as exc:
            adam_step_sync(st, ps, g, OptimizerConfig())
        assert 2 in exc.value.ids
        for k in ps:                                            # aborted before mutation
            assert torch.equal(ps[k], before[k])
        assert int(st.clock.sum()) == 0 and st.global_t == 0

    def test_pure_decay_of_zero_gradient_rows(self, rng, layout):      # :123-139
        from paper_2601_16736_b200.reference_api import OptimizerConfig, adam_step_sync
        ps, st = small_set(rng, 2, layout)
        m0, v0 = 0.37, 0.021
        st.m["tau"][:] = m0
        st.v["tau"][:] = v0
        for _ in range(50):
            adam_step_sync(st, ps, zero_grads(2), OptimizerConfig())
        assert np.allclose(st.m["tau"].cpu().numpy(), m0 * 0.9 ** 50, rtol=1e-6)
        assert np.allclose(st.v["tau"].cpu().numpy(), v0 * 0.999 ** 50, rtol=1e-6)


@pytest.mark.parametrize("layout", LAYOUTS)
class TestSparseAdam:
    def test_full_visibility_equals_sync(self, rng, layout):           # :143-156
        from paper_2601_16736_b200.reference_api import (MomentState, OptimizerConfig,
                                                         adam_step_sync, sparse_adam_step)
        ps_a, st_a = small_set(rng, 6, layout)
        ps_b = {k: t.clone() for k, t in ps_a.items()}
        st_b = MomentState.zeros_like(ps_b, layout)
        cfg = OptimizerConfig()
        g_rng = np.random.default_rng(0)
        vis = np.ones(6, bool)
        for _ in range(200):
            g = make_grads(g_rng, 6)
            adam_step_sync(st_a, ps_a, g, cfg)
            sparse_adam_step(st_b, ps_b, g, vis, cfg)
        for k in ps_a:
            # identical kernels on identical inputs: bitwise
            assert torch.equal(ps_a[k], ps_b[k])

    def test_invisible_rows_bitwise_frozen(self, rng, layout):         # :158-169
        from paper_2601_16736_b200.reference_api import OptimizerConfig, sparse_adam_step
        ps, st = small_set(rng, 5, layout)
        st.m["mu"][:] = torch.tensor(rng.standard_normal((5, 2)), dtype=torch.float32)
        before = {k: t.clone() for k, t in ps.items()}
        m_before = {k: t.clone() for k, t in st.m.items()}
        clock_before = st.clock.clone()
        vis = np.array([True, False, True, False, False])
        sparse_adam_step(st, ps, make_grads(rng, 5), vis, OptimizerConfig())
        frozen = torch.tensor(~vis, device=DEV)
        for k in ps:
            assert torch.equal(ps[k][frozen], before[k][frozen])
            assert torch.equal(st.m[k][frozen], m_before[k][frozen])
        assert torch.equal(st.clock[frozen], clock_before[frozen])

    def test_alternating_mask_matches_masked_oracle(self, rng, layout):  # :171-186
        from paper_2601_16736_b200.reference_api import OptimizerConfig, sparse_adam_step
        ps, st = small_set(rng, 1, layout)
        cfg = OptimizerConfig(lr_tau=0.05)
        theta0 = float(ps["tau"][0, 0])
        g_rng = np.random.default_rng(42)
        grads_seq = g_rng.standard_normal(50)
        mask_seq = g_rng.random(50) < 0.5
        for gv, mk in zip(grads_seq, mask_seq):
            g = zero_grads(1)
            g["tau"][:] = float(gv)
            sparse_adam_step(st, ps, g, np.array([mk]), cfg)
        m = v = 0.0
        t = 0
        theta = theta0
        for gv, mk in zip(grads_seq, mask_seq):                 # oracles.py:33-46
            if not mk:
                continue
            gv = float(np.float32(gv))
            t += 1
            m = 0.9 * m + 0.1 * gv
            v = 0.999 * v + 0.001 * gv * gv
            theta -= 0.05 * (m / (1 - 0.9 ** t)) / (np.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
        assert float(ps["tau"][0, 0]) == pytest.approx(theta, rel=1e-6, abs=1e-6)
        assert int(st.clock[0]) == t


@pytest.mark.parametrize("layout", LAYOUTS)
class TestDar:
    def test_denominator_dominance_keeps_plain_step(self, rng, layout):  # :190-201
        from paper_2601_16736_b200.reference_api import (MomentState, OptimizerConfig, dar_step,
                                                         sparse_adam_step)
        ps, st = small_set(rng, 3, layout)
        cfg = OptimizerConfig(mode="adamw-gs", lambda_o=0.001, lambda_s=1e-5)
        g = make_grads(rng, 3, scale=1e3)
        vis = np.ones(3, bool)
        ps_plain = {k: t.clone() for k, t in ps.items()}
        st_plain = MomentState.zeros_like(ps_plain, layout)
        dar_step(st, ps, g, vis, cfg, n_pixels=1024)
        sparse_adam_step(st_plain, ps_plain, g, vis, cfg)
        assert float((ps["tau"] - ps_plain["tau"]).abs().max()) < 1e-6

    def test_clip_engages_on_tiny_second_moment(self, rng, layout):  # :203-212
        from paper_2601_16736_b200.reference_api import OptimizerConfig, dar_step
        ps, st = small_set(rng, 2, layout)
        ps["tau"][:] = 0.0
        cfg = OptimizerConfig(mode="adamw-gs", lambda_o=10.0, ct_opacity=10.0, lr_tau=1.0)
        dar_step(st, ps, zero_grads(2), np.ones(2, bool), cfg, n_pixels=100)
        assert np.allclose(-ps["tau"].cpu().numpy(), 10.0, rtol=1e-7)

    def test_trace_matches_scalar_oracle(self, rng, layout):          # :219-240
        from paper_2601_16736_b200.reference_api import OptimizerConfig, dar_step
        ps, st = small_set(rng, 1, layout)
        cfg = OptimizerConfig(mode="adamw-gs", lambda_o=0.001, lr_tau=0.05, ct_opacity=10.0)
        theta0 = float(ps["tau"][0, 0])
        g_rng = np.random.default_rng(9)
        grads_seq = g_rng.standard_normal(60) * 0.01
        mask_seq = g_rng.random(60) < 0.7
        for gv, mk in zip(grads_seq, mask_seq):
            g = zero_grads(1)
            g["tau"][:] = float(gv)
            dar_step(st, ps, g, np.array([mk]), cfg, n_pixels=1024)

        def reg(tau):
            o = O.sigmoid_f64(np.array([tau]))[0]
            return o * (1 - o)
        ref, *_ = scalar_dar(theta0, [float(np.float32(x)) for x in grads_seq], mask_seq,
                             lr=0.05, lam=0.001, reg_grad=reg, n_pixels_rounded=100.0, ct=10.0)
        assert float(ps["tau"][0, 0]) == pytest.approx(ref, rel=1e-6)

    def test_decoupling_invariant(self, rng, layout):                 # :242-254
        from paper_2601_16736_b200.reference_api import OptimizerConfig, dar_step
        ps, st = small_set(rng, 4, layout)
        cfg = OptimizerConfig(mode="adamw-gs", lambda_o=0.001)
        vis = np.ones(4, bool)
        tau_prev = ps["tau"].clone()
        for _ in range(20):
            dar_step(st, ps, zero_grads(4), vis, cfg, n_pixels=4096)
            assert torch.all(ps["tau"] < tau_prev)
            tau_prev = ps["tau"].clone()
        assert torch.all(st.m["tau"] == 0.0)
        assert torch.all(st.v["tau"] == 0.0)

    def test_bad_clip_rejected(self, rng, layout):                    # :256-262
        from paper_2601_16736_b200.reference_api import ConfigError, OptimizerConfig, dar_step
        ps, st = small_set(rng, 1, layout)
        cfg = OptimizerConfig(mode="adamw-gs")
        cfg.ct_opacity = -1.0
        with pytest.raises(ConfigError):
            dar_step(st, ps, zero_grads(1), np.ones(1, bool), cfg, n_pixels=64)

    def test_domain_error_on_visible_kappa(self, rng, layout):        # primitives.py:78-84
        from paper_2601_16736_b200.reference_api import DomainError, OptimizerConfig, dar_step
        ps, st = small_set(rng, 4, layout)
        ps["kappa"][1, 0] = 81.0
        cfg = OptimizerConfig(mode="adamw-gs", lambda_s=1e-5)
        before = {k: t.clone() for k, t in ps.items()}
        with pytest.raises(DomainError) as exc:
            dar_step(st, ps, make_grads(rng, 4), np.ones(4, bool), cfg, n_pixels=1024)
        assert list(exc.value.ids) == [1]
        for k in ps:
            assert torch.equal(ps[k], before[k])
        # invisible out-of-domain rows are not an error
        vis = np.array([True, False, True, True])
        dar_step(st, ps, make_grads(rng, 4), vis, cfg, n_pixels=1024)

    def test_gradient_error_on_invisible_row(self, rng, layout):      # gradients.py:50-58
        from paper_2601_16736_b200.reference_api import GradientError, OptimizerConfig, dar_step
        ps, st = small_set(rng, 4, layout)
        g = make_grads(rng, 4)
        g["color"][3, 2] = float("inf")
        with pytest.raises(GradientError) as exc:
            dar_step(st, ps, g, np.array([True, True, False, False]), OptimizerConfig(
                mode="adamw-gs"), n_pixels=1024)
        assert list(exc.value.ids) == [3]


def scalar_dar(theta, grads, visible, lr, lam, reg_grad, n_pixels_rounded, ct, beta1=0.9,
               beta2=0.999, eps=1e-8):
    """R/pkg/tests/oracles.py:49-69 restated (independent scalar loop)."""
    m = v = 0.0
    t = 0
    for g, vis in zip(grads, visible):
        if not vis:
            continue
        t += 1
        m = beta1 * m + (1.0 - beta1) * g
        v = beta2 * v + (1.0 - beta2) * g * g
        m_hat = m / (1.0 - beta1 ** t)
        v_hat = v / (1.0 - beta2 ** t)
        denom = np.sqrt(v_hat) + eps
        extra = min(lam * (reg_grad(theta) / n_pixels_rounded) / denom, ct)
        theta = theta - lr * (m_hat / denom + extra)
    return theta, m, v, t


@pytest.mark.parametrize("layout", LAYOUTS)
class TestAdamwConst:
    def test_zero_lambda_equals_sparse(self, rng, layout):            # :266-279
        from paper_2601_16736_b200.reference_api import (MomentState, OptimizerConfig,
                                                         adamw_const_step, sparse_adam_step)
        ps_a, st_a = small_set(rng, 4, layout)
        ps_b = {k: t.clone() for k, t in ps_a.items()}
        st_b = MomentState.zeros_like(ps_b, layout)
        cfg = OptimizerConfig(mode="adamw-const", lambda_o=0.0, lambda_s=0.0)
        g_rng = np.random.default_rng(3)
        for _ in range(50):
            g = make_grads(g_rng, 4)
            vis = g_rng.random(4) < 0.6
            adamw_const_step(st_a, ps_a, g, vis, cfg)
            sparse_adam_step(st_b, ps_b, g, vis, cfg)
        for k in ps_a:   # one op order in both modes: bitwise over the whole set
            assert torch.equal(ps_a[k], ps_b[k])

    def test_uniform_pressure(self, rng, layout):                     # :281-298
        from paper_2601_16736_b200.reference_api import (MomentState, OptimizerConfig,
                                                         adamw_const_step, sparse_adam_step)
        ps, st = small_set(rng, 3, layout)
        ps["tau"][:] = 0.3
        cfg = OptimizerConfig(mode="adamw-const", lambda_o=0.1, lr_tau=1.0)
        g = zero_grads(3)
        g["tau"][:, 0] = torch.tensor([1.0, -2.0, 0.0])
        vis = np.ones(3, bool)
        ps_ref = {k: t.clone() for k, t in ps.items()}
        st_ref = MomentState.zeros_like(ps_ref, layout)
        sparse_adam_step(st_ref, ps_ref, g, vis, OptimizerConfig(mode="sparse-adam", lr_tau=1.0))
        o = 1 / (1 + np.exp(-np.float64(np.float32(0.3))))
        extra = 0.1 * o * (1 - o)
        adamw_const_step(st, ps, g, vis, cfg)
        # difference of two fp32 parameters near 1: absolute resolution ~1e-7
        assert np.allclose((ps_ref["tau"] - ps["tau"]).cpu().numpy(), extra, rtol=1e-6, atol=5e-7)

    def test_clip_applies(self, rng, layout):                         # :300-308
        from paper_2601_16736_b200.reference_api import OptimizerConfig, adamw_const_step
        ps, st = small_set(rng, 2, layout)
        ps["tau"][:] = 0.0
        cfg = OptimizerConfig(mode="adamw-const-clip", lambda_o=100.0, lr_tau=1.0)
        adamw_const_step(st, ps, zero_grads(2), np.ones(2, bool), cfg, clip=10.0)
        assert np.allclose(-ps["tau"].cpu().numpy(), 10.0, rtol=1e-7)


@pytest.mark.parametrize("layout", LAYOUTS)
class TestRsrResetStats:
    def test_defaults_scale_moments_exactly(self, layout):            # :333-341
        from paper_2601_16736_b200.reference_api import MomentState, rsr_apply
        st = MomentState.zeros_like({k: torch.zeros((4, w), device=DEV) for k, w in REF2D},
                                    layout)
        st.m["tau"][:] = 0.5
        st.v["tau"][:] = 0.01
        st.clock[:] = 7
        rsr_apply(st, np.arange(4), 0.2, 0.04)
        assert torch.all(st.m["tau"] == np.float32(0.5 * 0.2))
        assert torch.all(st.v["tau"] == np.float32(np.float32(0.01) * 0.04))
        assert torch.all(st.clock == 7)

    def test_zero_factors_equal_fresh_and_selected_rows_only(self, rng, layout):  # :343-371
        from paper_2601_16736_b200.reference_api import MomentState, rsr_apply
        st = MomentState.zeros_like({k: torch.zeros((5, w), device=DEV) for k, w in REF2D},
                                    layout)
        st.m["mu"][:] = 1.0
        rsr_apply(st, np.array([1, 3]), 0.2, 0.04)
        m = st.m["mu"].cpu().numpy()
        assert np.all(m[[0, 2, 4]] == 1.0) and np.all(m[[1, 3]] == np.float32(0.2))
        rsr_apply(st, np.arange(5), 0.0, 0.0)
        for k in st.m:
            assert torch.all(st.m[k] == 0) and torch.all(st.v[k] == 0)

    def test_rsr_golden(self, layout):
        from paper_2601_16736_b200.reference_api import MomentState, rsr_apply
        z = np.load(GOLDEN / "rsr_stats.npz")
        st = MomentState.zeros_like({k: torch.zeros((64, w), device=DEV) for k, w in REF2D},
                                    layout)
        for k, _ in REF2D:
            st.m[k][:] = torch.from_numpy(z[f"rsr_m0_{k}"])
            st.v[k][:] = torch.from_numpy(z[f"rsr_v0_{k}"])
        rsr_apply(st, z["rsr_idx"], 0.2, 0.04)
        for k, _ in REF2D:
            assert np.array_equal(st.m[k].cpu().numpy(), z[f"rsr_m1_{k}"].astype(np.float32))
            assert np.array_equal(st.v[k].cpu().numpy(), z[f"rsr_v1_{k}"].astype(np.float32))

    def test_reset_then_first_step_uses_raw_gradient(self, rng, layout):  # :533-547
        from paper_2601_16736_b200.reference_api import (OptimizerConfig, reset_rows,
                                                         sparse_adam_step)
        ps, st = small_set(rng, 2, layout)
        cfg = OptimizerConfig(lr_tau=0.05)
        for _ in range(10):
            sparse_adam_step(st, ps, make_grads(rng, 2), np.ones(2, bool), cfg)
        reset_rows(st, np.array([0]))
        assert int(st.clock[0]) == 0 and int(st.clock[1]) == 10
        g = zero_grads(2)
        g["tau"][:] = 0.5
        tau0 = ps["tau"].clone()
        sparse_adam_step(st, ps, g, np.ones(2, bool), cfg)
        step0 = float(tau0[0, 0] - ps["tau"][0, 0])
        assert step0 == pytest.approx(0.05 * 0.5 / (0.5 + cfg.eps), rel=1e-6)

    def test_moment_stats_golden_and_known(self, layout):              # :567-582
        from paper_2601_16736_b200.reference_api import MomentState, moment_stats
        z = np.load(GOLDEN / "rsr_stats.npz")
        meta = json.loads(str(z["meta"]))
        st = MomentState.zeros_like({k: torch.zeros((64, w), device=DEV) for k, w in REF2D},
                                    layout)
        for k, _ in REF2D:
            st.m[k][:] = torch.from_numpy(z[f"ms_m_{k}"])
            st.v[k][:] = torch.from_numpy(z[f"ms_v_{k}"])
        out = moment_stats(st, z["ms_alive"])
        for k, _ in REF2D:
            for f, want in meta["moment_stats"][k].items():
                assert out[k][f] == pytest.approx(want, rel=1e-12), (k, f)
        st2 = MomentState.zeros_like({k: torch.zeros((2, w), device=DEV) for k, w in REF2D},
                                     layout)
        st2.m["tau"][:, 0] = torch.tensor([0.3, -0.6])
        st2.v["tau"][:, 0] = torch.tensor([0.09, 0.04])
        o = moment_stats(st2, None)["tau"]
        assert o["mean_sqrt_v"] == pytest.approx(0.25, rel=1e-6)
        assert o["max_sqrt_v"] == pytest.approx(0.3, rel=1e-6)
        assert o["mean_abs_m_over_sqrt_v"] == pytest.approx(2.0, rel=1e-6)
        assert o["max_abs_m_over_sqrt_v"] == pytest.approx(3.0, rel=1e-6)


def test_classify_active_golden():
    from paper_2601_16736_b200.reference_api import classify_active
    z = np.load(GOLDEN / "rsr_stats.npz")
    meta = json.loads(str(z["meta"]))
    tau = torch.from_numpy(z["ca_tau"].astype(np.float32)).to(DEV)
    n_a, n_d, _ = classify_active({"tau": tau}, alive=z["ca_alive"])
    assert [n_a, n_d] == meta["classify_active"]


@pytest.mark.parametrize("check", ["fused", "strict"])
def test_optimizer_error_semantics(check):
    """Fused: bad rows skipped, others stepped, error raised after.
    Strict: nothing mutated (optimizer.py:248 aborts before mutation)."""
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS, GradientError
    cfg = S.WorkloadConfig(n=5000, p_vis=0.5, seed=2)
    host = S.make_params(cfg)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5,
                  check=check, errors="raise")
    vis = S.visibility(cfg, 0)
    g = {k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, 0, vis).items()}
    bad_row = int(np.flatnonzero(vis)[7])
    g["f_rest"][bad_row, 11] = float("nan")
    before = {k: t.clone() for k, t in params.items()}
    with pytest.raises(GradientError) as exc:
        opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, grads=g)
    assert list(exc.value.ids) == [bad_row]
    clock = opt.state.clock.cpu().numpy()
    if check == "strict":
        assert clock.sum() == 0
        for k in params:
            assert torch.equal(params[k], before[k])
    else:
        want = vis.astype(np.int32)
        want[bad_row] = 0
        assert np.array_equal(clock, want)
        for k in params:
            assert torch.equal(params[k][bad_row], before[k][bad_row])
        st = opt.last_stats()
        assert st["n_bad_grad"] == 1 and st["n_stepped"] == int(vis.sum()) - 1


@pytest.mark.parametrize("mode", ["adamw-gs", "sparse-adam", "adamw-const-clip",
                                  "coupled-adam"])
@pytest.mark.parametrize("check", ["fused", "strict"])
def test_step_kernels_all_identical(mode, check):
    """Every K2 implementation, tuning variant and parameter layout gives the
    same bits: the fixed-layout SH-3 kernels (2-D TMA, cp.async ring,
    per-attribute gathers, plus the measured alternatives when built), the
    generic row-record kernel (variants 0..6) and the per-group-state kernel, with
    per-attribute tensors, with parameters and gradients as views of
    row-interleaved records (records.py), and with only the parameters in a
    record (strided gathers)."""
    from paper_2601_16736_b200 import _lib
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    lib = _lib.load()
    cfg = S.WorkloadConfig(n=20_011, p_vis=0.4, seed=9)
    host = S.make_params(cfg)
    results = []
    runs = [("fixed", 0, "attr")] + [("rows", v, "attr") for v in range(7)]
    runs += [("groups", 0, "attr")]
    # record layouts: fixed 0 = the 2-D TMA gather4 / scatter4 kernel, 21 = the
    # cp.async ring kernel; "param-record" = only the parameters in a record
    runs += [(k, 0, lay) for k in ("fixed", "rows", "groups") for lay in ("record", "param-record")]
    runs += [("fixed", 21, "record")]
    if lib.gs_build_flags() & 1:  # measured alternatives compiled in (-DGS_BUILD_VARIANTS=1)
        runs += [("fixed", v, "attr") for v in (1, 2, 3, 4, 5, 6, 7, 19)]
        runs += [("fixed", v, "record") for v in (8, 9, 10, 11, 12, 13, 14, 16, 17, 18, 19, 20)]
    runs += [(k, 0, "record240") for k in ("fixed", "rows")]  # compact 240-byte rows
    if check == "strict":
        runs = [r for r in runs if r[1] in (0, 3, 7, 8, 11, 12, 21)]
    prev_f = lib.gs_set_fixed_variant(0)
    prev_r = lib.gs_set_rows_variant(0)
    try:
        for kind, variant, lay in runs:
            lib.gs_set_fixed_variant(variant if kind == "fixed" else -1)
            lib.gs_set_rows_variant(variant if kind == "rows" else 0)
            params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
            if lay != "attr":
                _, params = R.pack(params, align=4 if lay == "record240" else 16)
            layout = "groups" if kind == "groups" else "rows"
            opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=1e-3, lambda_s=1e-5,
                          state_layout=layout, check=check)
            for s in range(3):
                vis = S.visibility(cfg, s)
                g = {k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, s, vis).items()}
                if lay in ("record", "record240"):
                    _, g = R.pack(g, align=4 if lay == "record240" else 16)
                opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, grads=g)
            results.append(({k: p.cpu().numpy() for k, p in params.items()},
                            {k: t.contiguous().cpu().numpy() for k, t in opt.state.m.items()},
                            {k: t.contiguous().cpu().numpy() for k, t in opt.state.v.items()},
                            opt.state.clock.contiguous().cpu().numpy(), opt.last_stats()))
    finally:
        lib.gs_set_fixed_variant(prev_f)
        lib.gs_set_rows_variant(prev_r)
    ref = results[0]
    for run, res in zip(runs[1:], results[1:]):
        for i in range(3):
            for k in ref[i]:
                assert np.array_equal(res[i][k], ref[i][k]), (run, i, k)
        assert np.array_equal(res[3], ref[3]), run
        for f, x in ref[4].items():
            if f == "n_runs":  # layout hint: depends on the kernel's chunking
                continue
            if f.startswith("sum_"):
                assert res[4][f] == pytest.approx(x, rel=1e-12), (run, f)
            else:
                assert res[4][f] == x, (run, f)


def test_record_params_autograd_grad_and_state_ops():
    """Attribute views of a leaf record: backward fills record.grad, step()
    picks the matching view of it; AIU, stats, noise and the error paths
    work on the strided views, bitwise equal to per-attribute tensors."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.noise import NoiseConfig
    from paper_2601_16736_b200.optimizer import AdamWGS
    from paper_2601_16736_b200.sampling import AiuConfig
    cfg = S.WorkloadConfig(n=10_007, p_vis=0.3, seed=21)
    host = S.make_params(cfg)
    outs = []
    for lay in ("attr", "record"):
        params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
        if lay == "record":
            rec, params = R.pack(params, requires_grad=True)
        opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
        for s in range(3):
            vis = S.visibility(cfg, s)
            g = S.step_grads(cfg, s, vis)
            if lay == "record":
                # a toy loss whose gradient w.r.t. each view is the synthetic gradient
                rec.grad = None
                loss = sum((params[k] * torch.from_numpy(x).to(DEV).view(params[k].shape)).sum()
                           for k, x in g.items())
                loss.backward()
                opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels)
            else:
                opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels,
                         grads={k: torch.from_numpy(x).to(DEV) for k, x in g.items()})
        vis = torch.from_numpy(S.visibility(cfg, 7)).to(DEV)
        aiu = AiuConfig(start=0, end=100, prob_schedule=((0, 0.2),), eta_schedule=((0, 0.5),),
                        enabled=True)
        picked = opt.aiu_apply(vis, aiu, np.random.default_rng(3), 5)
        opt.noise_perturb(1e-3, NoiseConfig(enabled=True), seed=11, iteration=5)
        stats = opt.moment_stats()
        act = opt.classify_active()
        torch.cuda.synchronize()
        outs.append(({k: p.detach().cpu().numpy() for k, p in params.items()},
                     opt.state.record.cpu().numpy(), picked, stats, act))
    a, b = outs
    for k in a[0]:
        assert np.array_equal(a[0][k], b[0][k]), k
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])
    assert repr(a[3]) == repr(b[3]) and repr(a[4]) == repr(b[4])


def test_state_views_and_checkpoint_roundtrip():
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg = S.WorkloadConfig(n=3000, p_vis=0.5, seed=5)
    host = S.make_params(cfg)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    params["f_rest"] = params["f_rest"].view(-1, 15, 3)   # 3DGS shape (N, 15, 3)
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
    vis = S.visibility(cfg, 0)
    g = {k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, 0, vis).items()}
    g["f_rest"] = g["f_rest"].view(-1, 15, 3)
    opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, grads=g)
    st = opt.state
    assert st.m["f_rest"].shape == (3000, 15, 3)
    rec = st.record.cpu().numpy()
    # element 6 + 3*c + k of the record is f_rest[c, k]
    assert np.array_equal(st.m["f_rest"][:, 4, 2].cpu().numpy(), rec[:, 2 * (6 + 4 * 3 + 2)])
    assert np.array_equal(st.clock.cpu().numpy(), vis.astype(np.int32))
    sd = opt.state_dict()
    opt2 = AdamWGS(S.param_groups({k: p.clone() for k, p in params.items()}), mode="adamw-gs")
    opt2.load_state_dict(sd)
    assert torch.equal(opt2.state.record, opt.state.record)


@pytest.mark.parametrize("check", ["fused", "strict"])
@pytest.mark.parametrize("layout", ["attr", "record"])
def test_pinned_host_grads_zero_copy_identical(check, layout):
    """Gradients in pinned host memory are read zero-copy by the kernel and
    give bitwise the same step as device-resident gradients: per-attribute
    tensors (gather kernel) and a pinned gradient record with device
    parameter records (ring kernel, L1-allocating host copies)."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.engine import ConfigError
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg = S.WorkloadConfig(n=20_003, p_vis=0.3, seed=4)
    host = S.make_params(cfg)
    outs = []
    for where in ("device", "pinned"):
        params = {k: torch.from_numpy(v).to("cuda:0") for k, v in host.items()}
        if layout == "record":
            _, params = R.pack(params)
        opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5,
                      check=check)
        for s in range(3):
            vis = S.visibility(cfg, s)
            g = S.step_grads(cfg, s, vis)
            if where == "device":
                grads = {k: torch.from_numpy(x).to("cuda:0") for k, x in g.items()}
                if layout == "record":
                    grads = R.pack(grads)[1]
            elif layout == "record":
                grads = R.pack({k: torch.from_numpy(x) for k, x in g.items()},
                               pin_memory=True)[1]
            else:
                grads = {k: torch.from_numpy(x).pin_memory() for k, x in g.items()}
            opt.step(torch.from_numpy(vis).to("cuda:0"), cfg.n_pixels, grads=grads)
        torch.cuda.synchronize()
        outs.append(({k: v.cpu() for k, v in params.items()}, opt.state.record.cpu()))
    for k in outs[0][0]:
        assert torch.equal(outs[0][0][k], outs[1][0][k]), k
    assert torch.equal(outs[0][1], outs[1][1])
    # pageable host memory is refused, not silently copied
    with pytest.raises(ConfigError):
        opt.step(torch.from_numpy(vis).to("cuda:0"), cfg.n_pixels,
                 grads={k: torch.from_numpy(x) for k, x in g.items()})


@pytest.mark.parametrize("mode", ["adamw-gs", "sparse-adam"])
@pytest.mark.parametrize("check", ["fused", "strict"])
def test_captured_step_graph_matches_eager(mode, check):
    """AdamWGS.capture: K1 + K2 (+ strict check) replayed as one CUDA graph
    over refilled static buffers gives bitwise the eager steps, and a bad
    gradient still raises GradientError with its row after the replay."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.engine import ConfigError, GradientError
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg = S.WorkloadConfig(n=30_001, p_vis=0.3, seed=31)
    host = S.make_params(cfg)
    outs = []
    for how in ("eager", "graph"):
        _, params = R.pack({k: torch.from_numpy(v).to(DEV) for k, v in host.items()})
        opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=1e-3, lambda_s=1e-5,
                      check=check, errors="raise")
        grec, grads = R.pack({k: torch.zeros(v.shape, device=DEV) for k, v in host.items()})
        vis_buf = torch.zeros(cfg.n, dtype=torch.bool, device=DEV)
        graph = opt.capture(vis_buf, cfg.n_pixels, grads=grads) if how == "graph" else None
        for s in range(4):
            vis = S.visibility(cfg, s)
            g = S.step_grads(cfg, s, vis)
            vis_buf.copy_(torch.from_numpy(vis))
            for k, x in g.items():
                grads[k].copy_(torch.from_numpy(x).view(grads[k].shape))
            if graph is None:
                opt.step(vis_buf, cfg.n_pixels, grads=grads)
            else:
                graph.replay()
        torch.cuda.synchronize()
        outs.append(({k: p.cpu().numpy() for k, p in params.items()},
                     opt.state.record.cpu().numpy(), opt.last_stats()))
        if graph is not None:
            assert graph.launches_per_replay >= 1
            bad = int(np.flatnonzero(vis)[5])
            grads["f_rest"][bad, 2] = float("nan")
            with pytest.raises(GradientError) as ei:
                graph.replay()
            assert bad in ei.value.ids.tolist()
    a, b = outs
    for k in a[0]:
        assert np.array_equal(a[0][k], b[0][k]), k
    assert np.array_equal(a[1], b[1])
    assert a[2] == b[2]
    with pytest.raises(ConfigError):
        AdamWGS(S.param_groups({k: torch.from_numpy(v).to(DEV) for k, v in host.items()}),
                mode="coupled-adam").capture(vis_buf, None)
