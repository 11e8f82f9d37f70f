"""Multi-step parity at the BASELINE configurations C2, C3 and C4, with the
reference's boundary events interleaved between steps (marked gpu).

The loop is run_training's (pipeline.py:300-370): a step per iteration;
on boundaries RSR (stss_sample + rsr_apply, :365-370), random state resets
and MCMC relocation (mcmc_relocate -> reset_rows, :346-349, :229).  The GPU
runs every row through the product path (records, the default kernels);
the oracles follow a sample of rows:

* ``step_fp32`` (the kernels' fp32 order): bit-exact on every sampled row;
* the float64 restatement of the reference (``*_f64``, pinned to the
  reference's golden vectors): normwise max|d|/max|ref| <= 1e-6 per tensor.

Rows are independent, so a row sample is an exact
sub-problem; the events are applied to the sampled rows they touch.  The
sample holds >= 64k uniform rows, the first and last row, every row a reset
touches and every relocated row with its target.  Every RSR event is also
checked on ALL the rows it picked (before/after, bit-exact).  Inputs (cloud,
gradients, masks) are generated on the device and the sampled rows are read
back, so the oracles see exactly the GPU's inputs.
"""

import numpy as np
import pytest
import torch

from _golden import normwise
from oracle import adamw_gs_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
NORM_TOL = 1e-6


def _rows_of(t: torch.Tensor, idx: torch.Tensor) -> np.ndarray:
    return t.index_select(0, idx).cpu().numpy()


def _run(n, mode, steps, *, p=0.3, lo=1e-3, ls=1e-5, rsr_every=0, rsr_ratio=0.25,
         reset_every=0, reset_frac=0.02, relocate_every=0, sample=65_536, seed=0):
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    from paper_2601_16736_b200.sampling import StSSchedule, stream, stss_sample
    from paper_2601_16736_b200.structural import mcmc_plan

    dev = torch.device(DEV)
    cfg = S.WorkloadConfig(n=n, p_vis=p, seed=seed, lambda_o=lo, lambda_s=ls)
    lay = O.LAYOUT_SH3
    names = [g.name for g in lay]
    _, params = R.pack(S.make_params_device(cfg, dev))
    grec, gviews = R.pack({k: torch.zeros_like(v) for k, v in params.items()})
    opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=lo, lambda_s=ls, errors="raise")
    hp = O.Hyper(lr=S.LR_SH3, lambda_o=lo, lambda_s=ls)

    # boundary events (drawn up front from the reference's RNG contract)
    resets = {}
    if reset_every:
        for b in range(reset_every, steps + 1, reset_every):
            rng = stream(seed, "reset", b)
            resets[b] = np.sort(rng.choice(n, int(reset_frac * n), replace=False))
    sched = StSSchedule(milestones=((0, rsr_ratio),), interval=max(rsr_every, 1))
    rsr = {b: stss_sample(sched, b, n, stream(seed, "stss", b))
           for b in range(rsr_every, steps + 1, rsr_every)} if rsr_every else {}

    rng = np.random.default_rng(seed + 99)
    samp = set(rng.choice(n, sample, replace=False).tolist()) | {0, n - 1}
    for r in resets.values():
        samp |= set(r.tolist())
    samp = np.array(sorted(samp), np.int64)
    pos = {int(r): i for i, r in enumerate(samp)}
    idx_t = torch.from_numpy(samp).to(dev)
    ns = samp.size

    p32 = {k: _rows_of(params[k], idx_t).reshape(ns, -1).astype(np.float32) for k in names}
    p64 = {k: x.astype(np.float64) for k, x in p32.items()}
    m32 = {g.name: np.zeros((ns, g.width), np.float32) for g in lay}
    v32 = {g.name: np.zeros((ns, g.width), np.float32) for g in lay}
    m64 = {g.name: np.zeros((ns, g.width)) for g in lay}
    v64 = {g.name: np.zeros((ns, g.width)) for g in lay}
    c32 = np.zeros(ns, np.int32)
    t64 = np.zeros(ns, np.int64)
    gt = 0
    lut = O.bias_lut_f32(hp.beta1, hp.beta2, steps + 2)
    n_relocated = n_rsr_checked = 0

    for it in range(steps):
        vis_t = S.visibility_device(cfg, it, dev)
        for k, x in S.grads_device(cfg, it, dev, vis_t).items():
            gviews[k].copy_(x.view(gviews[k].shape))
        nv_global = int(vis_t.sum().item())
        opt.step(vis_t, cfg.n_pixels, grads=gviews)
        # oracles on the sampled rows, same inputs
        vis_s = vis_t.index_select(0, idx_t).cpu().numpy()
        g32 = {k: _rows_of(gviews[k], idx_t).reshape(ns, -1) for k in names}
        rows = np.flatnonzero(vis_s)
        if mode == "adamw-gs":
            O.step_fp32(mode, lay, p32, g32, m32, v32, c32, rows, hp, n_pixels=cfg.n_pixels,
                        lut=lut)
            O.dar_step_f64(lay, p64, {k: x.astype(np.float64) for k, x in g32.items()}, m64,
                           v64, t64, vis_s, hp, cfg.n_pixels)
        elif mode == "sparse-adam":
            O.step_fp32(mode, lay, p32, g32, m32, v32, c32, rows, hp, lambda_o=lo, lambda_s=ls,
                        n_visible_norm=nv_global, lut=lut)
            # coupled_reg_grad with the global N_v (loss.py:177-198), then sparse_adam_step
            g64 = {k: x.astype(np.float64) for k, x in g32.items()}
            reg = O.coupled_reg_grad_f64(lay, p64, vis_s, lo, ls)
            scale = vis_s.sum() / nv_global if nv_global else 0.0  # local normaliser -> global
            for k, r in reg.items():
                g64[k] = g64[k] + r * scale
            O.sparse_adam_step_f64(lay, p64, g64, m64, v64, t64, vis_s, hp)
        else:
            raise AssertionError(mode)
        b = it + 1
        if b in rsr:  # every picked row checked on the device state, then the sample
            picked = rsr[b]
            pk = torch.from_numpy(picked).to(dev)
            before = opt.state.record.index_select(0, pk)[:, :118].double()
            opt.rsr_apply(picked, 0.2, 0.04)
            after = opt.state.record.index_select(0, pk)[:, :118]
            want = before.clone()
            want[:, 0::2] *= 0.2
            want[:, 1::2] *= 0.04
            assert torch.equal(after, want.float()), f"RSR at {b}"
            n_rsr_checked += picked.size
            loc = np.array([pos[int(r)] for r in picked if int(r) in pos], np.int64)
            for k in names:
                m32[k][loc] = (m32[k][loc].astype(np.float64) * 0.2).astype(np.float32)
                v32[k][loc] = (v32[k][loc].astype(np.float64) * 0.04).astype(np.float32)
            O.rsr_apply_f64(lay, m64, v64, loc, 0.2, 0.04)
        if b in resets:
            opt.reset_rows(resets[b])
            loc = np.array([pos[int(r)] for r in resets[b]], np.int64)
            for k in names:
                m32[k][loc] = 0.0
                v32[k][loc] = 0.0
            c32[loc] = 0
            O.reset_rows_f64(lay, m64, v64, t64, loc)
        if relocate_every and b % relocate_every == 0:
            # mcmc_relocate (pipeline.py:197-233): the plan on the host from the
            # device opacities; rows move on the device (gs_relocate_rows)
            tau_all = params["opacity"].reshape(-1).cpu().numpy()
            plan = mcmc_plan(tau_all, None, np.random.default_rng(seed * 7 + b))
            pre = {k: params[k].reshape(n, -1).index_select(
                0, torch.from_numpy(plan.targets).to(dev)).cpu().numpy() for k in names}
            opt.relocate_rows(plan)
            n_relocated += plan.count
            tau32 = plan.tau_new.astype(np.float32)
            for j, (d, t) in enumerate(zip(plan.dead.tolist(), plan.targets.tolist())):
                if t in pos:
                    p32["opacity"][pos[t], 0] = tau32[j]
                    p64["opacity"][pos[t], 0] = np.float64(tau32[j])
                if d in pos:
                    i = pos[d]
                    for k in names:
                        p32[k][i] = pre[k][j]
                        p64[k][i] = pre[k][j].astype(np.float64)
                    p32["opacity"][i, 0] = tau32[j]
                    p64["opacity"][i, 0] = np.float64(tau32[j])
                    for k in names:
                        m32[k][i] = v32[k][i] = 0.0
                        m64[k][i] = v64[k][i] = 0.0
                    c32[i] = 0
                    t64[i] = 0
            # the moved rows on the device: every dead row equals its target
            dead_t = torch.from_numpy(plan.dead).to(dev)
            got = params["xyz"].index_select(0, dead_t).cpu().numpy()
            assert np.array_equal(got, pre["xyz"]), f"relocation at {b}"
            assert int(opt.state.clock.index_select(0, dead_t).abs().sum().item()) == 0
    torch.cuda.synchronize()
    opt.check_errors()
    gt = gt  # noqa: F841
    clock = _rows_of(opt.state.clock, idx_t)
    assert np.array_equal(clock, c32)
    assert np.array_equal(clock, t64)
    for k in names:
        got_p = _rows_of(params[k], idx_t).reshape(ns, -1)
        got_m = _rows_of(opt.state.m[k], idx_t).reshape(ns, -1)
        got_v = _rows_of(opt.state.v[k], idx_t).reshape(ns, -1)
        assert np.array_equal(got_p, p32[k]), f"{k}/param vs fp32 order"
        assert np.array_equal(got_m, m32[k]), f"{k}/m vs fp32 order"
        assert np.array_equal(got_v, v32[k]), f"{k}/v vs fp32 order"
        assert normwise(got_p, p64[k]) <= NORM_TOL, (k, normwise(got_p, p64[k]))
        assert normwise(got_m, m64[k]) <= NORM_TOL, (k, normwise(got_m, m64[k]))
        assert normwise(got_v, v64[k]) <= NORM_TOL, (k, normwise(got_v, v64[k]))
    return ns, n_rsr_checked, n_relocated


def test_c2_1m_sparse_adam_coupled_100_steps():
    """C2: 1M SH-3 rows, 30% i.i.d., sparse Adam + coupled opacity decay
    (lambda_o = 0.01, presets.py:51-57), 100 steps; the coupled normaliser is
    the global N_v."""
    ns, _, _ = _run(1_000_000, "sparse-adam", 100, lo=0.01, ls=0.0, seed=2)
    assert ns >= 65_536


def test_c3_6m_adamw_gs_rsr_100_steps():
    """C3: 6M SH-3 rows, 30% i.i.d., full AdamW-GS (DAR) with RSR (ratio 0.25,
    alpha 0.2 / 0.04) every 25 iterations, so 4 events fall inside the 100
    steps; every RSR event is checked on all 1.5M rows it picked."""
    ns, n_rsr, _ = _run(6_000_000, "adamw-gs", 100, rsr_every=25, seed=3)
    assert n_rsr == 4 * 1_500_000


def test_c4_3m_mcmc_resets_and_relocation_100_steps():
    """C4: 3M-row MCMC cloud, opacity / scale regularisation (lambda 0.01),
    30% visibility, 2% random state resets every 50 iterations, MCMC
    relocation every 25 and RSR every 50."""
    ns, n_rsr, n_rel = _run(3_000_000, "adamw-gs", 100, lo=0.01, ls=0.01, rsr_every=50,
                            reset_every=50, relocate_every=25, seed=4)
    assert n_rel > 0 and n_rsr == 2 * 750_000


@pytest.mark.parametrize("p,steps", [(0.01, 12), (0.03, 8)])
def test_c5_50m_sparse_masks_multi_step(p, steps):
    """C5 at the sparse end of its visibility sweep: 50M SH-3 rows, 1% and 3%
    i.i.d. visibility.  From the second step on the layout hints select the
    sparse-mask shape (bias warp, 3 CTAs per SM, 512-byte mask tiles) and, at
    3%, the dynamic tail of the tile dealing; every sampled row stays
    bit-exact against the fp32 order and within 1e-6 normwise of the
    reference's float64 step."""
    ns, _, _ = _run(50_000_000, "adamw-gs", steps, p=p, seed=5)
    assert ns >= 65_536


def test_c5_20m_dense_mask_dynamic_tail_multi_step():
    """20M rows at 30%: the streaming kernel's dynamic tail (claims from a
    counter re-armed by the last CTA) over consecutive steps with an RSR
    event in between."""
    ns, n_rsr, _ = _run(20_000_003, "adamw-gs", 6, rsr_every=3, seed=6)
    assert n_rsr >= 2 * 5_000_000  # two events, a quarter of the rows each
