"""GPU parity: the CUDA path through the C ABI vs the oracle (marked gpu).

Tiers:
  * indices / counts / clocks: bit-exact;
  * vs the fp32 kernel-order restatement (oracle.step_fp32): bit-exact
    (ULP_TOL = 0) — the kernels use only correctly rounded fp32 operations
    and their own deterministic exp, all mirrored op for op;
  * vs the float64 reference (golden vectors from the unmodified reference):
    normwise max|d|/max|ref| <= 1e-6 per tensor.
"""

import numpy as np
import pytest
import torch

from _golden import STEP_CASES, Case, normwise
from oracle import adamw_gs_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
ULP_TOL = 0
NORM_TOL = 1e-6


def ulp_diff(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    a = np.where(a < 0, np.int64(-2**31) - a, a)
    b = np.where(b < 0, np.int64(-2**31) - b, b)
    return np.abs(a - b)


def assert_close_ulp(got, want, what, tol=ULP_TOL):
    d = ulp_diff(got, want)
    assert d.max(initial=0) <= tol, f"{what}: max ulp diff {d.max()} (at {np.argmax(d)})"


# --------------------------------------------------------------------------
# K1 compaction
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 4095, 4096, 4097, 100_003, 1_000_000, 6_000_000])
@pytest.mark.parametrize("p", [0.0, 0.01, 0.3, 1.0])
def test_compaction_bit_exact(n, p):
    from paper_2601_16736_b200.engine import StepEngine
    rng = np.random.default_rng(n + int(p * 100))
    mask = rng.random(n) < p
    eng = StepEngine(n, torch.device(DEV), 0.9, 0.999)
    vis = torch.from_numpy(mask).to(DEV)
    for _ in range(2):  # second call exercises the epoch-tagged workspace reuse
        idx, cnt = eng.compact(vis)
        c = int(cnt.item())
        ref = np.flatnonzero(mask)
        assert c == ref.size
        assert np.array_equal(idx[:c].cpu().numpy(), ref)


def test_compaction_coherent_misaligned_and_radii():
    from paper_2601_16736_b200.engine import StepEngine
    rng = np.random.default_rng(3)
    n = 300_001
    blocks = rng.random((n + 63) // 64) < 0.3
    mask = np.repeat(blocks, 64)[:n]
    eng = StepEngine(n, torch.device(DEV), 0.9, 0.999)
    big = torch.zeros(n + 1, dtype=torch.bool, device=DEV)
    big[1:] = torch.from_numpy(mask).to(DEV)
    idx, cnt = eng.compact(big[1:])  # pointer not 16-byte aligned -> scalar path
    assert np.array_equal(idx[: int(cnt.item())].cpu().numpy(), np.flatnonzero(mask))
    radii = rng.integers(-3, 4, n).astype(np.int32)
    idx, cnt = eng.compact(torch.from_numpy(radii).to(DEV))
    assert np.array_equal(idx[: int(cnt.item())].cpu().numpy(), np.flatnonzero(radii > 0))


def test_compaction_many_launches_same_workspace():
    from paper_2601_16736_b200.engine import StepEngine
    rng = np.random.default_rng(5)
    n = 50_000
    eng = StepEngine(n, torch.device(DEV), 0.9, 0.999)
    for i in range(50):
        mask = rng.random(n) < rng.random()
        idx, cnt = eng.compact(torch.from_numpy(mask).to(DEV))
        ref = np.flatnonzero(mask)
        assert int(cnt.item()) == ref.size
        assert np.array_equal(idx[: ref.size].cpu().numpy(), ref)


# --------------------------------------------------------------------------
# K2 step on the golden cases
# --------------------------------------------------------------------------

def _gpu_case_run(case: Case, check="fused", layout="rows"):
    from paper_2601_16736_b200.optimizer import AdamWGS
    hp = case.hyper()
    meta = case.meta
    init = case.init(np.float32)
    params = {g.name: torch.from_numpy(init[g.name]).to(DEV) for g in case.layout}
    coupled = case.layout is O.LAYOUT_REF2D
    opt = AdamWGS([{"params": [params[g.name]], "lr": hp.lr[g.name], "name": g.name}
                   for g in case.layout], mode=case.mode, betas=(hp.beta1, hp.beta2), eps=hp.eps,
                  lambda_o=hp.lambda_o if (coupled or case.mode != "sparse-adam") else 0.0,
                  lambda_s=hp.lambda_s if (coupled or case.mode != "sparse-adam") else 0.0,
                  ct_opacity=hp.ct_opacity, ct_scale=hp.ct_scale, check=check,
                  state_layout=layout)
    stats = []
    for s in range(case.steps):
        gr = case.grads(s, np.float32)
        grads = {k: torch.from_numpy(v).to(DEV) for k, v in gr.items()}
        vis = torch.from_numpy(case.vis[s]).to(DEV)
        opt.step(vis, meta.get("n_pixels"), mu_lr_scale=meta["mu_lr_scale"],
                 clip=meta.get("clip"), grads=grads)
        stats.append(opt.last_stats())
    out = {k: p.cpu().numpy() for k, p in params.items()}
    m = {k: t.contiguous().cpu().numpy() for k, t in opt.state.m.items()}
    v = {k: t.contiguous().cpu().numpy() for k, t in opt.state.v.items()}
    return out, m, v, opt.state.clock.contiguous().cpu().numpy(), stats


def _oracle_fp32(case: Case):
    from test_oracle import coupled_lambdas
    hp = case.hyper()
    p = case.init(np.float32)
    m = {g.name: np.zeros((case.n, g.width), np.float32) for g in case.layout}
    v = {g.name: np.zeros((case.n, g.width), np.float32) for g in case.layout}
    clock = np.zeros(case.n, np.int32)
    lut = O.bias_lut_f32(hp.beta1, hp.beta2, 20000)
    stats = []
    for s in range(case.steps):
        g = case.grads(s, np.float32)
        vis = case.vis[s]
        rows = np.flatnonzero(vis) if case.mode != "coupled-adam" else np.arange(case.n)
        stats.append(O.step_fp32(case.mode, case.layout, p, g, m, v, clock, rows, hp,
                                 n_pixels=case.meta.get("n_pixels"),
                                 mu_lr_scale=case.meta["mu_lr_scale"], clip=case.meta.get("clip"),
                                 n_visible_norm=int(vis.sum()), global_t=s + 1, lut=lut,
                                 **coupled_lambdas(case)))
    return p, m, v, clock, stats


@pytest.mark.parametrize("name", STEP_CASES)
@pytest.mark.parametrize("check", ["fused", "strict"])
@pytest.mark.parametrize("layout", ["rows", "groups"])
def test_golden_step_parity(name, check, layout):
    case = Case(name)
    out, m, v, clock, stats = _gpu_case_run(case, check, layout)
    # tier (i): vs the float64 reference
    eo, em, ev, et = case.expected()
    assert np.array_equal(clock, et)
    for g in case.layout:
        assert normwise(out[g.name], eo[g.name]) <= NORM_TOL, g.name
        assert normwise(m[g.name], em[g.name]) <= NORM_TOL, g.name
        assert normwise(v[g.name], ev[g.name]) <= NORM_TOL, g.name
    # tier (ii): vs the fp32 restatement of the kernel
    po, mo, vo, co, so = _oracle_fp32(case)
    assert np.array_equal(clock, co)
    for g in case.layout:
        assert_close_ulp(out[g.name], po[g.name], f"{name}/{g.name}/param")
        assert_close_ulp(m[g.name], mo[g.name], f"{name}/{g.name}/m")
        assert_close_ulp(v[g.name], vo[g.name], f"{name}/{g.name}/v")
    if check == "fused":
        for s_gpu, s_ref in zip(stats, so):
            for k, want in s_ref.items():
                if k.startswith("sum_"):
                    assert s_gpu[k] == pytest.approx(want, rel=1e-6, abs=1e-30), k
                else:
                    assert s_gpu[k] == want, k


# --------------------------------------------------------------------------
# C1: 100k SH3, 50% visibility, 100 steps (BASELINE.json configs[0])
# --------------------------------------------------------------------------

@pytest.mark.parametrize("family,layout,params_layout", [
    ("bernoulli", "rows", "attr"), ("coherent", "rows", "attr"), ("bernoulli", "groups", "attr"),
    ("bernoulli", "rows", "record"), ("coherent", "rows", "record")])
def test_c1_100_steps_vs_oracles(family, layout, params_layout):
    """C1: 100 steps x 100k rows, bit-exact vs the fp32 order and
    within 1e-6 normwise of the float64 reference; per-attribute tensors and
    granule-aligned parameter/gradient records (the ring kernel)."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    n, steps = 100_000, 100
    cfg = S.WorkloadConfig(n=n, p_vis=0.5, mask_family=family, seed=1)
    host = S.make_params(cfg)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    if params_layout == "record":
        _, params = R.pack(params)
        grec, gviews = R.pack({k: torch.zeros_like(v) for k, v in params.items()})
    opt = AdamWGS(S.param_groups(params, cfg), mode="adamw-gs", lambda_o=cfg.lambda_o,
                  lambda_s=cfg.lambda_s, state_layout=layout)
    # oracles
    lay = O.LAYOUT_SH3
    hp = O.Hyper(lr=S.LR_SH3, lambda_o=cfg.lambda_o, lambda_s=cfg.lambda_s)
    p32 = {k: v.copy() for k, v in host.items()}
    m32 = {g.name: np.zeros((n, g.width), np.float32) for g in lay}
    v32 = {g.name: np.zeros((n, g.width), np.float32) for g in lay}
    c32 = np.zeros(n, np.int32)
    p64 = {k: v.astype(np.float64) for k, v in host.items()}
    m64 = {g.name: np.zeros((n, g.width)) for g in lay}
    v64 = {g.name: np.zeros((n, g.width)) for g in lay}
    t64 = np.zeros(n, np.int64)
    lut = O.bias_lut_f32(0.9, 0.999, steps + 2)
    for s in range(steps):
        vis = S.visibility(cfg, s)
        g = S.step_grads(cfg, s, vis)
        if params_layout == "record":
            for k, x in g.items():
                gviews[k].copy_(torch.from_numpy(x).view(gviews[k].shape))
            opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, grads=gviews)
        else:
            opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels,
                     grads={k: torch.from_numpy(x).to(DEV) for k, x in g.items()})
        O.step_fp32("adamw-gs", lay, p32, g, m32, v32, c32, np.flatnonzero(vis), hp,
                    n_pixels=cfg.n_pixels, lut=lut)
        O.dar_step_f64(lay, p64, {k: x.astype(np.float64) for k, x in g.items()}, m64, v64, t64,
                       vis, hp, cfg.n_pixels)
    clock = opt.state.clock.contiguous().cpu().numpy()
    assert np.array_equal(clock, c32)
    assert np.array_equal(clock, t64)
    for gname in host:
        got_p = params[gname].cpu().numpy()
        got_m = opt.state.m[gname].contiguous().cpu().numpy()
        got_v = opt.state.v[gname].contiguous().cpu().numpy()
        assert_close_ulp(got_p, p32[gname], f"{gname}/param")
        assert_close_ulp(got_m, m32[gname], f"{gname}/m")
        assert_close_ulp(got_v, v32[gname], f"{gname}/v")
        assert normwise(got_p, p64[gname]) <= NORM_TOL, gname
        assert normwise(got_m, m64[gname]) <= NORM_TOL, gname
        assert normwise(got_v, v64[gname]) <= NORM_TOL, gname


def test_adopted_parameters_backward_into_records_bit_exact():
    """records.adopt: per-attribute nn.Parameters re-homed into a record, their
    gradients filled by a real backward (loss = sum(theta * G), so dL/dtheta = G
    exactly) and read from p.grad by step(); 6 steps bit-exact vs the fp32
    order, and the kernel sees one row stride (64 floats) for every group."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    n, steps = 20_011, 6
    cfg = S.WorkloadConfig(n=n, p_vis=0.3, seed=5)
    host = S.make_params(cfg)
    params = {k: torch.nn.Parameter(torch.from_numpy(v).to(DEV)) for k, v in host.items()}
    rec, grec = R.adopt(params)
    assert all(p.stride(0) == 64 and p.grad.stride(0) == 64 for p in params.values())
    opt = AdamWGS(S.param_groups(params, cfg), mode="adamw-gs", lambda_o=cfg.lambda_o,
                  lambda_s=cfg.lambda_s)
    lay = O.LAYOUT_SH3
    hp = O.Hyper(lr=S.LR_SH3, lambda_o=cfg.lambda_o, lambda_s=cfg.lambda_s)
    p32 = {k: v.copy() for k, v in host.items()}
    m32 = {g.name: np.zeros((n, g.width), np.float32) for g in lay}
    v32 = {g.name: np.zeros((n, g.width), np.float32) for g in lay}
    c32 = np.zeros(n, np.int32)
    for s in range(steps):
        vis = S.visibility(cfg, s)
        g = S.step_grads(cfg, s, vis)
        opt.zero_grad()   # record-view gradients are zeroed in place, not dropped
        assert all(p.grad is not None for p in params.values())
        loss = sum((p * torch.from_numpy(g[k]).to(DEV).view(p.shape)).sum()
                   for k, p in params.items())
        loss.backward()
        assert torch.equal(R.views_like(grec, params)["f_rest"].cpu(),
                           torch.from_numpy(g["f_rest"]).view(n, 45))
        opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels)
        O.step_fp32("adamw-gs", lay, p32, g, m32, v32, c32, np.flatnonzero(vis), hp,
                    n_pixels=cfg.n_pixels)
    assert np.array_equal(opt.state.clock.contiguous().cpu().numpy(), c32)
    for k, p in params.items():
        assert p.data_ptr() == R.views_like(rec, params)[k].data_ptr()
        assert_close_ulp(p.detach().cpu().numpy(), p32[k], f"{k}/param")
        assert_close_ulp(opt.state.m[k].contiguous().cpu().numpy(), m32[k], f"{k}/m")
        assert_close_ulp(opt.state.v[k].contiguous().cpu().numpy(), v32[k], f"{k}/v")


# --------------------------------------------------------------------------
# Edge cases: empty, single-row and ragged visibility (chunk tails of the
# ring kernel, zero-length launches), every step mode, both layouts
# --------------------------------------------------------------------------

def _edge_masks(n, rng):
    out = [np.zeros(n, bool), np.ones(n, bool)]
    one = np.zeros(n, bool)
    one[n - 1] = True                      # only the last row
    out.append(one)
    out.append(rng.random(n) < 0.5)
    alt = np.zeros(n, bool)
    alt[::33] = True                       # one row per 33: never a full chunk-aligned run
    out.append(alt)
    return out


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1023])
@pytest.mark.parametrize("params_layout", ["attr", "record"])
@pytest.mark.parametrize("mode", ["adamw-gs", "sparse-adam", "adamw-const-clip"])
def test_edge_visibility_bit_exact_vs_fp32_order(n, params_layout, mode):
    """Empty, all-visible, last-row-only and ragged masks on tiny clouds: the
    step (K1 + K2, including zero-length and partial-chunk launches) stays
    bit-exact with the fp32 restatement, and invisible rows are untouched."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    rng = np.random.default_rng(n)
    cfg = S.WorkloadConfig(n=n, p_vis=0.5, seed=n + 7)
    host = S.make_params(cfg)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    if params_layout == "record":
        _, params = R.pack(params)
    lo = cfg.lambda_o if mode != "sparse-adam" else 0.01
    ls = cfg.lambda_s if mode != "sparse-adam" else 0.0
    opt = AdamWGS(S.param_groups(params, cfg), mode=mode, lambda_o=lo, lambda_s=ls)
    lay = O.LAYOUT_SH3
    hp = O.Hyper(lr=S.LR_SH3, lambda_o=lo, lambda_s=ls)
    p32 = {k: v.copy() for k, v in host.items()}
    m32 = {g.name: np.zeros((n, g.width), np.float32) for g in lay}
    v32 = {g.name: np.zeros((n, g.width), np.float32) for g in lay}
    c32 = np.zeros(n, np.int32)
    masks = _edge_masks(n, rng)
    lut = O.bias_lut_f32(0.9, 0.999, len(masks) + 2)
    for s, vis in enumerate(masks):
        g = S.step_grads(cfg, s, vis)
        before = {k: p.detach().cpu().numpy().copy() for k, p in params.items()}
        opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels,
                 grads={k: torch.from_numpy(x).to(DEV) for k, x in g.items()})
        kw = dict(lambda_o=lo, lambda_s=ls, n_visible_norm=int(vis.sum())) \
            if mode == "sparse-adam" else {}
        O.step_fp32(mode, lay, p32, g, m32, v32, c32, np.flatnonzero(vis), hp,
                    n_pixels=cfg.n_pixels, lut=lut, **kw)
        st = opt.last_stats()
        assert st["n_visible"] == int(vis.sum()) == st["n_stepped"], (s, st)
        for k, p in params.items():
            now = p.detach().cpu().numpy()
            assert np.array_equal(now[~vis], before[k][~vis]), (s, k)
    assert np.array_equal(opt.state.clock.contiguous().cpu().numpy(), c32)
    for gname in host:
        assert_close_ulp(params[gname].cpu().numpy(), p32[gname], f"{gname}/param")
        assert_close_ulp(opt.state.m[gname].contiguous().cpu().numpy(), m32[gname], f"{gname}/m")
        assert_close_ulp(opt.state.v[gname].contiguous().cpu().numpy(), v32[gname], f"{gname}/v")


# --------------------------------------------------------------------------
# Maximum sizes: the fixed-layout kernels use 32-bit row offsets up to
# rows * row stride < 2^32 (60M granule-aligned rows); beyond that
# (70M rows) records run the ring kernel with 64-bit row offsets
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [60_000_000, 70_000_000])
def test_max_size_clouds_sampled_rows_vs_fp32_order(n):
    """A 60M-row cloud (the ring kernel right below its 32-bit offset limit)
    and a 70M-row cloud (past it: the 64-bit-offset ring kernel) in
    granule-aligned records (~72 GB in HBM).  Two steps; 4096 sampled visible rows, including
    the last rows of the cloud, are bit-exact with the fp32 restatement and a
    sample of invisible rows is untouched."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    if torch.cuda.get_device_properties(0).total_memory < 150 * 2**30:
        pytest.skip("needs a 180 GB B200")
    g = torch.Generator(device=DEV)
    g.manual_seed(n)
    shapes = {name: (w,) for name, w in S.SH3_LAYOUT}
    prec = torch.zeros((n, 64), dtype=torch.float32, device=DEV)
    params = R.views(prec, shapes)
    for name, p in params.items():  # in place, no full-size temporaries
        if name == "scaling":
            p.uniform_(-6.9, -0.7, generator=g)
        elif name == "opacity":
            p.normal_(-1.0, 2.0, generator=g)
        else:
            p.normal_(0.0, 1.0, generator=g)
    grec = torch.zeros((n, 64), dtype=torch.float32, device=DEV)
    grads = R.views(grec, shapes)
    for gv in grads.values():
        gv.normal_(0.0, 1e-3, generator=g)
    vis = torch.rand(n, device=DEV, generator=g) < 0.3
    vis[-3:] = True
    vis[-4] = False
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
    rng = np.random.default_rng(n)
    vis_idx = torch.nonzero(vis).view(-1)
    pick = torch.from_numpy(np.unique(np.concatenate([
        rng.choice(vis_idx.numel(), 4093, replace=False), [vis_idx.numel() - k for k in (1, 2, 3)]])))
    rows = vis_idx[pick.to(DEV)]
    frozen = torch.tensor([n - 4, 0, n // 2 + 1], device=DEV)
    frozen = frozen[~vis[frozen]]
    host_p = {k: p[rows].cpu().numpy().reshape(rows.numel(), -1) for k, p in params.items()}
    host_g = {k: x[rows].cpu().numpy().reshape(rows.numel(), -1) for k, x in grads.items()}
    before_frozen = prec[frozen].cpu().numpy()
    for _ in range(2):
        opt.step(vis, 1_000_000, grads=grads)
    k = rows.numel()
    lay = O.LAYOUT_SH3
    hp = O.Hyper(lr=S.LR_SH3, lambda_o=1e-3, lambda_s=1e-5)
    m32 = {gr.name: np.zeros((k, gr.width), np.float32) for gr in lay}
    v32 = {gr.name: np.zeros((k, gr.width), np.float32) for gr in lay}
    c32 = np.zeros(k, np.int32)
    lut = O.bias_lut_f32(0.9, 0.999, 4)
    for _ in range(2):
        O.step_fp32("adamw-gs", lay, host_p, host_g, m32, v32, c32, np.arange(k), hp,
                    n_pixels=1_000_000, lut=lut)
    assert np.array_equal(opt.state.clock[rows].cpu().numpy(), c32)
    for name, p in params.items():
        assert_close_ulp(p[rows].cpu().numpy().reshape(k, -1), host_p[name], f"{name}/param")
        assert_close_ulp(opt.state.m[name][rows].cpu().numpy().reshape(k, -1), m32[name], f"{name}/m")
        assert_close_ulp(opt.state.v[name][rows].cpu().numpy().reshape(k, -1), v32[name], f"{name}/v")
    assert np.array_equal(prec[frozen].cpu().numpy(), before_frozen)
    del opt, prec, grec, params, grads
    torch.cuda.empty_cache()
