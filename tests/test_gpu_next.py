"""§8(f) rows on the GPU: fused densification statistics, AIU, position
noise and structural state ops (marked gpu)."""

import numpy as np
import pytest
import torch

from oracle import adamw_gs_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.mark.parametrize("path", ["fixed", "record", "rows", "groups"])
def test_densify_stats_fused(path):
    """DensifyStats.observe (pipeline.py:77-82) fused into K2: the gather
    kernel, the ring kernel on parameter/gradient records, the generic
    row-record kernel and the per-group-state kernel."""
    from paper_2601_16736_b200 import _lib
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    lib = _lib.load()
    cfg = S.WorkloadConfig(n=30_011, p_vis=0.3, seed=12)
    host = S.make_params(cfg)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    if path == "record":
        _, params = R.pack(params)
    prev = lib.gs_set_fixed_variant(0 if path in ("fixed", "record") else -1)
    try:
        opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5,
                      state_layout="groups" if path == "groups" else "rows")
        opt.enable_densify_stats()
        acc32 = np.zeros(cfg.n, np.float32)
        cnt32 = np.zeros(cfg.n, np.int32)
        acc64 = np.zeros(cfg.n)
        cnt64 = np.zeros(cfg.n, np.int64)
        scale = 24.0
        for s in range(4):
            vis = S.visibility(cfg, s)
            g = S.step_grads(cfg, s, vis)
            gd = {k: torch.from_numpy(x).to(DEV) for k, x in g.items()}
            if path == "record":
                gd = R.pack(gd)[1]
            opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, densify_scale=scale, grads=gd)
            O.densify_observe_fp32(g["xyz"], np.flatnonzero(vis), acc32, cnt32, scale)
            O.densify_observe_f64(g["xyz"], vis, acc64, cnt64, scale)
        acc, cnt = opt.densify_stats()
        acc = acc.cpu().numpy()
        cnt = cnt.cpu().numpy()
    finally:
        lib.gs_set_fixed_variant(prev)
    assert np.array_equal(cnt, cnt32) and np.array_equal(cnt, cnt64)
    assert np.array_equal(acc, acc32)                     # bit-exact vs the fp32 order
    assert np.abs(acc - acc64).max() <= 1e-6 * np.abs(acc64).max()


def test_aiu_matches_reference_golden():
    """aiu_apply (optimizer.py:425-450): picked rows bit-exact (host RNG),
    parameters bit-exact vs the fp32 kernel order and within 1e-6 normwise of
    the float64 reference."""
    import json
    from _golden import GOLDEN, normwise
    from paper_2601_16736_b200.optimizer import AdamWGS
    from paper_2601_16736_b200.sampling import AiuConfig
    z = np.load(GOLDEN / "aiu.npz")
    meta = json.loads(str(z["meta"]))
    lay = O.LAYOUT_REF2D
    params = {g.name: torch.from_numpy(z[f"init_{g.name}"]).to(DEV) for g in lay}
    opt = AdamWGS([{"params": [params[g.name]], "lr": meta["lr"][g.name], "name": g.name}
                   for g in lay], mode="adamw-gs")
    for g in lay:
        opt.state.m[g.name][:] = torch.from_numpy(z[f"m_{g.name}"])
        opt.state.v[g.name][:] = torch.from_numpy(z[f"v_{g.name}"])
    opt.state.clock[:] = torch.from_numpy(z["t"].astype(np.int32))
    aiu = AiuConfig(start=0, end=100, prob_schedule=((0, meta["prob"]),),
                    eta_schedule=((0, meta["eta"]),), enabled=True)
    picked = opt.aiu_apply(torch.from_numpy(z["vis"]).to(DEV), aiu,
                           np.random.default_rng(meta["draw_seed"]), meta["iteration"],
                           alive=torch.from_numpy(z["alive"]).to(DEV))
    assert np.array_equal(picked, z["picked"])
    p32 = {g.name: z[f"init_{g.name}"].copy() for g in lay}
    O.aiu_apply_fp32(lay, p32, {g.name: z[f"m_{g.name}"] for g in lay},
                     {g.name: z[f"v_{g.name}"] for g in lay}, z["t"], picked, meta["lr"],
                     meta["eta"], meta["eps"], opt.engine.lut.cpu().numpy())
    for g in lay:
        got = params[g.name].cpu().numpy()
        assert np.array_equal(got, p32[g.name]), g.name
        assert normwise(got, z[f"out_{g.name}"]) <= 1e-6, g.name
    # state untouched (optimizer.py:430)
    for g in lay:
        assert np.array_equal(opt.state.m[g.name].cpu().numpy(), z[f"m_{g.name}"])
    assert np.array_equal(opt.state.clock.cpu().numpy(), z["t"].astype(np.int32))


def _noise_inputs(n, dims, tau, alive=None):
    pos = torch.zeros((n, dims), dtype=torch.float32, device=DEV)
    ks = torch.zeros((n, dims), dtype=torch.float32, device=DEV)
    if dims == 2:
        rot = torch.zeros((n,), dtype=torch.float32, device=DEV)
    else:
        rot = torch.zeros((n, 4), dtype=torch.float32, device=DEV)
        rot[:, 0] = 1.0
    tau_t = torch.full((n, 1), tau, dtype=torch.float32, device=DEV)
    return pos, ks, rot, tau_t


@pytest.mark.parametrize("dims", [2, 3])
def test_noise_gate_saturates_for_solid(dims):                      # test_optimizer.py:493-498
    from paper_2601_16736_b200.noise import NoiseConfig, noise_perturb
    pos, ks, rot, tau = _noise_inputs(100, dims, 6.0)
    d = noise_perturb(pos, ks, rot, tau, 1.0, NoiseConfig(enabled=True), seed=0, iteration=0)
    assert float(d.abs().max()) < 1e-20


@pytest.mark.parametrize("dims", [2, 3])
def test_noise_monte_carlo_covariance(dims):                       # test_optimizer.py:508-522
    from paper_2601_16736_b200.noise import NoiseConfig, noise_perturb
    n = 100_000
    pos, ks, rot, tau = _noise_inputs(n, dims, -3.0)
    cfg = NoiseConfig(enabled=True, eta_ratio=1.0)
    d = noise_perturb(pos, ks, rot, tau, 1.0, cfg, seed=7, iteration=3).cpu().numpy()
    o = 1.0 / (1.0 + np.exp(3.0))
    gate = 1.0 / (1.0 + np.exp(cfg.lambda_mu * (o - cfg.lambda_t)))
    cov = np.cov(d.T)
    for k in range(dims):
        assert cov[k, k] == pytest.approx(gate ** 2, rel=0.02)
    for a in range(dims):
        for b in range(a + 1, dims):
            assert abs(cov[a, b]) < 0.02 * gate ** 2


@pytest.mark.parametrize("dims", [2, 3])
def test_noise_shapes_by_covariance_and_skips_dead(dims):
    from paper_2601_16736_b200.noise import NoiseConfig, noise_perturb
    n = 200_000
    pos, ks, rot, tau = _noise_inputs(n, dims, -3.0)
    ks[:, 0] = np.log(2.0)                     # Sigma = diag(4, 1[, 1]) with identity rotation
    alive = torch.ones(n, dtype=torch.bool, device=DEV)
    alive[::7] = False
    cfg = NoiseConfig(enabled=True)
    before = pos.clone()
    d = noise_perturb(pos, ks, rot, tau, 0.5, cfg, seed=1, iteration=9, alive=alive, add=True)
    dn = d.cpu().numpy()
    assert np.all(dn[::7] == 0.0)
    assert torch.equal(pos, before + d)
    live = np.ones(n, bool)
    live[::7] = False
    o = 1.0 / (1.0 + np.exp(3.0))
    gate = 1.0 / (1.0 + np.exp(cfg.lambda_mu * (o - cfg.lambda_t)))
    var = dn[live].var(axis=0)
    assert var[0] == pytest.approx((0.5 * gate * 4.0) ** 2, rel=0.03)
    assert var[1] == pytest.approx((0.5 * gate) ** 2, rel=0.03)
    # reproducible per (seed, iteration), fresh per iteration
    d2 = noise_perturb(pos, ks, rot, tau, 0.5, cfg, seed=1, iteration=9, alive=alive)
    d3 = noise_perturb(pos, ks, rot, tau, 0.5, cfg, seed=1, iteration=10, alive=alive)
    assert torch.equal(d, d2) and not torch.equal(d, d3)


def test_noise_rotation_3d_matches_dense_covariance():
    """Quaternion rotation: delta = -lr*gate * R S^2 R^T gamma (3DGS build_rotation)."""
    from paper_2601_16736_b200.noise import NoiseConfig, noise_perturb
    n = 200_000
    rng = np.random.default_rng(0)
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    s = np.log([0.5, 1.0, 2.0])
    pos, ks, rot, tau = _noise_inputs(n, 3, -3.0)
    ks[:] = torch.tensor(s, dtype=torch.float32)
    rot[:] = torch.tensor(q, dtype=torch.float32)
    d = noise_perturb(pos, ks, rot, tau, 1.0, NoiseConfig(enabled=True), seed=5,
                      iteration=1).cpu().numpy().astype(np.float64)
    w, x, y, z = q
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    sigma = R @ np.diag(np.exp(2 * s)) @ R.T
    o = 1.0 / (1.0 + np.exp(3.0))
    gate = 1.0 / (1.0 + np.exp(100.0 * (o - 0.005)))
    want = gate ** 2 * sigma @ sigma.T           # cov(Sigma gamma) = Sigma Sigma^T
    got = np.cov(d.T)
    assert np.abs(got - want).max() <= 0.03 * np.abs(want).max()


def test_structural_select_concat_keep_rows_consistent():
    """MomentState.select / concatenate (optimizer.py:141-156) on the row
    record: pruning and appending rows keeps every view aligned."""
    from paper_2601_16736_b200.optimizer import MomentState
    n = 1000
    params = {"xyz": torch.zeros((n, 3), device=DEV), "opacity": torch.zeros((n, 1), device=DEV),
              "f_rest": torch.zeros((n, 15, 3), device=DEV)}
    st = MomentState.zeros_like(params)
    st.m["xyz"][:] = torch.arange(n, device=DEV, dtype=torch.float32)[:, None]
    st.v["f_rest"][:, 7, 1] = torch.arange(n, device=DEV, dtype=torch.float32)
    st.clock[:] = torch.arange(n, device=DEV, dtype=torch.int32)
    keep = torch.arange(0, n, 3, device=DEV)
    sub = st.select(keep)
    assert torch.equal(sub.m["xyz"][:, 0], keep.float())
    assert torch.equal(sub.v["f_rest"][:, 7, 1], keep.float())
    assert torch.equal(sub.clock, keep.int())
    fresh = MomentState.zeros_like({k: v[:10] for k, v in params.items()})
    cat = MomentState.concatenate(sub, fresh)
    assert len(cat) == keep.numel() + 10
    assert torch.equal(cat.clock[-10:], torch.zeros(10, dtype=torch.int32, device=DEV))
    assert torch.equal(cat.m["xyz"][: keep.numel(), 0], keep.float())


@pytest.mark.parametrize("state_layout", ["rows", "groups"])
@pytest.mark.parametrize("params_layout", ["attr", "record", "adopt"])
def test_mcmc_relocate_matches_reference_golden(state_layout, params_layout):
    """AdamWGS.mcmc_relocate (pipeline.py:197-233) against the reference run:
    relocated attributes bit-exact, shared opacity = fp32 of the reference's
    float64 logit, respawn moments and clocks reset, other rows untouched."""
    import json

    from _golden import GOLDEN
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200.optimizer import AdamWGS
    z = np.load(GOLDEN / "relocate.npz")
    meta = json.loads(str(z["meta"]))
    lay = O.LAYOUT_REF2D
    params = {g.name: torch.from_numpy(z[f"init_{g.name}"]).to(DEV) for g in lay}
    if params_layout == "record":
        _, params = R.pack(params)
    elif params_layout == "adopt":
        params = {k: torch.nn.Parameter(t) for k, t in params.items()}
        R.adopt(params, grads=False)
    opt = AdamWGS([{"params": [params[g.name]], "lr": 1e-3, "name": g.name} for g in lay],
                  mode="adamw-gs", state_layout=state_layout)
    for g in lay:
        opt.state.m[g.name][:] = torch.from_numpy(z[f"m_{g.name}"])
        opt.state.v[g.name][:] = torch.from_numpy(z[f"v_{g.name}"])
    opt.state.clock[:] = torch.from_numpy(z["t"].astype(np.int32))
    plan = opt.mcmc_relocate(np.random.default_rng(meta["draw_seed"]),
                             alive=torch.from_numpy(z["alive"]).to(DEV))
    torch.cuda.synchronize()
    assert plan.count == meta["event_count"] and plan.ids_hash() == meta["event_hash"]
    for g in lay:
        got = params[g.name].detach().cpu().numpy()
        assert np.array_equal(got, z[f"out_{g.name}"].astype(np.float32)), g.name
        assert np.array_equal(opt.state.m[g.name].cpu().numpy(),
                              z[f"out_m_{g.name}"].astype(np.float32)), g.name
        assert np.array_equal(opt.state.v[g.name].cpu().numpy(),
                              z[f"out_v_{g.name}"].astype(np.float32)), g.name
    assert np.array_equal(opt.state.clock.cpu().numpy(), z["out_t"].astype(np.int32))


@pytest.mark.parametrize("state_layout", ["rows", "groups"])
@pytest.mark.parametrize("params_layout", ["attr", "record", "adopt"])
def test_densify_adc_matches_reference_golden(state_layout, params_layout):
    """structural.densify_adc (pipeline.py:116-185) against the reference run:
    clone / split (same rng draws) / prune decisions and events identical,
    every output row bit-equal to fp32 of the reference's float64 value,
    children with fresh state, parents' state carried."""
    import json

    from _golden import GOLDEN
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200.optimizer import AdamWGS
    from paper_2601_16736_b200.structural import DensifyConfig, densify_adc
    z = np.load(GOLDEN / "densify.npz")
    meta = json.loads(str(z["meta"]))
    lay = O.LAYOUT_REF2D
    params = {g.name: torch.from_numpy(z[f"init_{g.name}"]).to(DEV) for g in lay}
    if params_layout == "record":
        _, params = R.pack(params)
    elif params_layout == "adopt":
        params = {k: torch.nn.Parameter(t) for k, t in params.items()}
        R.adopt(params, grads=False)
    opt = AdamWGS([{"params": [params[g.name]], "lr": 1e-3, "name": g.name} for g in lay],
                  mode="adamw-gs", state_layout=state_layout)
    for g in lay:
        opt.state.m[g.name][:] = torch.from_numpy(z[f"m_{g.name}"])
        opt.state.v[g.name][:] = torch.from_numpy(z[f"v_{g.name}"])
    opt.state.clock[:] = torch.from_numpy(z["t"].astype(np.int32))
    res = densify_adc(opt, z["accum"], z["count"], DensifyConfig(**meta["cfg"]),
                      np.random.default_rng(meta["draw_seed"]), alive=z["alive"], iteration=5)
    torch.cuda.synchronize()
    assert [{k: e[k] for k in ("kind", "count", "affected_ids_hash")} for e in res.events] == \
        meta["events"]
    assert opt.n_rows == meta["n_out"] and len(opt.state) == meta["n_out"]
    assert np.array_equal(res.src, z["out_src"]) and np.array_equal(res.alive, z["out_alive"])
    # packed and adopted parameters come back as views of one gathered record
    assert (R.record_of(res.params) is not None) == (params_layout != "attr")
    for g in lay:
        got = opt.param_groups[[x["name"] for x in opt.param_groups].index(g.name)]["params"][0]
        assert got is res.params[g.name]
        assert np.array_equal(got.cpu().numpy().reshape(meta["n_out"], -1),
                              z[f"out_{g.name}"].astype(np.float32)), g.name
        assert np.array_equal(opt.state.m[g.name].cpu().numpy().reshape(meta["n_out"], -1),
                              z[f"out_m_{g.name}"].astype(np.float32)), g.name
        assert np.array_equal(opt.state.v[g.name].cpu().numpy().reshape(meta["n_out"], -1),
                              z[f"out_v_{g.name}"].astype(np.float32)), g.name
    assert np.array_equal(opt.state.clock.cpu().numpy(), z["out_t"].astype(np.int32))
    # the rebound optimizer steps on the new rows
    vis = torch.rand(opt.n_rows, device=DEV) < 0.5
    grads = {g.name: torch.randn_like(res.params[g.name]) * 1e-3 for g in lay}
    opt.step(vis, 4096, grads=grads)
    assert opt.last_stats()["n_stepped"] == int(vis.sum())


def test_sharded_aiu_single_rank_matches_unsharded():
    """ShardedAdamWGS.aiu_apply (collective draw path) on a one-rank group
    equals AdamWGS.aiu_apply: same picks, same parameters."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    from paper_2601_16736_b200.sampling import AiuConfig
    from paper_2601_16736_b200.sharded import ShardedAdamWGS
    cfg = S.WorkloadConfig(n=20_000, p_vis=0.3, seed=8)
    host = S.make_params(cfg)
    aiu = AiuConfig(start=0, end=100, prob_schedule=((0, 0.25),), eta_schedule=((0, 0.5),),
                    enabled=True)
    vis = torch.from_numpy(S.visibility(cfg, 0)).to(DEV)
    out = []
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        for sharded in (False, True):
            params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
            kw = dict(mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
            if sharded:
                opt = ShardedAdamWGS(S.param_groups(params), cfg.n, **kw)
                inner = opt.opt
            else:
                opt = inner = AdamWGS(S.param_groups(params), **kw)
            g = {k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, 0, S.visibility(
                cfg, 0)).items()}
            inner.step(vis, cfg.n_pixels, grads=g)
            picked = opt.aiu_apply(vis, aiu, np.random.default_rng(3), 5)
            out.append((np.asarray(picked), {k: p.cpu().numpy() for k, p in params.items()}))
    finally:
        dist.destroy_process_group()
    assert out[0][0].size > 0 and np.array_equal(out[0][0], out[1][0])
    for k in out[0][1]:
        assert np.array_equal(out[0][1][k], out[1][1][k]), k
