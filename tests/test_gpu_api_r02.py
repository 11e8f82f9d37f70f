"""Drop-in behaviour of AdamWGS on the GPU (marked gpu): deferred errors with
no host synchronisation, NumPy index semantics of the state scatters,
visible-only densification statistics in the dense mode, automatic record
adoption of per-attribute parameters, and the 2-D TMA record kernel on bad
rows and ragged chunks."""

import time

import numpy as np
import pytest
import torch

from oracle import adamw_gs_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _cloud(n, p=0.3, seed=1):
    from paper_2601_16736_b200 import synthetic as S
    cfg = S.WorkloadConfig(n=n, p_vis=p, seed=seed)
    return cfg, S.make_params(cfg)


def _fp32_state(host, n):
    lay = O.LAYOUT_SH3
    return ({k: v.copy() for k, v in host.items()},
            {g.name: np.zeros((n, g.width), np.float32) for g in lay},
            {g.name: np.zeros((n, g.width), np.float32) for g in lay},
            np.zeros(n, np.int32))


# --------------------------------------------------------------------------
# errors="defer" (default): no host synchronisation inside step()
# --------------------------------------------------------------------------

def test_default_step_never_waits_for_the_gpu():
    """With the default deferred error check, step() only enqueues work: with
    the GPU held busy by a ~0.5 s sleep kernel, three steps return to the
    host long before the GPU has finished, and torch's sync debug mode sees
    no synchronising call."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(200_003)
    _, params = R.pack({k: torch.from_numpy(v).to(DEV) for k, v in host.items()})
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
    assert opt.errors == "defer"
    _, grads = R.pack({k: torch.from_numpy(x).to(DEV) for k, x in
                       S.step_grads(cfg, 0, S.visibility(cfg, 0)).items()})
    masks = [torch.from_numpy(S.visibility(cfg, s)).to(DEV) for s in range(3)]
    opt.step(masks[0], cfg.n_pixels, grads=grads)  # warm the host caches
    opt.check_errors()
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000_000)  # ~0.5 s of GPU time ahead of the steps
    t0 = time.perf_counter()
    torch.cuda.set_sync_debug_mode("error")
    try:
        for s in range(3):
            opt.step(masks[s], cfg.n_pixels, grads=grads)
    finally:
        torch.cuda.set_sync_debug_mode(0)
    host_s = time.perf_counter() - t0
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    gpu_left = time.perf_counter() - t1
    assert gpu_left > 0.1, "the sleep kernel did not keep the GPU busy"
    assert host_s < 0.5 * gpu_left, (host_s, gpu_left)
    opt.check_errors()


def test_mirror_to_host_stores_through_mapped_pointers():
    """gs_mirror_to_host (the deferred check's statistics store): both
    buffers land in pinned host memory in stream order; a pageable or
    unaligned destination is refused with an error, not written."""
    from paper_2601_16736_b200 import _lib as L
    lib = L.load()
    src0 = torch.arange(11, dtype=torch.float64, device=DEV) * 1.5
    src1 = torch.tensor([7], dtype=torch.int32, device=DEV)
    dst0 = torch.zeros(11, dtype=torch.float64, pin_memory=True)
    dst1 = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    s = torch.cuda.current_stream().cuda_stream
    assert lib.gs_mirror_to_host(src0.data_ptr(), dst0.data_ptr(), 88, src1.data_ptr(),
                                 dst1.data_ptr(), 4, s) == 0
    torch.cuda.synchronize()
    assert dst0.tolist() == src0.tolist() and int(dst1.item()) == 7
    # one buffer only (the fused check has no abort flag)
    src0.mul_(2.0)
    assert lib.gs_mirror_to_host(src0.data_ptr(), dst0.data_ptr(), 88, None, None, 0, s) == 0
    torch.cuda.synchronize()
    assert dst0.tolist() == src0.tolist()
    pageable = torch.zeros(11, dtype=torch.float64)
    assert lib.gs_mirror_to_host(src0.data_ptr(), pageable.data_ptr(), 88, None, None, 0, s) != 0
    assert b"page-locked" in lib.gs_last_error()
    assert lib.gs_mirror_to_host(src0.data_ptr(), dst0.data_ptr(), 6, None, None, 0, s) != 0
    assert pageable.abs().sum().item() == 0


def test_deferred_error_surfaces_at_check_with_ids():
    """A non-finite gradient under errors="defer": the step returns, the
    error (with the reference's row ids, gradients.py:50-58) surfaces at
    check_errors(); the bad row is untouched and the others stepped."""
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.engine import GradientError
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(10_007)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
    vis = S.visibility(cfg, 0)
    g = {k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, 0, vis).items()}
    bad = int(np.flatnonzero(vis)[3])
    g["xyz"][bad, 1] = float("inf")
    opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, grads=g)
    with pytest.raises(GradientError) as ei:
        opt.check_errors()
    assert ei.value.ids.tolist() == [bad]
    clock = opt.state.clock.cpu().numpy()
    assert clock[bad] == 0 and clock.sum() == vis.sum() - 1
    opt.check_errors()  # reported once


def test_strict_abort_rolls_back_the_coupled_global_clock():
    """coupled-adam + strict: an aborted step mutates nothing and does not
    advance global_t (the reference checks before the increment,
    optimizer.py:225-226); the next step uses the right bias correction."""
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.engine import GradientError
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(5_003)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    opt = AdamWGS(S.param_groups(params), mode="coupled-adam", check="strict")
    vis = S.visibility(cfg, 0)
    g = {k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, 0, vis).items()}
    opt.step(torch.from_numpy(vis).to(DEV), grads=g)
    g["f_rest"][17, 3] = float("nan")  # an invisible row: the all-row check still aborts
    before = {k: p.clone() for k, p in params.items()}
    opt.step(torch.from_numpy(vis).to(DEV), grads=g)
    with pytest.raises(GradientError):
        opt.check_errors()
    assert opt.state.global_t == 1
    for k in params:
        assert torch.equal(params[k], before[k])


# --------------------------------------------------------------------------
# K3 index semantics (NumPy fancy indexing)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["bool", "negative", "duplicates", "torch-dup", "torch-neg"])
def test_state_scatter_index_semantics(kind):
    """rsr_apply / reset_rows take indices as the reference's NumPy
    assignment does: a boolean mask selects its rows, negative ids count
    from the end, a repeated id acts once; out-of-range ids raise."""
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(4_099)
    n = cfg.n
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
    for s in range(2):
        vis = S.visibility(cfg, s)
        opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels,
                 grads={k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, s, vis).items()})
    rng = np.random.default_rng(7)
    sel = np.sort(rng.choice(n, 300, replace=False))
    if kind == "bool":
        idx = np.zeros(n, bool)
        idx[sel] = True
    elif kind == "negative":
        idx = np.where(np.arange(sel.size) % 2 == 0, sel - n, sel)
    elif kind == "duplicates":
        idx = np.concatenate([sel, sel[::3]])[::-1]
    elif kind == "torch-dup":
        idx = torch.from_numpy(np.concatenate([sel, sel[:50]])).to(DEV)
    else:
        idx = torch.from_numpy(sel - n).to(DEV)
    m0 = {k: t.contiguous().cpu().numpy().astype(np.float64) for k, t in opt.state.m.items()}
    v0 = {k: t.contiguous().cpu().numpy().astype(np.float64) for k, t in opt.state.v.items()}
    opt.rsr_apply(idx, 0.2, 0.04)
    m_ref = {k: x.copy() for k, x in m0.items()}
    v_ref = {k: x.copy() for k, x in v0.items()}
    O.rsr_apply_f64(O.LAYOUT_SH3, m_ref, v_ref, sel, 0.2, 0.04)
    for k in m_ref:
        assert np.array_equal(opt.state.m[k].contiguous().cpu().numpy(), m_ref[k].astype(np.float32))
        assert np.array_equal(opt.state.v[k].contiguous().cpu().numpy(), v_ref[k].astype(np.float32))
    clock0 = opt.state.clock.cpu().numpy().copy()
    opt.reset_rows(idx)
    clock = opt.state.clock.cpu().numpy()
    want = clock0.copy()
    want[sel] = 0
    assert np.array_equal(clock, want)
    for bad in (np.array([n]), np.array([-n - 1]), torch.tensor([n + 5], device=DEV)):
        with pytest.raises(IndexError):
            opt.rsr_apply(bad, 0.2, 0.04)
    with pytest.raises(IndexError):
        opt.reset_rows(np.zeros(n + 1, bool))


# --------------------------------------------------------------------------
# dense coupled-adam: densification statistics observe visible rows only
# --------------------------------------------------------------------------

@pytest.mark.parametrize("check", ["fused", "strict"])
def test_coupled_adam_densify_stats_visible_rows_only(check):
    """DensifyStats.observe(grads.mu, vis, scale) (pipeline.py:338-339) touches
    only visible rows, also in the dense coupled-adam mode whose step
    updates every row: accum / count bit-exact vs the fp32 order over the
    visible lists."""
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(30_011)
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    opt = AdamWGS(S.param_groups(params), mode="coupled-adam", lambda_o=0.01, lambda_s=0.001,
                  check=check)
    opt.enable_densify_stats()
    acc = np.zeros(cfg.n, np.float32)
    cnt = np.zeros(cfg.n, np.int32)
    for s in range(3):
        vis = S.visibility(cfg, s)
        g = S.step_grads(cfg, s, vis)
        opt.step(torch.from_numpy(vis).to(DEV), grads={k: torch.from_numpy(x).to(DEV)
                                                       for k, x in g.items()},
                 densify_scale=0.5)
        O.densify_observe_fp32(g["xyz"], np.flatnonzero(vis), acc, cnt, 0.5)
    a, c = opt.densify_stats()
    assert np.array_equal(c.cpu().numpy(), cnt)
    assert np.array_equal(a.cpu().numpy(), acc)


# --------------------------------------------------------------------------
# adopt="auto": per-attribute nn.Parameters get the record kernel
# --------------------------------------------------------------------------

def test_auto_adopt_parameters_bit_exact_and_on_records():
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(20_011)
    n = cfg.n
    params = {k: torch.nn.Parameter(torch.from_numpy(v).to(DEV)) for k, v in host.items()}
    ids = {k: id(p) for k, p in params.items()}
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
    assert opt.param_record is not None and opt.grad_record is not None
    assert all(id(p) == ids[k] for k, p in params.items())          # same Parameter objects
    assert all(p.stride(0) == 64 and p.grad.stride(0) == 64 for p in params.values())
    lay = O.LAYOUT_SH3
    hp = O.Hyper(lr=S.LR_SH3, lambda_o=1e-3, lambda_s=1e-5)
    p32, m32, v32, c32 = _fp32_state(host, n)
    for s in range(4):
        vis = S.visibility(cfg, s)
        g = S.step_grads(cfg, s, vis)
        opt.zero_grad()
        loss = sum((p * torch.from_numpy(g[k]).to(DEV).view(p.shape)).sum()
                   for k, p in params.items())
        loss.backward()
        opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels)
        O.step_fp32("adamw-gs", lay, p32, g, m32, v32, c32, np.flatnonzero(vis), hp,
                    n_pixels=cfg.n_pixels)
    opt.check_errors()
    for k in host:
        assert np.array_equal(params[k].detach().cpu().numpy(), p32[k]), k
        assert np.array_equal(opt.state.v[k].contiguous().cpu().numpy(), v32[k]), k
    assert np.array_equal(opt.state.clock.cpu().numpy(), c32)
    plain = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    assert AdamWGS(S.param_groups(plain)).param_record is None        # plain tensors: untouched


# --------------------------------------------------------------------------
# the 2-D TMA record kernel: ragged chunks, bad rows, every mode
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 31, 33, 4_099, 70_001])
@pytest.mark.parametrize("mode", ["adamw-gs", "sparse-adam", "adamw-const-clip", "coupled-adam"])
def test_tma_record_kernel_ragged_and_bad_rows(n, mode):
    """Records (TMA path) vs the cp.async ring (GS_FIXED_VARIANT 21) and the
    fp32 order: ragged last chunks (rows past the list are out of the
    tensor maps' bounds), a non-finite gradient row and a kappa > 80 row are
    skipped whole and left bit-identical, statistics agree."""
    from paper_2601_16736_b200 import _lib
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    lib = _lib.load()
    cfg, host = _cloud(n, p=0.6, seed=n)
    vis = S.visibility(cfg, 0)
    vis[0] = True
    rows = np.flatnonzero(vis)
    g = S.step_grads(cfg, 0, vis)
    if rows.size > 2:
        g["f_rest"][rows[1], 44] = float("nan")
        host = {k: v.copy() for k, v in host.items()}
        host["scaling"][rows[-1], 2] = 81.0
    outs = []
    prev = lib.gs_set_fixed_variant(0)
    try:
        for variant in (0, 21):
            lib.gs_set_fixed_variant(variant)
            _, params = R.pack({k: torch.from_numpy(v).to(DEV) for k, v in host.items()})
            _, gr = R.pack({k: torch.from_numpy(x).to(DEV) for k, x in g.items()})
            opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=1e-3, lambda_s=1e-5,
                          errors="ignore")
            for _ in range(2):
                opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, grads=gr)
            outs.append(({k: p.cpu().numpy() for k, p in params.items()},
                         opt.state.record.cpu().numpy(), opt.last_stats()))
    finally:
        lib.gs_set_fixed_variant(prev)
    (pa, ra, sa), (pb, rb, sb) = outs
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k
    assert np.array_equal(ra[:, :120].view(np.int32), rb[:, :120].view(np.int32))
    for f in sa:  # the fused compaction groups rows into chunks differently: sums reorder
        if f == "n_runs":  # layout hint, depends on the chunking
            continue
        if f.startswith("sum_"):
            assert sa[f] == pytest.approx(sb[f], rel=1e-12, abs=0), f
        else:
            assert sa[f] == sb[f], f
    if rows.size > 2 and mode != "coupled-adam":
        for k in pa:
            assert np.array_equal(pa[k][rows[1]], host[k][rows[1]])
        assert sa["n_bad_grad"] == 1 and sa["n_bad_domain"] == 1


# --------------------------------------------------------------------------
# densify_adc on the 3DGS SH-3 record layout
# --------------------------------------------------------------------------

@pytest.mark.parametrize("params_layout", ["record", "attr"])
def test_densify_adc_sh3_vs_oracle(params_layout):
    """Clone / split / prune (pipeline.py:116-185) on SH-3 rows after real
    steps: the split child is sampled in the parent's 3-D footprint
    (quaternion rotation, oracle.densify_adc_sh3_f64, same rng draws);
    every output row equals fp32 of the oracle's float64 value, children
    start with fresh state, parents keep theirs, and the rebound optimizer
    steps the new rows."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    from paper_2601_16736_b200.structural import DensifyConfig
    cfg, host = _cloud(3_001, p=0.5, seed=21)
    n = cfg.n
    params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
    if params_layout == "record":
        _, params = R.pack(params)
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
    opt.enable_densify_stats()
    for s in range(3):
        vis = S.visibility(cfg, s)
        g = {k: torch.from_numpy(x * 1e3).to(DEV) for k, x in S.step_grads(cfg, s, vis).items()}
        opt.step(torch.from_numpy(vis).to(DEV), cfg.n_pixels, grads=g, densify_scale=1.0)
    opt.check_errors()
    torch.cuda.synchronize()
    acc, cnt = opt.densify_stats()
    acc_h, cnt_h = acc.cpu().numpy().astype(np.float64), cnt.cpu().numpy().astype(np.int64)
    alive = np.random.default_rng(4).random(n) < 0.97
    dcfg = dict(grad_threshold=float(np.quantile(acc_h / np.maximum(cnt_h, 1), 0.8)),
                prune_opacity=0.01, split_scale_px=0.1, split_shrink=1.6, max_primitives=10_000)
    p0 = {k: t.cpu().numpy().reshape(n, -1) for k, t in params.items()}
    m0 = {k: t.contiguous().cpu().numpy().reshape(n, -1) for k, t in opt.state.m.items()}
    v0 = {k: t.contiguous().cpu().numpy().reshape(n, -1) for k, t in opt.state.v.items()}
    t0 = opt.state.clock.cpu().numpy()
    want = O.densify_adc_sh3_f64(p0, m0, v0, t0, alive, acc_h, cnt_h, dcfg,
                                 np.random.default_rng(77))
    res = opt.densify_adc(DensifyConfig(**dcfg), np.random.default_rng(77), alive=alive,
                          iteration=9)
    wp, wm, wv, wt, walive, wsrc, counts = want
    assert counts[0] > 0 and counts[1] > 0 and counts[2] > 0, counts
    kinds = {e["kind"]: e["count"] for e in res.events}
    assert (kinds.get("clone", 0), kinds.get("split", 0), kinds.get("prune", 0)) == counts
    n_out = wsrc.size
    assert opt.n_rows == n_out and np.array_equal(res.src, wsrc) and np.array_equal(res.alive,
                                                                                    walive)
    for k in host:
        got = res.params[k].cpu().numpy().reshape(n_out, -1)
        assert np.array_equal(got, wp[k].astype(np.float32)), k
        assert np.array_equal(opt.state.m[k].contiguous().cpu().numpy().reshape(n_out, -1),
                              wm[k].astype(np.float32)), k
        assert np.array_equal(opt.state.v[k].contiguous().cpu().numpy().reshape(n_out, -1),
                              wv[k].astype(np.float32)), k
    assert np.array_equal(opt.state.clock.cpu().numpy(), wt.astype(np.int32))
    vis = torch.rand(n_out, device=DEV) < 0.5
    grads = {k: torch.randn_like(t) * 1e-3 for k, t in res.params.items()}
    opt.step(vis, 4096, grads=grads)
    opt.check_errors()
    assert opt.last_stats()["n_stepped"] == int(vis.sum())


# --------------------------------------------------------------------------
# K1 fused into K2 (gs_step_rows_masked)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n,kind", [(n, k) for n in (1, 2047, 100_003, 1_300_001)
                                    for k in ("bool", "radii", "offset-bool", "offset-radii")]
                         + [(4_900_001, "bool")])
@pytest.mark.parametrize("mode", ["adamw-gs", "sparse-adam", "sparse-coupled", "adamw-const"])
def test_fused_compaction_equals_index_path(n, kind, mode):
    if n > 2_000_000 and mode != "adamw-gs":
        pytest.skip("the largest cloud runs in one mode (host-side data generation time)")
    """The one-launch step (the loader compacts the mask: uint8 or int32
    radii, aligned or not, ragged tails) equals K1 + K2 bit for bit:
    parameters, moment records, clocks, statistics (n_visible included)."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(n, p=0.3, seed=n + 5)
    outs = []
    for fused in (True, False):
        _, params = R.pack({k: torch.from_numpy(v).to(DEV) for k, v in host.items()})
        lo, ls = (0.0, 0.0) if mode == "sparse-adam" else (1e-3, 1e-5)
        # sparse-coupled: the coupled normaliser from the count pass, then the fused step
        opt = AdamWGS(S.param_groups(params), mode="sparse-adam" if mode == "sparse-coupled"
                      else mode, lambda_o=lo, lambda_s=ls, fused_compaction=fused)
        stats = []
        for s in range(3):
            vis = S.visibility(cfg, s)
            if "radii" in kind:
                m = torch.from_numpy(np.where(vis, np.arange(n) % 7 + 1, 0).astype(np.int32))
            else:
                m = torch.from_numpy(vis)
            if kind.startswith("offset"):
                big = torch.zeros(n + 3, dtype=m.dtype)
                big[3:] = m
                m = big.to(DEV)[3:]
            else:
                m = m.to(DEV)
            _, g = R.pack({k: torch.from_numpy(x).to(DEV) for k, x in S.step_grads(cfg, s, vis).items()})
            opt.step(m, cfg.n_pixels, grads=g)
            # K1 + K2 for unaligned masks (offset views: both fused kernels
            # read the mask in 16-byte pieces); clouds under 16 mask tiles per
            # CTA slot (1 KB tiles: 1024 uint8 rows, 256 radii) run the
            # two-phase kernel, larger ones the streaming loader; a one-row
            # cloud has no row stride to describe records by (index path)
            eligible = not kind.startswith("offset") and n > 1
            assert (opt._last_ctx[1] is None) == (fused and eligible)
            stats.append(opt.last_stats())
        opt.check_errors()
        outs.append(({k: p.cpu().numpy() for k, p in params.items()},
                     opt.state.record.cpu().numpy(), stats))
    (pa, ra, sa), (pb, rb, sb) = outs
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k
    assert np.array_equal(ra.view(np.int32), rb.view(np.int32))
    for x, y in zip(sa, sb):
        for f in x:
            if f == "n_runs":
                continue
            if f.startswith("sum_"):
                assert x[f] == pytest.approx(y[f], rel=1e-12, abs=0), f
            else:
                assert x[f] == y[f], f


@pytest.mark.parametrize("pattern", ["empty", "all", "last-row", "first-tile", "burst", "every-17th"])
@pytest.mark.parametrize("n,kind", [(4_099, "bool"), (300_017, "bool"), (300_017, "radii"),
                                    (77, "radii")])
def test_small_cloud_fused_edge_masks(pattern, n, kind):
    """The fused kernels of small clouds (under 16 mask tiles per CTA slot)
    on degenerate masks: nothing visible, everything, one row at the ragged
    end, one dense tile, one dense burst inside one CTA's mask slice, a
    regular stride.  adamw-gs steps stream per-CTA mask slices (the second
    step of a coherent pattern takes the balanced two-phase kernel: the
    burst's ids are served to every CTA); coupled sparse-adam runs two-phase
    (it counts the mask's N_v itself).  Equals K1 + K2 bit for bit over two
    steps (the grid barrier re-arms)."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(n, seed=n + 11)
    vis = np.zeros(n, bool)
    if pattern == "all":
        vis[:] = True
    elif pattern == "last-row":
        vis[-1] = True
    elif pattern == "first-tile":
        vis[:1024] = True
    elif pattern == "burst":
        vis[n // 3:n // 3 + min(n // 10 + 1, 40_000)] = True
    elif pattern == "every-17th":
        vis[::17] = True
    outs = []
    for fused in (True, False):
        for mode in ("adamw-gs", "sparse-coupled"):
            _, params = R.pack({k: torch.from_numpy(v).to(DEV) for k, v in host.items()})
            opt = AdamWGS(S.param_groups(params), mode="sparse-adam" if mode != "adamw-gs" else mode,
                          lambda_o=1e-3, lambda_s=1e-5, fused_compaction=fused)
            stats = []
            for s in range(2):
                m = (torch.from_numpy(np.where(vis, np.arange(n) % 5 + 1, 0).astype(np.int32))
                     if kind == "radii" else torch.from_numpy(vis)).to(DEV)
                _, g = R.pack({k: torch.from_numpy(x).to(DEV)
                               for k, x in S.step_grads(cfg, s, vis).items()})
                opt.step(m, cfg.n_pixels, grads=g)
                assert (opt._last_ctx[1] is None) == fused
                stats.append(opt.last_stats())
            opt.check_errors()
            outs.append(({k: p.cpu().numpy() for k, p in params.items()},
                         opt.state.record.cpu().numpy(), stats))
    for (pa, ra, sa), (pb, rb, sb) in zip(outs[:2], outs[2:]):
        for k in pa:
            assert np.array_equal(pa[k], pb[k]), k
        assert np.array_equal(ra.view(np.int32), rb.view(np.int32))
        for x, y in zip(sa, sb):
            assert x["n_visible"] == y["n_visible"] == int(vis.sum())
            for f in x:
                if f != "n_runs" and not f.startswith("sum_"):
                    assert x[f] == y[f], f


# --------------------------------------------------------------------------
# the AIU Bernoulli draw on the device (reference Philox stream, bit for bit)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("skip", [0, 1, 3, 4, 6])
@pytest.mark.parametrize("n_total,first,n", [(1, 0, 1), (3, 0, 3), (4_099, 0, 4_099),
                                             (1_000_003, 0, 1_000_003), (50_001, 17, 30_000),
                                             (50_001, 2, 1), (10, 10, 0)])
def test_device_bernoulli_is_host_draw(skip, n_total, first, n):
    """sampling.device_bernoulli == (rng.random(n_total) < prob)[first:first+n]
    for every buffer position, and the generator ends in the same state as
    after the host draw (the next draws agree)."""
    from paper_2601_16736_b200.sampling import device_bernoulli, stream
    a, b = stream(5, "aiu", 3), stream(5, "aiu", 3)
    a.random(skip)
    b.random(skip)
    want = (a.random(n_total) < 0.3)[first:first + n]
    got = device_bernoulli(b, n_total, 0.3, first, n, torch.device(DEV)).cpu().numpy()
    assert np.array_equal(got.astype(bool), want)
    assert np.array_equal(a.random(9), b.random(9))


def test_noise_record_fast_path_matches_generic():
    """gs_noise_perturb on SH-3 parameter records (16-byte row accesses)
    draws the same noise as the generic strided path: same Philox counters,
    same arithmetic (agreement to fp32 rounding)."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.noise import NoiseConfig
    from paper_2601_16736_b200.optimizer import AdamWGS
    cfg, host = _cloud(50_001, seed=3)
    outs = []
    for rec in (True, False):
        params = {k: torch.from_numpy(v).to(DEV) for k, v in host.items()}
        if rec:
            _, params = R.pack(params)
        opt = AdamWGS(S.param_groups(params), mode="adamw-gs", adopt=False)
        alive = torch.from_numpy(np.random.default_rng(1).random(cfg.n) < 0.9).to(DEV)
        d = opt.noise_perturb(1e-3, NoiseConfig(enabled=True), seed=77, iteration=5, alive=alive)
        outs.append((d.cpu().numpy(), params["xyz"].cpu().numpy()))
    (da, xa), (db, xb) = outs
    assert np.abs(da - db).max() <= 1e-6 * np.abs(db).max()
    assert np.abs(xa - xb).max() <= 1e-6 * np.abs(xb).max()
    assert np.count_nonzero(da) > 0
