"""Index-sharded multi-GPU host logic on CPU: world_size 2 over gloo.

Each rank plays one GPU: it owns a contiguous row shard, compacts its local
mask, takes the coupled normaliser N_v from an all-reduce, applies the
per-rank step (here the fp32 oracle stands in for the kernel — this test
covers the host-side composition, the GPU tests cover the kernel), slices
the shared RSR sample, and all-reduces the step statistics.  The gathered
result must equal the single-process run bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import adamw_gs_oracle as O

N = 10_007
STEPS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from paper_2601_16736_b200 import synthetic as S
    cfg = S.WorkloadConfig(n=N, p_vis=0.3, seed=4)
    params = S.make_params(cfg)
    masks = [S.visibility(cfg, s) for s in range(STEPS)]
    grads = [S.step_grads(cfg, s, masks[s]) for s in range(STEPS)]
    return cfg, params, masks, grads


def _run_global(mode, lo, ls):
    cfg, params, masks, grads = _problem()
    lay = O.LAYOUT_SH3
    from paper_2601_16736_b200.synthetic import LR_SH3
    hp = O.Hyper(lr=LR_SH3, lambda_o=lo, lambda_s=ls)
    p = {k: v.copy() for k, v in params.items()}
    m = {g.name: np.zeros((N, g.width), np.float32) for g in lay}
    v = {g.name: np.zeros((N, g.width), np.float32) for g in lay}
    c = np.zeros(N, np.int32)
    lut = O.bias_lut_f32(0.9, 0.999, 16)
    stats = []
    for s in range(STEPS):
        rows = np.flatnonzero(masks[s])
        stats.append(O.step_fp32(mode, lay, p, grads[s], m, v, c, rows, hp, n_pixels=cfg.n_pixels,
                                 lambda_o=lo, lambda_s=ls, n_visible_norm=rows.size, lut=lut))
    from paper_2601_16736_b200.sampling import StSSchedule, stream, stss_sample
    picked = stss_sample(StSSchedule(((0, 0.25),), 10), 100, N, stream(0, "stss", 100))
    m = {k: x.astype(np.float64) for k, x in m.items()}
    v = {k: x.astype(np.float64) for k, x in v.items()}
    O.rsr_apply_f64(lay, m, v, picked, 0.2, 0.04)
    return p, m, v, c, stats, picked


def _worker(rank, world, port, mode, lo, ls, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_16736_b200.sampling import StSSchedule, shard_rows, stream, stss_sample
        from paper_2601_16736_b200.sharded import allreduce_stats, global_visible_count, shard_range
        from paper_2601_16736_b200.synthetic import LR_SH3
        cfg, params, masks, grads = _problem()
        a, b = shard_range(N, rank, world)
        lay = O.LAYOUT_SH3
        hp = O.Hyper(lr=LR_SH3, lambda_o=lo, lambda_s=ls)
        p = {k: v[a:b].copy() for k, v in params.items()}
        m = {g.name: np.zeros((b - a, g.width), np.float32) for g in lay}
        v = {g.name: np.zeros((b - a, g.width), np.float32) for g in lay}
        c = np.zeros(b - a, np.int32)
        lut = O.bias_lut_f32(0.9, 0.999, 16)
        stats_all, idx_all = [], []
        for s in range(STEPS):
            local_rows = np.flatnonzero(masks[s][a:b])
            cnt = torch.tensor([local_rows.size], dtype=torch.int32)
            nv = int(global_visible_count(cnt).item())
            st = O.step_fp32(mode, lay, p, {k: x[a:b] for k, x in grads[s].items()}, m, v, c,
                             local_rows, hp, n_pixels=cfg.n_pixels, lambda_o=lo, lambda_s=ls,
                             n_visible_norm=nv, lut=lut)
            vec = torch.tensor([float(st[k]) for k in O.STAT_FIELDS], dtype=torch.float64)
            stats_all.append(allreduce_stats(vec).numpy())
            idx_all.append(local_rows + a)
        picked = stss_sample(StSSchedule(((0, 0.25),), 10), 100, N, stream(0, "stss", 100))
        loc = shard_rows(picked, a, b)
        m64 = {k: x.astype(np.float64) for k, x in m.items()}
        v64 = {k: x.astype(np.float64) for k, x in v.items()}
        O.rsr_apply_f64(lay, m64, v64, loc, 0.2, 0.04)
        q.put((rank, p, m64, v64, c, stats_all, idx_all, loc + a))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,lo,ls", [("adamw-gs", 1e-3, 1e-5), ("sparse-adam", 0.01, 0.001)])
def test_two_rank_shards_equal_single_process(mode, lo, ls):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, lo, ls, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, m, v, c, stats, picked = _run_global(mode, lo, ls)
    # state: concatenation of shards == global, bitwise
    for k in p:
        assert np.array_equal(np.concatenate([r[1][k] for r in res]), p[k])
        assert np.array_equal(np.concatenate([r[2][k] for r in res]), m[k])
        assert np.array_equal(np.concatenate([r[3][k] for r in res]), v[k])
    assert np.array_equal(np.concatenate([r[4] for r in res]), c)
    # compaction: rank-ordered concatenation of local lists == flatnonzero
    _, _, masks, _ = _problem()
    for s in range(STEPS):
        assert np.array_equal(np.concatenate([r[6][s] for r in res]), np.flatnonzero(masks[s]))
        want = np.array([float(stats[s][k]) for k in O.STAT_FIELDS])
        for r in res:
            got = r[5][s]
            assert np.array_equal(got[:8], want[:8])
            assert np.allclose(got[8:], want[8:], rtol=1e-12, atol=0)
    assert np.array_equal(np.concatenate([r[7] for r in res]), picked)


def _aiu_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_16736_b200.sampling import aiu_shard_select
        from paper_2601_16736_b200.sharded import shard_range
        vis, alive = _aiu_problem()
        a, b = shard_range(N, rank, world)
        local_inv = np.flatnonzero(alive[a:b] & ~vis[a:b])
        mine = torch.tensor([local_inv.size], dtype=torch.int64)
        allc = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allc, mine)
        sel = aiu_shard_select(np.random.default_rng(77), 0.3, [int(x) for x in allc], rank)
        q.put((rank, local_inv[sel] + a))
    finally:
        dist.destroy_process_group()


def _aiu_problem():
    rng = np.random.default_rng(5)
    return rng.random(N) < 0.4, rng.random(N) < 0.9


def test_two_rank_aiu_picks_equal_single_process():
    """AIU under index sharding: an all-gather of the per-rank
    invisible counts plus the shared global draw reproduces the single-process
    picks (optimizer.py:437-440) bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_aiu_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    vis, alive = _aiu_problem()
    invisible = np.flatnonzero(alive & ~vis)
    want = invisible[np.random.default_rng(77).random(invisible.size) < 0.3]
    assert np.array_equal(np.concatenate([r[1] for r in res]), want)
