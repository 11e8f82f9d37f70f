"""ShardedAdamWGS on the device kernels, world size 2 (marked gpu).

Two processes share cuda:0 over gloo (this box has one GPU; the collectives
are host-side scalars, so no kernel waits on another rank).  Each rank owns
a contiguous row shard and runs the product path — K1 + K2 through
ShardedAdamWGS.step, the shared RSR sample sliced per shard, the sharded
AIU draw — and the rank-ordered concatenation must equal one unsharded
AdamWGS bit for bit, statistics included (the coupled normaliser N_v is the
global count).  A non-finite gradient on one shard makes both ranks raise
the same GradientError with the global row id, and under the strict check
neither shard is mutated.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
N = 40_009
STEPS = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from paper_2601_16736_b200 import synthetic as S
    cfg = S.WorkloadConfig(n=N, p_vis=0.3, seed=11)
    host = S.make_params(cfg)
    masks = [S.visibility(cfg, s) for s in range(STEPS)]
    grads = [S.step_grads(cfg, s, masks[s]) for s in range(STEPS)]
    return cfg, host, masks, grads


def _aiu():
    from paper_2601_16736_b200.sampling import AiuConfig
    return AiuConfig(start=0, end=100, prob_schedule=((0, 0.3),), eta_schedule=((0, 0.5),),
                     enabled=True)


def _drive(opt, lo, hi, mode, check, sharded):
    """The run_training order (pipeline.py:300-370): step, AIU, RSR on
    boundary 3.  Returns (params, record, stats per step, aiu picks)."""
    from paper_2601_16736_b200.sampling import StSSchedule, stream, stss_sample
    cfg, host, masks, grads = _problem()
    dev = torch.device(DEV)
    inner = opt.opt if sharded else opt
    stats, picks = [], []
    for s in range(STEPS):
        vis = torch.from_numpy(masks[s][lo:hi]).to(dev)
        g = {k: torch.from_numpy(x[lo:hi]).to(dev) for k, x in grads[s].items()}
        if sharded:
            st = opt.step(vis, cfg.n_pixels, grads=g)
            opt.wait_stats()
            stats.append(st.cpu().numpy().copy())
        else:
            opt.step(vis, cfg.n_pixels, grads=g)
            stats.append(opt.engine.stats.cpu().numpy().copy())
        pk = opt.aiu_apply(vis, _aiu(), np.random.default_rng(100 + s), s)
        picks.append(np.asarray(pk, np.int64) + (0 if sharded else lo))
        if s == 2:
            picked = stss_sample(StSSchedule(((0, 0.25),), 3), 3, N, stream(0, "stss", 3))
            opt.rsr_apply(picked if sharded else picked[(picked >= lo) & (picked < hi)] - lo,
                          0.2, 0.04)
    opt.check_errors()
    torch.cuda.synchronize()
    return ({g["name"]: g["params"][0].cpu().numpy() for g in inner.param_groups},
            inner.state.record.cpu().numpy(), stats, picks)


def _worker(rank, world, port, mode, check, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_16736_b200 import synthetic as S
        from paper_2601_16736_b200.engine import GradientError
        from paper_2601_16736_b200.sharded import ShardedAdamWGS, shard_range
        cfg, host, masks, grads = _problem()
        lo, hi = shard_range(N, rank, world)
        params = {k: torch.from_numpy(v[lo:hi].copy()).to(DEV) for k, v in host.items()}
        opt = ShardedAdamWGS(S.param_groups(params), N, mode=mode, lambda_o=0.01,
                             lambda_s=0.001, check=check)
        out = _drive(opt, lo, hi, mode, check, True)
        # a NaN gradient on rank 1's rows only: both ranks raise with the global id
        bad = int(np.flatnonzero(masks[0])[-3])
        vis = torch.from_numpy(masks[0][lo:hi]).to(DEV)
        g = {k: torch.from_numpy(x[lo:hi].copy()).to(DEV) for k, x in grads[0].items()}
        if lo <= bad < hi:
            g["rotation"][bad - lo, 0] = float("nan")
        before = {k: p.clone() for k, p in params.items()}
        err = None
        try:
            opt.step(vis, cfg.n_pixels, grads=g)
            opt.check_errors()
        except GradientError as e:
            err = e.ids.tolist()
        unchanged = all(torch.equal(params[k], before[k]) for k in params)
        q.put((rank, out, err, bad, unchanged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,check", [("adamw-gs", "fused"), ("sparse-adam", "fused"),
                                        ("adamw-gs", "strict")])
def test_two_rank_sharded_step_equals_single_process(mode, check):
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, check, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    cfg, host, masks, grads = _problem()
    params = {k: torch.from_numpy(v.copy()).to(DEV) for k, v in host.items()}
    opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=0.01, lambda_s=0.001, check=check)
    ref_p, ref_rec, ref_stats, ref_picks = _drive(opt, 0, N, mode, check, False)
    for k in ref_p:
        got = np.concatenate([r[1][0][k] for r in res])
        assert np.array_equal(got, ref_p[k]), k
    assert np.array_equal(np.concatenate([r[1][1] for r in res]).view(np.int32),
                          ref_rec.view(np.int32))
    for s in range(STEPS):
        for r in res:  # every rank holds the all-reduced statistics
            got = r[1][2][s]
            assert np.array_equal(got[:8], ref_stats[s][:8]), (s, got, ref_stats[s])
            assert np.allclose(got[8:10], ref_stats[s][8:10], rtol=1e-12, atol=0)  # [10]: hint
        assert np.array_equal(np.concatenate([r[1][3][s] for r in res]), ref_picks[s])
    bad = res[0][3]
    for r in res:
        assert r[2] == [bad], r[2]
        if check == "strict":
            assert r[4], "a strict abort on one shard must leave every shard unmutated"


def test_sharded_capture_nccl_single_rank_matches_eager():
    """ShardedAdamWGS.capture on an NCCL group (one rank on this box): the
    captured step — compaction, the fused step, the statistics all-reduce on
    the side stream joined inside the graph — replays bitwise like eager
    steps, with the reduced statistics."""
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.sharded import ShardedAdamWGS
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        cfg, host, masks, grads = _problem()
        outs = []
        for how in ("eager", "graph"):
            _, params = R.pack({k: torch.from_numpy(v.copy()).to(DEV) for k, v in host.items()})
            _, gv = R.pack({k: torch.zeros(v.shape, device=DEV) for k, v in host.items()})
            sh = ShardedAdamWGS(S.param_groups(params), N, mode="adamw-gs", lambda_o=1e-3,
                                lambda_s=1e-5)
            vis_buf = torch.zeros(N, dtype=torch.bool, device=DEV)
            graph = sh.capture(vis_buf, cfg.n_pixels, grads=gv) if how == "graph" else None
            stats = []
            for s in range(STEPS):
                vis_buf.copy_(torch.from_numpy(masks[s]))
                for k, x in grads[s].items():
                    gv[k].copy_(torch.from_numpy(x).view(gv[k].shape))
                st = graph.replay() if graph is not None else sh.step(vis_buf, cfg.n_pixels,
                                                                      grads=gv)
                stats.append(sh.wait_stats().cpu().numpy().copy())
            sh.check_errors()
            outs.append(({k: p.cpu().numpy() for k, p in params.items()},
                         sh.opt.state.record.cpu().numpy(), stats))
        (pa, ra, sa), (pb, rb, sb) = outs
        for k in pa:
            assert np.array_equal(pa[k], pb[k]), k
        assert np.array_equal(ra.view(np.int32), rb.view(np.int32))
        for x, y in zip(sa, sb):
            assert np.array_equal(x, y)
        assert sa[-1][0] == masks[-1].sum()
    finally:
        dist.destroy_process_group()
