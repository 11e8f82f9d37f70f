"""Device time and roofline of every kernel around the step, on c3 (6M SH-3
rows, granule-aligned records, 30% i.i.d. visibility).  One CUDA-event-timed
launch of each op after warm-up; NVTX ranges name them for ncu / nsys.

    python scripts/prof_ops.py [--n 6000000] [--reps 5]

Algorithmic bytes per op:
  K1 compact     N (mask) + N/8 (bitmap) + 4 N_v (indices)
  K2 step        1664 N_v
  K3 RSR         k * 2 * 8(P+1)    (read + write the moment record; clock untouched but
                                    in the same 16-byte piece)
  K3 reset       k * 8(P+1)        (write)
  K4 stats       N * (8(P+1) + 1 + 4)   (moment record, alive byte, opacity)
  noise          N * (2*12 + 12 + 16 + 4 + 1)   (xyz r/w, scale, rotation, opacity, alive)
  AIU            k * (8(P+1) + 2 * 4P)          (moment record read, theta r/w)
  AIU draw       n_invisible                    (one selection byte written per draw)
  relocate       k * (2 * 4P + 8(P+1) + 2*4)    (theta copy, record reset, two taus)
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.noise import NoiseConfig  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402
from paper_2601_16736_b200.sampling import AiuConfig, StSSchedule, stream, stss_sample  # noqa: E402
from paper_2601_16736_b200.structural import mcmc_plan  # noqa: E402


def timed(fn, reps, graph=True):
    """Device time per call: the calls captured once as a CUDA graph and
    replayed between two events (no host work inside the timed region)."""
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        g.replay()
        b.record()
    else:
        a.record()
        for _ in range(reps):
            fn()
        b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6_000_000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json")
                      .read_text())["hbm_gbs"] if (Path(__file__).resolve().parent.parent /
                                                   "MEASURED_PEAKS.json").exists() else 6650.0
    n = args.n
    P = 59
    cfg = S.WorkloadConfig(n=n, p_vis=0.3, seed=5)
    _, params = R.pack(S.make_params_device(cfg, dev))
    _, grads = R.pack(S.grads_device(cfg, 0, dev))
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5,
                  errors="ignore")
    opt._capturing = True  # no host-side error bookkeeping inside the captures
    vis = S.visibility_device(cfg, 0, dev)
    nv = int(vis.sum())
    for _ in range(3):
        opt.step(vis, cfg.n_pixels, grads=grads)
    torch.cuda.synchronize()
    eng = opt.engine
    rows = {}

    def rec(name, ms, nbytes, note=""):
        gbs = nbytes / (ms / 1e3) / 1e9
        rows[name] = {"ms": ms, "bytes": nbytes, "GB/s": gbs, "frac": gbs / peak, "note": note}

    torch.cuda.nvtx.range_push("K1 compact")
    ms = timed(lambda: eng.compact(vis), args.reps)
    torch.cuda.nvtx.range_pop()
    rec("K1 compact (2 launches)", ms, n + n // 8 + 4 * nv)
    ms = timed(lambda: opt.step(vis, cfg.n_pixels, grads=grads), args.reps)
    rec("K1 fused into K2 (one launch)", ms, n + nv * (28 * P + 8))
    opt.fused_compaction = False
    ms = timed(lambda: opt.step(vis, cfg.n_pixels, grads=grads), args.reps)
    rec("K1 + K2 (index list)", ms, n + n // 8 + nv * (28 * P + 12))
    opt.fused_compaction = True
    picked = stss_sample(StSSchedule(((0, 0.25),), 100), 100, n, stream(0, "stss", 100))
    pk = torch.from_numpy(picked.astype(np.int32)).to(dev)
    k = int(picked.size)
    ms = timed(lambda: opt.rsr_apply(pk, 0.2, 0.04), args.reps)
    rec("K3 RSR (25% of rows)", ms, k * 2 * 8 * (P + 1), f"k={k}")
    dead = torch.from_numpy(np.sort(np.random.default_rng(1).choice(n, n // 50, replace=False))
                            .astype(np.int32)).to(dev)
    ms = timed(lambda: opt.reset_rows(dead), args.reps)
    rec("K3 reset (2% of rows)", ms, dead.numel() * 8 * (P + 1), f"k={dead.numel()}")
    alive = torch.ones(n, dtype=torch.bool, device=dev)
    ms = timed(lambda: eng.stats_all(opt._state_bindings(), alive, opt.state.record), args.reps)
    rec("K4 stats (all rows)", ms, n * (8 * (P + 1) + 1 + 4))
    ncfg = NoiseConfig(enabled=True)
    ms = timed(lambda: opt.noise_perturb(1e-4, ncfg, 7, 3, alive=alive), args.reps)
    rec("noise (all rows)", ms, n * (2 * 12 + 12 + 16 + 4 + 1))
    aiu = AiuConfig(start=0, end=100, prob_schedule=((0, 0.1),), eta_schedule=((0, 0.5),),
                    enabled=True)
    opt._capturing = False
    # one step with every row visible, so every AIU pick has a clock > 0 and
    # takes the full update (the byte count below assumes it)
    opt.step(torch.ones(n, dtype=torch.bool, device=dev), cfg.n_pixels, grads=grads)
    opt.aiu_apply(vis, aiu, stream(0, "aiu", 4), 4)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    picked_aiu = opt.aiu_apply(vis, aiu, stream(0, "aiu", 5), 5)
    t1.record()
    torch.cuda.synchronize()
    rec("AIU end to end (K1 select + Philox draw + K1 + apply, host syncs)", t0.elapsed_time(t1),
        picked_aiu.size * (8 * (P + 1) + 2 * 4 * P), f"k={picked_aiu.size}")
    # the AIU update kernel alone, on the lists of that call
    inv_idx, inv_cnt = eng.compact_select(vis, None, invert=True)
    from paper_2601_16736_b200.sampling import device_bernoulli
    jm = device_bernoulli(stream(0, "aiu", 5), int(inv_cnt.item()), 0.1, 0,
                          int(inv_cnt.item()), dev)
    jl, jc = eng.compact_positions(jm)
    jl, jc = jl.clone(), jc.clone()
    k_aiu = int(jc.item())
    ms = timed(lambda: eng.aiu(opt._state_bindings(), opt.state.record, inv_idx, jl, jc, k_aiu,
                               0.5, opt.eps), args.reps)
    rec("AIU apply kernel", ms, k_aiu * (8 * (P + 1) + 2 * 4 * P), f"k={k_aiu}")
    nd = int(inv_cnt.item())
    ctr = np.zeros(4, np.uint64)
    from paper_2601_16736_b200 import _lib as L
    lib = L.load()
    c4 = (L.C.c_uint64 * 4)(0, 0, 0, 0)
    k2 = (L.C.c_uint64 * 2)(1, 2)
    ms = timed(lambda: lib.gs_philox_bernoulli(c4, k2, 0, nd, 0.1, jm.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream), args.reps)
    rec("AIU Philox draw (device)", ms, nd, f"n={nd} draws (1 B written each)")
    del ctr
    plan = mcmc_plan(params["opacity"].reshape(-1).cpu().numpy(), None,
                     np.random.default_rng(3))
    dead = torch.from_numpy(plan.dead.astype(np.int32)).to(dev)
    targets = torch.from_numpy(plan.targets.astype(np.int32)).to(dev)
    tau_new = torch.from_numpy(plan.tau_new.astype(np.float32)).to(dev)
    opac = [i for i, g in enumerate(opt.param_groups) if g["name"] == "opacity"][0]
    ms = timed(lambda: eng.relocate(opt._state_bindings(), opt.state.record, opac, dead, targets,
                                    tau_new), 1)
    rec("relocate kernel", ms, plan.count * (2 * 4 * P + 8 * (P + 1) + 8), f"k={plan.count}")
    out = {"n": n, "n_visible": nv, "peak_gbs": peak, "ops": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
