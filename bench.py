"""AdamW-GS optimizer-step benchmark (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload c3] [--mask bernoulli|coherent] [--vis P]

A *step* is one pass of the hot path over one batch of synthetic input:
visibility compaction (K1) + the fused AdamW-GS step (K2, with the per-step
statistics) + the Re-State Regularization scatter on RSR boundaries (K3),
exactly as ``run_training`` composes them (pipeline.py:316-370), through the
public optimizer (``AdamWGS.step``; ``ShardedAdamWGS.step`` on N > 1 GPUs,
which adds the statistics all-reduce).

Default workload: BASELINE.json configs[2] — 6M Gaussians per GPU, SH-3,
30% i.i.d. visibility, full AdamW-GS (DAR lambda_o=1e-3, lambda_s=1e-5,
N_I=1e6) with RSR (ratio 0.25, alpha 0.2/0.04, interval 100); N GPUs own
N index shards of 6M rows each (weak scaling; ``--strong`` splits one cloud).
Every line also carries the north star's scaling cloud as extra legs:
``c5_strong`` = 50M Gaussians in total split over the N GPUs (strong
scaling) at 30% and at 1% visibility.

``--gpus N`` without torchrun launches N ranks itself (torch.distributed.run,
127.0.0.1); under torchrun N must equal WORLD_SIZE.

``value``  visible Gaussians updated / s, inputs resident in HBM, device time
           (CUDA events on the launching stream around one CUDA graph of the
           K steps, max over ranks), RSR amortised at its interval.
``e2e``    the same metric through the public API with host buffers: per
           step a fresh mask is copied H2D from pinned memory, the step
           kernel gathers the visible rows' gradients zero-copy from pinned
           host memory, and the step statistics are read back D2H (the dense
           H2D-copy variant is reported beside it as ``dense_copy``).
``roofline`` the fused step kernel (K2): algorithmic bytes per launch /
           its CUDA-event duration vs the measured HBM copy peak.
``cpu_baseline`` the reference algorithm (oracle float64 port of
           optimizer.py:241-298) on a bounded sample, rank 0 at N=1.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (n rows per GPU, p_vis, mode, lambda_o, lambda_s, rsr, resets, description)
    "c1": dict(n=100_000, p=0.5, mode="adamw-gs", lo=1e-3, ls=1e-5, rsr=False, reset=0.0,
               desc="100k SH3 Gaussians, 50% visibility, adamw-gs (DAR)"),
    "c2": dict(n=1_000_000, p=0.3, mode="sparse-adam", lo=0.01, ls=0.0, rsr=False, reset=0.0,
               desc="1M SH3 Gaussians, 30% visibility, sparse Adam + coupled opacity decay 0.01"),
    "c3": dict(n=6_000_000, p=0.3, mode="adamw-gs", lo=1e-3, ls=1e-5, rsr=True, reset=0.0,
               desc="6M SH3 Gaussians, 30% visibility, adamw-gs DAR + RSR(0.25, a=0.2/0.04, "
                    "every 100)"),
    "c4": dict(n=3_000_000, p=0.3, mode="adamw-gs", lo=0.01, ls=0.01, rsr=True, reset=0.02,
               desc="3M-cap MCMC cloud, 30% visibility, adamw-gs + RSR + 2% relocation resets "
                    "every 100"),
    "c5": dict(n=50_000_000, p=0.3, mode="adamw-gs", lo=1e-3, ls=1e-5, rsr=False, reset=0.0,
               desc="50M SH3 Gaussians index-sharded, adamw-gs"),
}
RSR_INTERVAL = 100
RSR_RATIO = 0.25
ALPHA1, ALPHA2 = 0.2, 0.04
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
NOMINAL_HBM_GBS = 8000.0   # B200 spec sheet, the north star's "~8 TB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--mask", default="bernoulli", choices=["bernoulli", "coherent"])
    ap.add_argument("--vis", type=float, default=None, help="override visibility fraction")
    ap.add_argument("--rows", type=int, default=None,
                    help="override rows per GPU (not --n: torchrun would claim it as an "
                    "abbreviation of its own --nnodes/--nproc-per-node)")
    ap.add_argument("--strong", action="store_true", help="split --rows across ranks (strong)")
    ap.add_argument("--check", default="fused", choices=["fused", "strict"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-legs", action="store_true", help="skip the c5 strong-scaling legs")
    ap.add_argument("--no-fused", dest="fused", action="store_false",
                    help="K1 then K2 on the index list instead of the fused one-launch step")
    ap.add_argument("--sharded", action="store_true",
                    help="run ShardedAdamWGS (NCCL process group) even on one GPU")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=150.0,
                    help="budget of the whole --impl reference run")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the timed steps eagerly instead of as one CUDA graph")
    ap.add_argument("--layout", default="rows", choices=["rows", "groups"],
                    help="optimizer-state layout (row records or per-group tensors)")
    ap.add_argument("--state-align", type=int, default=16,
                    help="moment-record rows padded to a multiple of this many floats "
                         "(16: 512-byte SH-3 rows, whole 64-byte granules; 2: 480 bytes)")
    ap.add_argument("--record-align", type=int, default=16,
                    help="parameter / gradient record rows padded to a multiple of this "
                         "many floats (16: 256-byte SH-3 rows, whole granules; 4: 240 bytes)")
    ap.add_argument("--host-record-align", type=int, default=16,
                    help="e2e: pinned host gradient record rows padded to a multiple of this "
                         "many floats (16: 256-byte SH-3 rows, two PCIe read lines)")
    ap.add_argument("--params", default="record", choices=["record", "attr"],
                    help="parameter / gradient HBM layout: attribute views of one "
                         "row-interleaved record (records.py) or one tensor per attribute")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(workload, mask, p_vis, params):
    p = ROOT / "profiles" / "traffic.json"
    try:
        d = json.loads(p.read_text())
        return d.get(f"{workload}/{mask}/{p_vis:g}/{params}")
    except Exception:
        return None


REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        reasons = set()
        for _, _, r in busy:
            for bit, name in REASON_BITS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy),
                "sm_max_mhz": max(s[1] for s in busy), "reasons": sorted(reasons),
                "samples": len(busy)}


# ------------------------------------------------------------ CPU baseline
def _ref_shard_worker(wid, n_rows, p_vis, mask, seed, wl, n_steps, barrier, out_q):
    """One host process of the reference arm: the float64 port of the
    reference step (oracle/adamw_gs_oracle.py, optimizer.py:231-298) over its
    own row shard. Rows are independent, so shards run in parallel. Every
    step starts behind a barrier, and the step time is the slowest shard's."""
    import numpy as np

    from oracle import adamw_gs_oracle as O
    from paper_2601_16736_b200 import synthetic as S

    cfg = S.WorkloadConfig(n=n_rows, p_vis=p_vis, mask_family=mask, seed=seed * 1000 + wid)
    lay = O.LAYOUT_SH3
    host = S.make_params(cfg)
    p = {k: v.astype(np.float64) for k, v in host.items()}
    m = {g.name: np.zeros((n_rows, g.width)) for g in lay}
    v = {g.name: np.zeros((n_rows, g.width)) for g in lay}
    t = np.zeros(n_rows, np.int64)
    hp = O.Hyper(lr=S.LR_SH3, lambda_o=wl["lo"], lambda_s=wl["ls"])
    grad_sets, masks = [], []
    for s in range(min(n_steps, 3)):
        vis = S.visibility(cfg, s)
        masks.append(vis)
        grad_sets.append({k: x.astype(np.float64) for k, x in S.step_grads(cfg, s, vis).items()})
    times, nv = [], []
    for s in range(n_steps):
        vis = masks[s % len(masks)]
        g = {k: x.copy() for k, x in grad_sets[s % len(grad_sets)].items()}
        if barrier is not None:
            barrier.wait()
        t0 = time.perf_counter()
        if wl["mode"] == "adamw-gs":
            O.dar_step_f64(lay, p, g, m, v, t, vis, hp, cfg.n_pixels)
        else:
            reg = O.coupled_reg_grad_f64(lay, p, vis, wl["lo"], wl["ls"])
            for k, r in reg.items():
                g[k] = g[k] + r
            O.sparse_adam_step_f64(lay, p, g, m, v, t, vis, hp)
        times.append(time.perf_counter() - t0)
        nv.append(int(vis.sum()))
    if out_q is None:
        return times, nv
    out_q.put((wid, times, nv))
    return None


def host_workers() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_reference_rate(wl: dict, p_vis: float, mask: str, budget_s: float, steps=None, warmup=1,
                       seed=0, workers: int = 1):
    """Time the reference algorithm (float64 oracle port of dar_step /
    sparse_adam_step, optimizer.py:231-298) on a bounded sample of the
    workload: the same layout, distributions, visibility fraction and mode.
    ``workers`` host processes each own one row shard (rows are independent;
    NumPy's elementwise kernels are single-threaded). Returns (visible/s,
    sample description, rows, per-step times)."""
    import multiprocessing as mp

    # calibrate one process on a small shard, then size the sample to the budget
    n0 = 20_000
    tt, nv = _ref_shard_worker(0, n0, p_vis, mask, seed, wl, 2, None, None)
    rate1 = nv[-1] / max(tt[-1], 1e-9)
    n_steps = steps if steps is not None else 4
    total = n_steps + warmup
    workers = max(1, int(workers))
    # memory-bandwidth contention: assume half the per-process rate when parallel
    eff = rate1 * (workers if workers == 1 else workers / 2)
    rows = int(min(wl["n"], max(n0 * workers, eff * budget_s / max(total, 1) / p_vis)))
    shard = rows // workers
    rows = shard * workers
    if workers == 1:
        per = [_ref_shard_worker(0, shard, p_vis, mask, seed, wl, total, None, None)]
    else:
        ctx = mp.get_context("spawn")
        barrier = ctx.Barrier(workers)
        q = ctx.Queue()
        procs = [ctx.Process(target=_ref_shard_worker,
                             args=(w, shard, p_vis, mask, seed, wl, total, barrier, q))
                 for w in range(workers)]
        for pr in procs:
            pr.start()
        got = [q.get() for _ in procs]
        for pr in procs:
            pr.join()
        per = [(tm, n) for _, tm, n in sorted(got)]
    step_t = [max(p[0][s] for p in per) for s in range(warmup, total)]
    step_nv = [sum(p[1][s] for p in per) for s in range(warmup, total)]
    value = sum(step_nv) / sum(step_t)
    sample = (f"{rows} of {wl['n']} rows in {workers} row shard(s), {n_steps} timed steps after "
              f"{warmup} warm-up, float64 NumPy port of the reference step "
              f"(oracle/adamw_gs_oracle.py), {workers} host process(es) x 1 thread; "
              f"step time = slowest shard")
    return value, sample, rows, step_t


def reference_arm(args, wl, p_vis):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    budget = args.ref_seconds
    import numpy as np  # noqa: F401
    cores = host_workers()
    value, sample, rows, tt = cpu_reference_rate(
        wl, p_vis, args.mask, budget_s=budget * 0.8, steps=args.steps, warmup=args.warmup,
        seed=args.seed, workers=cores)
    line = {
        "metric": "visible Gaussians updated/sec per optimizer step",
        "value": value, "unit": "visible Gaussians/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.mean(tt),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(args, wl, p_vis, world),
        "cpu_baseline": {"value": value, "unit": "visible Gaussians/s", "cores": cores,
                         "kind": "port", "sample": sample,
                         "host_cpus": os.cpu_count(),
                         "affinity_cpus": len(os.sched_getaffinity(0))},
        "e2e": {"value": value, "unit": "visible Gaussians/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, wl, p_vis, world, strong=None, mask=None):
    strong = args.strong if strong is None else strong
    mask = args.mask if mask is None else mask
    n = wl["n"]
    return {"workload": f"{wl['name']}: {wl['desc']}",
            "n_per_gpu": n // world if strong else n, "n_total": n if strong else n * world,
            "p_visible": p_vis, "mask": mask, "mode": wl["mode"],
            "layout": "SH3 (59 fp32 / Gaussian)",
            "lambda_o": wl["lo"], "lambda_s": wl["ls"], "n_pixels": 1_000_000,
            "rsr": {"ratio": RSR_RATIO, "alpha1": ALPHA1, "alpha2": ALPHA2,
                    "interval": RSR_INTERVAL} if wl["rsr"] else None,
            "reset_fraction": wl["reset"] or None, "check": args.check,
            "state_layout": args.layout,
            "param_layout": (f"record (attribute views of one (n, "
                             f"{(59 + args.record_align - 1) // args.record_align * args.record_align}"
                             f") fp32 row record, gradients likewise; moment record rows of "
                             f"{(120 + args.state_align - 1) // args.state_align * args.state_align * 4}"
                             f" B)") if args.params == "record" else "one tensor per attribute",
            "l2": "inputs larger than L2 (working set >> 126 MB)"
                  if l2_replicas(n // world if strong else n, p_vis) == 1
                  else f"{l2_replicas(n, p_vis)} independent clouds of this size stepped round "
                       "robin, so each step's rows are L2-cold (>= 4x L2 of traffic between uses)",
            "parallelism": f"index-sharded x{world} ({'strong' if strong else 'weak'})",
            "launch": "one CUDA graph of the K timed steps per rank" if args.graph else "eager"}


L2_BYTES = 126 * 2**20


def l2_replicas(n, p_vis):
    """Clouds needed so that, stepping them round robin, >= 4x L2 of K2
    traffic passes between two steps of the same cloud (1 for big clouds)."""
    touched = max(1.0, n * p_vis * (28 * 59 + 12))
    if touched >= 4 * L2_BYTES:
        return 1
    # at most 64 clouds and ~32 GB of them (a cloud holds ~1.1 KB per row):
    # near-empty masks touch so little that L2 residency no longer matters
    cap = max(1, min(64, int(32e9 // (1100 * max(n, 1)))))
    return min(cap, 1 + math.ceil(4 * L2_BYTES / touched))


# --------------------------------------------------------------- our arm
class Workload:
    """One rank's shard of a benchmark cloud: optimizers (replicas for small
    clouds), gradient records, per-step masks and the RSR / reset samples."""

    def __init__(self, args, wl, p_vis, rank, world, dev, strong, mask, steps, warmup):
        import numpy as np
        import torch

        from paper_2601_16736_b200 import records as R
        from paper_2601_16736_b200 import synthetic as S
        from paper_2601_16736_b200.optimizer import AdamWGS
        from paper_2601_16736_b200.sampling import StSSchedule, shard_rows, stream, stss_sample
        from paper_2601_16736_b200.sharded import ShardedAdamWGS, shard_range

        self.wl, self.world, self.dev, self.args = wl, world, dev, args
        n_total = wl["n"] * (1 if strong else world)
        lo, hi = shard_range(n_total, rank, world)
        n = hi - lo
        self.n, self.n_total, self.lo = n, n_total, lo
        seed = args.seed * 1000 + rank
        self.cfg = S.WorkloadConfig(n=n, p_vis=p_vis, mask_family=mask, seed=seed,
                                    lambda_o=wl["lo"], lambda_s=wl["ls"])
        self.n_rep = l2_replicas(n, p_vis)
        kw = dict(mode=wl["mode"], lambda_o=wl["lo"], lambda_s=wl["ls"], check=args.check,
                  errors="ignore", state_layout=args.layout, state_row_align=args.state_align,
                  adopt=False, fused_compaction=args.fused)
        self.opts, self.shards, self.grad_sets = [], [], []
        for j in range(self.n_rep):
            cj = S.WorkloadConfig(n=n, p_vis=p_vis, mask_family=mask,
                                  seed=seed * 1000 + j if j else seed, lambda_o=wl["lo"],
                                  lambda_s=wl["ls"])
            params = S.make_params_device(cj, dev)
            if args.params == "record":
                _, params = R.pack(params, align=args.record_align)
            if world > 1 or args.sharded:
                sh = ShardedAdamWGS(S.param_groups(params), n_total, **kw)
                self.shards.append(sh)
                self.opts.append(sh.opt)
            else:
                self.opts.append(AdamWGS(S.param_groups(params), **kw))
                self.shards.append(None)
            gs = [S.grads_device(cj, s, dev) for s in range(2 if self.n_rep == 1 else 1)]
            if args.params == "record":
                gs = [R.pack(g, align=args.record_align)[1] for g in gs]
            self.grad_sets.append(gs)
        self.total = warmup + steps
        self.warmup, self.steps = warmup, steps
        self.masks = [S.visibility_device(self.cfg, s, dev) for s in range(self.total)]
        self.n_vis = torch.stack([m.sum() for m in self.masks]).cpu().numpy().astype(np.int64)
        # RSR / relocation samples: host-drawn with the reference RNG contract
        # (optimizer.py:379-386, rng.py:17-30), sliced per shard, uploaded
        # before timing (rank-identical global draws)
        self.events = {}
        sched = StSSchedule(milestones=((0, RSR_RATIO),), interval=RSR_INTERVAL)
        for it in range(self.total):
            boundary = it + 1
            if boundary % RSR_INTERVAL:
                continue
            self.events[it] = self._event(boundary, sched, stss_sample, stream, shard_rows)
        self.rsr_probe = (self._event(RSR_INTERVAL, sched, stss_sample, stream, shard_rows)
                          if (wl["rsr"] or wl["reset"]) else None)

    def _event(self, boundary, sched, stss_sample, stream, shard_rows):
        import numpy as np
        import torch
        ev = {}
        hi = self.lo + self.n
        if self.wl["rsr"]:
            picked = stss_sample(sched, boundary, self.n_total,
                                 stream(self.args.seed, "stss", boundary))
            ev["rsr"] = torch.from_numpy(shard_rows(picked, self.lo, hi).astype(np.int32)).to(
                self.dev)
        if self.wl["reset"]:
            rng = stream(self.args.seed, "relocate", boundary)
            dead = np.sort(rng.choice(self.n_total, int(self.wl["reset"] * self.n_total),
                                      replace=False))
            ev["reset"] = torch.from_numpy(shard_rows(dead, self.lo, hi).astype(np.int32)).to(
                self.dev)
        return ev

    def replica(self, it):
        j = it % self.n_rep
        return self.opts[j], self.shards[j], self.grad_sets[j][it % len(self.grad_sets[j])]

    def apply_events(self, opt, ev):
        if "rsr" in ev:
            opt.rsr_apply(ev["rsr"], ALPHA1, ALPHA2)
        if "reset" in ev:
            opt.reset_rows(ev["reset"])

    def one_step(self, it):
        """The public step (K1 + K2, + the statistics all-reduce on N > 1),
        then K3 on RSR / relocation boundaries."""
        opt, sh, grads = self.replica(it)
        if sh is not None:
            sh.step(self.masks[it], 1_000_000, grads=grads)
        else:
            opt.step(self.masks[it], 1_000_000, grads=grads)
        ev = self.events.get(it)
        if ev:
            self.apply_events(opt, ev)

    def launches(self):
        return sum(o.engine.launches for o in self.opts)


def _prep_capture(w):
    """No outstanding host-side event waits may cross into a capture, and the
    warm-up steps' statistics are read, so the layout hints they carry
    (visible fraction, run length) steer the captured steps as they steer a
    training loop's later steps (without the poll, whether a warm-up step
    had completed when the host issued the next one decides the shape)."""
    import torch
    torch.cuda.synchronize()
    for o in w.opts:
        o.check_errors()
    for sh in w.shards:
        if sh is not None:
            sh.capture_begin()


def _time_steps(w, use_graph):
    """Device time of the K timed steps (CUDA events on the launching stream
    around one graph replay, or around eager launches)."""
    import torch
    import torch.distributed as dist
    timed = range(w.warmup, w.total)
    l0 = w.launches()
    graph = None
    if use_graph:
        _prep_capture(w)
        graph = torch.cuda.CUDAGraph()
        for o in w.opts:
            o._capturing = True
        try:
            with torch.cuda.graph(graph):
                for it in timed:
                    w.one_step(it)
                for sh in w.shards:
                    if sh is not None:
                        sh.wait_stats()  # join the side stream inside the graph
        finally:
            for o in w.opts:
                o._capturing = False
            for sh in w.shards:
                if sh is not None:
                    sh.capture_end()
    launches = w.launches() - l0
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if w.world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start.record()
    if graph is not None:
        graph.replay()
    else:
        for it in timed:
            w.one_step(it)
        launches = w.launches() - l0
    end.record()
    torch.cuda.synchronize()
    if w.world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    del graph
    return ms, launches


def _time_k2(w, use_graph):
    """The dominant kernel alone, for the roofline, launched K times back to
    back (as a graph) between two CUDA events on the launching stream.
    Fused path (the default on records): the one-launch compaction + step
    kernel, i.e. opt.step without the statistics all-reduce or RSR.  Index
    path: K2 on index lists compacted up front.  Returns (ms per launch,
    fused?)."""
    import torch
    timed = list(range(w.warmup, w.total))
    o0 = w.replica(timed[0])[0]
    o0.step(w.masks[timed[0]], 1_000_000, grads=w.replica(timed[0])[2])
    fused = o0._last_ctx[1] is None
    if fused:
        def k2_only():
            for it in timed:
                o, _, grads = w.replica(it)
                o.step(w.masks[it], 1_000_000, grads=grads)
    else:
        idx_lists = []
        for it in timed:
            rows, count = w.replica(it)[0].engine.compact(w.masks[it])
            idx_lists.append((rows.clone(), count.clone()))

        def k2_only():
            for j, it in enumerate(timed):
                o, _, grads = w.replica(it)
                _step_k2(o, grads, idx_lists[j][0], idx_lists[j][1], w.wl)

    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if use_graph:
        g2 = torch.cuda.CUDAGraph()
        for o in w.opts:
            o._capturing = True
        try:
            with torch.cuda.graph(g2):
                k2_only()
        finally:
            for o in w.opts:
                o._capturing = False
        torch.cuda.synchronize()
        k0.record()
        g2.replay()
        k1.record()
    else:
        torch.cuda.synchronize()
        k0.record()
        k2_only()
        k1.record()
    torch.cuda.synchronize()
    return k0.elapsed_time(k1) / len(timed), fused


def _time_rsr(w):
    """Device time of one RSR / reset event (K3) of this workload: the event
    captured as a CUDA graph (its index list is already on the device and
    validated at upload), replayed between two CUDA events."""
    import torch
    if not w.rsr_probe:
        return 0.0
    opt = w.opts[0]
    w.apply_events(opt, w.rsr_probe)  # warm (eager: validates the lists)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(3):
            w.apply_events(opt, w.rsr_probe)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 3


def run_workload(args, wl, p_vis, rank, world, dev, *, strong, mask, steps, warmup, e2e,
                 clocks=None):
    """Time one workload on this rank; every rank returns the same dict
    (times max-reduced over ranks, counts summed)."""
    import torch
    import torch.distributed as dist

    from paper_2601_16736_b200 import synthetic as S
    w = Workload(args, wl, p_vis, rank, world, dev, strong, mask, steps, warmup)
    for it in range(w.warmup):
        w.one_step(it)
    # untimed: every replica steps at least once (small clouds rotate up to
    # 64 replicas), so the statistics its layout hints come from exist
    for j in range(w.warmup, w.n_rep):
        opt, sh, grads = w.opts[j], w.shards[j], w.grad_sets[j][0]
        (sh if sh is not None else opt).step(w.masks[j % len(w.masks)], 1_000_000, grads=grads)
    torch.cuda.synchronize()
    for o in w.opts:
        o.last_stats()  # the visible fraction the optimizer picks its kernel shape by
    use_graph = args.graph
    if clocks is not None:
        with clocks:
            ms, launches = _time_steps(w, use_graph)
    else:
        ms, launches = _time_steps(w, use_graph)
    # the statistics of the last timed step: no skipped rows anywhere
    o_last, sh_last, _ = w.replica(w.total - 1)
    st_vec = (sh_last.wait_stats() if sh_last is not None else o_last.engine.stats).tolist()
    from paper_2601_16736_b200.optimizer import _stats_dict
    st = _stats_dict(st_vec)
    if st["n_bad_grad"] or st["n_bad_domain"] or st["n_stepped"] != st["n_visible"]:
        raise RuntimeError(f"step statistics report skipped rows: {st}")
    k2_ms, fused = _time_k2(w, use_graph)
    rsr_ms = _time_rsr(w)
    # RSR / reset events at their interval: the ones inside the timed window
    # ran; when the window is shorter than the interval the expected share of
    # one event is added from its measured device time
    ev_in = sum(1 for it in range(w.warmup, w.total) if w.events.get(it))
    ev_due = w.steps / RSR_INTERVAL if (wl["rsr"] or wl["reset"]) else 0.0
    extra_ms = max(0.0, ev_due - ev_in) * rsr_ms
    nvis_local = float(w.n_vis[w.warmup:].sum())
    vec = torch.tensor([ms, ms + extra_ms, k2_ms, rsr_ms, nvis_local, float(launches)],
                       dtype=torch.float64, device=dev)
    if world > 1:
        mx = vec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vec.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        vec = torch.cat([mx[:4], sm[4:]])
    ms_max, ms_amort, k2_max, rsr_max, total_visible, launches_all = vec.tolist()
    width = S.SH3_WIDTH
    # algorithmic bytes per launch of the timed kernel: the
    # fused kernel reads the mask (1 B/row) and writes no index list
    per_vis = 28 * width + (8 if fused else 12)
    k2_bytes = [int(nv) * per_vis + (w.n if fused else 0) for nv in w.n_vis[w.warmup:]]
    achieved = (sum(k2_bytes) / len(k2_bytes)) / (k2_ms / 1000.0) / 1e9  # this rank's K2
    peak, peak_src = measured_hbm_peak()
    step_bytes = sum(S.algorithmic_bytes(w.n, int(nv)) for nv in w.n_vis[w.warmup:])
    out = {
        "value": total_visible / (ms_amort / 1000.0),
        "value_no_rsr_amortisation": total_visible / (ms_max / 1000.0),
        "ms_per_step": ms_amort / w.steps, "ms_per_step_timed": ms_max / w.steps,
        "rsr_events_timed": ev_in, "rsr_ms_per_event": rsr_max,
        "rsr_amortised_ms": extra_ms, "visible_per_step": total_visible / w.steps,
        "gpu_launches": int(launches_all),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "k2_ms_avg": k2_ms, "k2_ms_max_over_ranks": k2_max,
                     "k2_bytes_per_launch": sum(k2_bytes) / len(k2_bytes),
                     "bytes_per_visible": per_vis, "bytes_per_row": 1 if fused else 0,
                     "fused_compaction": fused, "peak_source": peak_src,
                     "step_gbs_algorithmic": step_bytes / (ms / 1000.0) / 1e9,
                     "step_frac": step_bytes / (ms / 1000.0) / 1e9 / peak,
                     # the north star's phrasing: against the nominal ~8 TB/s
                     "frac_of_nominal_8tbs": achieved / NOMINAL_HBM_GBS},
        "config": workload_config(args, wl, p_vis, world, strong, mask),
    }
    if e2e:
        out["e2e"] = run_e2e(args, w, dev, world)
    del w
    torch.cuda.empty_cache()
    return out


def ours(args, wl, p_vis):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.sharded:
        # communicator lines (rank / nranks) for the driver's rank check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    clk = ClockSampler(local)
    main = run_workload(args, wl, p_vis, rank, world, dev, strong=args.strong, mask=args.mask,
                        steps=args.steps, warmup=args.warmup, e2e=not args.no_e2e, clocks=clk)
    legs = {}
    if not args.no_legs:
        c5 = dict(WORKLOADS["c5"], name="c5")
        for p, key in ((0.3, "c5_strong"), (0.01, "c5_strong_1pct")):
            r = run_workload(args, c5, p, rank, world, dev, strong=True, mask="bernoulli",
                             steps=min(args.steps, 20), warmup=max(3, min(args.warmup, 5)),
                             e2e=False)
            legs[key] = {"metric": "visible Gaussians updated/sec per optimizer step",
                         "value": r["value"], "unit": "visible Gaussians/s",
                         "ms_per_step": r["ms_per_step"], "n_gpus": world, "scaling": "strong",
                         "steps": min(args.steps, 20),
                         "roofline": {k: r["roofline"][k] for k in ("achieved", "peak", "frac",
                                                                    "k2_ms_avg", "step_frac")},
                         "gpu_launches": r["gpu_launches"], "config": r["config"]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = host_workers()
        v, sample, _, _ = cpu_reference_rate(wl, p_vis, args.mask, budget_s=args.cpu_seconds,
                                              seed=args.seed, workers=cores)
        cpu = {"value": v, "unit": "visible Gaussians/s", "cores": cores, "kind": "port",
               "sample": sample, "host_cpus": os.cpu_count()}
    if rank == 0:
        roof = dict(main["roofline"])
        roof.update({
            "traffic": traffic_from_profiles(
                args.workload, args.mask, p_vis,
                args.params if args.params != "record" or
                (args.record_align, args.state_align) == (16, 16) else
                f"record-a{args.record_align}-s{args.state_align}"),
            "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set "
                              "full capture of this K2 configuration (profiles/traffic.json; "
                              "not measured in this run)",
            "kernel": ("gs::step_kernel (K2, gs_step)" if args.layout != "rows" else
                       ("gs::step_tma4_kernel<LayoutSH3, ..., MASK=1> (K1 fused into K2: the "
                        "loader compacts the mask; 2-D TMA gather4 / scatter4 on the records; "
                        "via gs_step_rows_masked; on clouds under ~4.8M rows coherent masks "
                        "and coupled sparse-adam take MASK=3, the two-phase variant)"
                        if main["roofline"].get("fused_compaction")
                        else "gs::step_tma4_kernel<LayoutSH3, ...> (K2 on the K1 index list, "
                        "2-D TMA gather4 / scatter4, via gs_step_rows)")
                       if args.params == "record" else
                       "gs::step_ws_kernel<LayoutSH3> (K2, per-attribute gathers, via "
                       "gs_step_rows)")})
        line = {
            "metric": "visible Gaussians updated/sec per optimizer step",
            "value": main["value"], "unit": "visible Gaussians/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian cloud, SURVEY §8(d) distributions)",
            "config": dict(main["config"],
                           rsr_timing=f"{main['rsr_events_timed']} RSR event(s) inside the timed "
                                      f"window; {main['rsr_amortised_ms']:.4f} ms added = one "
                                      f"measured event ({main['rsr_ms_per_event']:.4f} ms) x "
                                      f"(K / {RSR_INTERVAL} - events timed)"),
            "roofline": roof, "e2e": main.get("e2e"), "gpu_launches": main["gpu_launches"],
            "clocks": clk.summary(), "cpu_baseline": cpu,
            "visible_per_step": main["visible_per_step"],
            "ms_per_step_timed": main["ms_per_step_timed"],
            "value_no_rsr_amortisation": main["value_no_rsr_amortisation"],
            "legs": legs or None,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def _step_k2(opt, grads, rows, count, wl):
    """The optimizer's K2 launch for an already-compacted index list
    (AdamWGS.step does K1 + K2; the bench splits them to time K2 alone).
    Graph-capturable: no host synchronisation, no error readback."""
    b = opt._bindings(grads)
    eng = opt.engine
    from paper_2601_16736_b200.engine import round_pixel_count
    if wl["mode"] == "adamw-gs":
        eng.step(b, "adamw-gs", opt.state.clock, rows=rows, count=count, eps=opt.eps,
                 lambda_opacity=wl["lo"], lambda_scale=wl["ls"], clip_opacity=opt.ct_opacity,
                 clip_scale=opt.ct_scale, n_pixels_rounded=round_pixel_count(1_000_000),
                 check=opt.check, record=opt.state.record)
    else:
        eng.step(b, wl["mode"], opt.state.clock, rows=rows, count=count, eps=opt.eps,
                 lambda_opacity=wl["lo"], lambda_scale=wl["ls"], n_visible_dev=count,
                 check=opt.check, record=opt.state.record)
    opt._last_ctx = (b, rows, count, wl["lo"], wl["ls"], wl["mode"], None)


def run_e2e(args, w, dev, world):
    """Public-API step with host buffers, every step: H2D copy of that step's
    mask from pinned memory (a fresh mask per step), the step (through
    ShardedAdamWGS on N > 1) with the gradients in pinned host memory, D2H
    read of the step statistics.  Default: the step kernel gathers the
    visible rows' gradients zero-copy over PCIe (only N_v rows cross the
    bus).  The dense-copy variant (every gradient row copied H2D first) is
    timed too and reported as ``dense_copy``."""
    import torch
    import torch.distributed as dist

    from paper_2601_16736_b200 import records as R
    opt, sh, _ = w.replica(0)
    like = {g["name"]: g["params"][0] for g in opt.param_groups}
    if args.params == "record":
        # one pinned gradient record; rows padded to 256 B = two 128-byte
        # lines, the granule the zero-copy reads cross PCIe in
        host_rec, host_grads = R.pack({k: torch.zeros(t.shape) for k, t in like.items()},
                                      align=args.host_record_align, pin_memory=True)
        dev_grads = R.views_like(torch.empty_like(host_rec, device=dev), like)
        host_dense = [host_rec]
        dev_dense = [dev_grads[next(iter(dev_grads))]._base]
        row_bytes = host_rec.shape[1] * 4
    else:
        host_grads = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                      for k, t in like.items()}
        dev_grads = {k: torch.empty_like(t) for k, t in like.items()}
        host_dense = list(host_grads.values())
        dev_dense = list(dev_grads.values())
        row_bytes = sum(t[0].numel() * 4 for t in host_grads.values())
    for t in host_grads.values():
        t.copy_(torch.randn(t.shape) * 1e-4)
    n_steps = max(1, args.e2e_steps)
    n_masks = min(n_steps, len(w.masks))
    host_masks = []
    for j in range(n_masks):
        hm = torch.empty(w.masks[j].shape, dtype=torch.bool, pin_memory=True)
        hm.copy_(w.masks[j].cpu())
        host_masks.append(hm)
    mask_vis = [float(m.sum()) for m in host_masks]
    dev_mask = torch.empty_like(w.masks[0])
    from paper_2601_16736_b200 import _lib as L
    stats_host = torch.empty(L.GS_STEP_STATS, dtype=torch.float64, pin_memory=True)
    dense = sum(t.numel() * 4 for t in host_dense)
    d2h = stats_host.numel() * 8
    step = sh.step if sh is not None else opt.step

    def one(j, zero_copy):
        dev_mask.copy_(host_masks[j % n_masks], non_blocking=True)
        if zero_copy:
            grads = host_grads
        else:
            for d, h in zip(dev_dense, host_dense):
                d.copy_(h, non_blocking=True)
            grads = dev_grads
        step(dev_mask, 1_000_000, grads=grads)
        st = sh.wait_stats() if sh is not None else opt.engine.stats
        stats_host.copy_(st, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def timed(zero_copy):
        for j in range(2):
            one(j, zero_copy)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for j in range(n_steps):
            one(j, zero_copy)
        ms = (time.perf_counter() - t0) * 1000.0 / n_steps
        ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        return float(ms_t.item())

    nv = sum(mask_vis[j % n_masks] for j in range(n_steps)) / n_steps
    nv_t = torch.tensor([nv], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(nv_t)
    nv_all = float(nv_t.item())
    ms_dense = timed(False)
    ms = timed(True)
    return {"value": nv_all / (ms / 1000.0), "unit": "visible Gaussians/s",
            "h2d_bytes_per_step": int(host_masks[0].numel() + nv * row_bytes),
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": n_steps,
            "masks": f"{n_masks} distinct pinned host masks, one per step (cycled)",
            "h2d_mode": "mask copied H2D; gradients gathered zero-copy from pinned host "
                        "memory by the step kernel (visible rows only)",
            "timing": "host wall clock around H2D + step + D2H + sync, max over ranks",
            "dense_copy": {"value": nv_all / (ms_dense / 1000.0), "ms_per_step": ms_dense,
                           "h2d_bytes_per_step": int(host_masks[0].numel() + dense)}}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args) -> int:
    """``--gpus N`` outside torchrun: start N ranks on this node."""
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}",
              file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    wl = dict(WORKLOADS[args.workload], name=args.workload)
    if args.rows is not None:
        wl["n"] = args.rows
    p_vis = args.vis if args.vis is not None else wl["p"]
    if args.impl == "reference":
        reference_arm(args, wl, p_vis)
        return
    ours(args, wl, p_vis)


if __name__ == "__main__":
    main()
