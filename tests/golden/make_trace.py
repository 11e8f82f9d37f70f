"""Golden trace: the reference's own training loop driving its optimizer.

Runs the UNMODIFIED reference ``run_training`` (pipeline.py:258-381) on the
TINY configuration of R/pkg/tests/test_pipeline.py:17-24 (32x32 canvas, 40
iterations, densification and relocation boundaries) in several optimizer
modes, and records every call the loop makes into the optimizer module —
``adam_step_sync``, ``sparse_adam_step``, ``dar_step``, ``adamw_const_step``,
``rsr_apply``, ``reset_rows``, ``aiu_apply`` — with its inputs (primitive
set, moment state, gradients from the real renderer, visibility mask,
scalars, the AIU generator's state) and its outputs.  The calls are wrapped
(monkeypatched names in ``splatlab.pipeline``), never changed.

tests/test_gpu_trace.py replays every recorded call through
paper_2601_16736_b200.reference_api on CUDA tensors and compares with the
recorded outputs.  This script needs /root/reference (this container only);
the .npz it writes travels with the repo.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_trace.py
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path(os.environ.get("SPLATLAB_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF_SRC))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba-cache")
sys.dont_write_bytecode = True

import splatlab.pipeline as PL  # noqa: E402
from splatlab.config import default_config  # noqa: E402

OUT = Path(__file__).resolve().parent / "trace_tiny.npz"
GROUPS = ("mu", "kappa", "rot", "tau", "color")

# R/pkg/tests/test_pipeline.py:17-24
TINY = {
    "scene.canvas": 32, "scene.gt_count": 8, "scene.redundancy": 1.0,
    "scene.crop_size": 16, "scene.crops_x": 2, "scene.crops_y": 2,
    "stages.warmup_end": 4, "stages.densify_end": 20, "stages.total_iters": 40,
    "stages.densify_interval": 4, "stages.reset_interval": 10,
    "densify.max_primitives": 64, "run.metrics_interval": 10,
    "run.dar_opacity_start": 6,
}
RUNS = {
    # AdamW-GS with DAR, RSR, AIU and position noise
    "gs": {"optimizer.mode": "adamw-gs", "optimizer.lambda_o": 1e-3, "optimizer.lambda_s": 1e-5,
           "rsr.enabled": True, "rsr.milestones": "0:0.25", "rsr.interval": 4,
           "aiu.enabled": True, "aiu.start": 0, "aiu.end": 30, "aiu.prob": "0:0.3",
           "aiu.eta": "0:0.5", "noise.enabled": True},
    # sparse Adam + coupled L1 (the "opacity decay" baseline)
    "sparse": {"optimizer.mode": "sparse-adam", "optimizer.lambda_o": 0.01},
    # synchronous Adam + coupled L1 on every row
    "coupled": {"optimizer.mode": "coupled-adam", "optimizer.lambda_o": 0.01,
                "optimizer.lambda_s": 0.001},
    # MCMC relocation (reset_rows) with the constant clipped penalty
    "mcmc": {"optimizer.mode": "adamw-const-clip", "optimizer.lambda_o": 0.01,
             "optimizer.lambda_s": 0.001, "densify.relocation": True, "rsr.enabled": True,
             "rsr.milestones": "0:0.25", "rsr.interval": 8},
}


def main():
    arrays, calls = {}, []
    orig = {name: getattr(PL, name) for name in
            ("adam_step_sync", "sparse_adam_step", "dar_step", "adamw_const_step", "rsr_apply",
             "reset_rows", "aiu_apply")}
    cur = {"run": None}

    def put(key, a):
        arrays[key] = np.array(a, copy=True)

    def snap(prefix, state=None, pset=None, grads=None):
        if pset is not None:
            for g in GROUPS:
                put(f"{prefix}_p_{g}", getattr(pset, g))
            put(f"{prefix}_alive", pset.alive)
        if state is not None:
            for g in GROUPS:
                put(f"{prefix}_m_{g}", state.m[g])
                put(f"{prefix}_v_{g}", state.v[g])
            put(f"{prefix}_t", state.t[GROUPS[0]])
        if grads is not None:
            for g in GROUPS:
                put(f"{prefix}_g_{g}", getattr(grads, g))

    def wrap(name):
        fn = orig[name]

        def wrapped(*args, **kw):
            i = len(calls)
            rec = {"run": cur["run"], "fn": name}
            p = f"c{i}"
            if name in ("adam_step_sync", "sparse_adam_step", "dar_step", "adamw_const_step"):
                state, pset, grads = args[0], args[1], args[2]
                rest = list(args[3:])
                kwp = dict(kw)  # parsed copy; the call gets the caller's arguments unchanged
                if name != "adam_step_sync":
                    put(f"{p}_vis", rest.pop(0))
                rest.pop(0)  # cfg (recorded once per run)
                if name == "dar_step":
                    rec["n_pixels"] = int(rest.pop(0)) if rest else int(kwp.pop("n_pixels"))
                if name == "adamw_const_step":
                    clip = rest.pop(0) if rest else kwp.pop("clip", None)
                    rec["clip"] = None if clip is None else float(clip)
                rec["mu_lr_scale"] = float(rest.pop(0)) if rest else float(kwp.pop("mu_lr_scale", 1.0))
                for k in ("lambda_o", "lambda_s"):
                    if k in kwp:
                        rec[k] = None if kwp[k] is None else float(kwp[k])
                rec["global_t"] = int(state.global_t)
                snap(f"{p}_in", state, pset, grads)
                out = fn(*args, **kw)
                snap(f"{p}_out", state, pset)
                rec["global_t_out"] = int(state.global_t)
            elif name in ("rsr_apply", "reset_rows"):
                state, idx = args[0], args[1]
                put(f"{p}_idx", idx)
                if name == "rsr_apply":
                    rec["alpha1"], rec["alpha2"] = float(args[2]), float(args[3])
                snap(f"{p}_in", state)
                out = fn(*args, **kw)
                snap(f"{p}_out", state)
            else:  # aiu_apply(state, pset, vis, cfg, aiu, rng, iteration)
                state, pset, vis, _cfg, aiu, rng, it = args
                rec["iteration"] = int(it)
                rec["aiu"] = {"start": aiu.start, "end": aiu.end,
                              "prob": list(map(list, aiu.prob_schedule)),
                              "eta": list(map(list, aiu.eta_schedule))}
                rec["rng_state"] = _jsonable(rng.bit_generator.state)
                put(f"{p}_vis", vis)
                snap(f"{p}_in", state, pset)
                out = fn(*args, **kw)
                put(f"{p}_picked", out)
                snap(f"{p}_out", state, pset)
            calls.append(rec)
            return out
        return wrapped

    meta = {"runs": {}, "tiny": TINY}
    for name in orig:
        setattr(PL, name, wrap(name))
    try:
        for run, extra in RUNS.items():
            cur["run"] = run
            cfg = default_config().with_overrides({**TINY, **extra})
            n0 = len(calls)
            res = PL.run_training(cfg)
            o = cfg.optimizer
            meta["runs"][run] = {
                "overrides": {k: (v if not isinstance(v, bool) else str(v).lower())
                              for k, v in extra.items()},
                "optimizer": {k: getattr(o, k) for k in (
                    "mode", "beta1", "beta2", "eps", "lr_mu", "lr_tau", "lr_kappa", "lr_rot",
                    "lr_color", "lambda_o", "lambda_s", "ct_opacity", "ct_scale",
                    "round_n_pixels")},
                "calls": [n0, len(calls)], "events": len(res.events),
                "final_psnr": float(res.metrics[-1].psnr) if res.metrics else None,
            }
    finally:
        for name, fn in orig.items():
            setattr(PL, name, fn)
    meta["calls"] = calls
    np.savez_compressed(OUT, meta=json.dumps(meta), **arrays)
    kinds = {}
    for c in calls:
        kinds[(c["run"], c["fn"])] = kinds.get((c["run"], c["fn"]), 0) + 1
    print(OUT, len(calls), "calls", {f"{a}/{b}": n for (a, b), n in sorted(kinds.items())},
          f"{OUT.stat().st_size / 1e6:.2f} MB")


def _jsonable(x):
    if isinstance(x, dict):
        return {k: _jsonable(v) for k, v in x.items()}
    if isinstance(x, np.ndarray):
        return [int(v) for v in x.tolist()]
    if isinstance(x, (np.integer,)):
        return int(x)
    return x


if __name__ == "__main__":
    main()
