"""Drop-in path timing on one B200: the c3 workload (6M SH-3 Gaussians, 30%
i.i.d. visibility, adamw-gs) stepped through the public API with gradients
read from ``p.grad`` of per-attribute ``nn.Parameter``s: the default
construction (``adopt="auto"``: AdamWGS re-homes them into records) and
``adopt=False`` (per-attribute gathers).  Eager ``opt.step(mask, n_pixels)`` calls, 10 warm-up and
50 timed steps between CUDA events, fresh mask per step (pre-generated).

usage: python scripts/adopt_bench.py [n]"""

import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402


def run(adopt: bool, n: int, warm: int = 10, steps: int = 50) -> dict:
    dev = torch.device("cuda", 0)
    cfg = S.WorkloadConfig(n=n, p_vis=0.3, seed=0)
    params = {k: torch.nn.Parameter(t) for k, t in S.make_params_device(cfg, dev).items()}
    grads = S.grads_device(cfg, 0, dev)
    for k, p in params.items():
        p.grad = grads[k].view(p.shape).clone()
    del grads
    # reference-style construction; the default adopt="auto" re-homes the
    # Parameters (and their .grad) into records
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=cfg.lambda_o,
                  lambda_s=cfg.lambda_s, adopt="auto" if adopt else False)
    assert (opt.param_record is not None) == adopt
    masks = [S.visibility_device(cfg, s, dev) for s in range(warm + steps)]
    n_vis = sum(int(m.sum()) for m in masks[warm:])
    for s in range(warm):
        opt.step(masks[s], cfg.n_pixels)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in range(warm, warm + steps):
        opt.step(masks[s], cfg.n_pixels)
    b.record()
    torch.cuda.synchronize()
    opt.check_errors()
    ms = a.elapsed_time(b) / steps
    st = opt.last_stats()
    assert st["n_stepped"] == st["n_visible"], st
    return {"params": "per-attribute nn.Parameters, AdamWGS(adopt='auto') (default)" if adopt
            else "per-attribute nn.Parameters, AdamWGS(adopt=False)",
            "n": n, "ms_per_step": ms, "visible_per_s": n_vis / steps / (ms / 1e3)}


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6_000_000
    for adopt in (False, True):
        print(json.dumps(run(adopt, n)))
        torch.cuda.empty_cache()
