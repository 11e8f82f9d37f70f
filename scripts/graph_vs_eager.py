"""Public-API step latency, eager opt.step() vs a captured StepGraph.replay(),
for small clouds where host launch overhead matters (run on a GPU box)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for n in (10_000, 100_000, 1_000_000):
        cfg = S.WorkloadConfig(n=n, p_vis=0.3, seed=1)
        _, params = R.pack(S.make_params_device(cfg, dev))
        _, grads = R.pack(S.grads_device(cfg, 0, dev))
        vis = S.visibility_device(cfg, 0, dev)
        res = {}
        for how in ("eager", "graph"):
            opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5,
                          errors="defer")
            g = opt.capture(vis, cfg.n_pixels, grads=grads) if how == "graph" else None
            step = (lambda: g.replay()) if g else (lambda: opt.step(vis, cfg.n_pixels, grads=grads))
            for _ in range(20):
                step()
            torch.cuda.synchronize()
            k = 500
            t0 = time.perf_counter()
            for _ in range(k):
                step()
            torch.cuda.synchronize()
            res[how] = (time.perf_counter() - t0) / k * 1e6
            opt.check_errors()
        print(f"n={n:>9,d}  eager {res['eager']:7.1f} us/step  graph {res['graph']:7.1f} us/step  "
              f"x{res['eager'] / res['graph']:.2f}", flush=True)


if __name__ == "__main__":
    main()
