"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): K1, K2 (TMA records, the cp.async ring via
GS_FIXED_VARIANT=21 in a second run, per-attribute tensors), the strict
check, K3 (RSR, reset), K4, AIU, relocation, noise.

    compute-sanitizer --tool racecheck python scripts/sanitize.py
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.noise import NoiseConfig  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402
from paper_2601_16736_b200.sampling import AiuConfig  # noqa: E402
from paper_2601_16736_b200.structural import mcmc_plan  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    cfg = S.WorkloadConfig(n=20_011, p_vis=0.3, seed=9)
    host = S.make_params(cfg)
    for layout in ("record", "attr"):
        for check in ("fused", "strict"):
            params = {k: torch.from_numpy(v).to(dev) for k, v in host.items()}
            if layout == "record":
                _, params = R.pack(params)
            opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3,
                          lambda_s=1e-5, check=check)
            for s in range(3):
                vis = S.visibility(cfg, s)
                g = {k: torch.from_numpy(x).to(dev) for k, x in S.step_grads(cfg, s, vis).items()}
                if layout == "record":
                    _, g = R.pack(g)
                opt.step(torch.from_numpy(vis).to(dev), cfg.n_pixels, grads=g)
            opt.check_errors()
            opt.rsr_apply(np.arange(0, cfg.n, 3), 0.2, 0.04)
            opt.reset_rows(np.arange(0, cfg.n, 50))
            opt.moment_stats()
            if layout == "record":
                vis_t = torch.from_numpy(S.visibility(cfg, 0)).to(dev)
                opt.aiu_apply(vis_t, AiuConfig(start=0, end=10, prob_schedule=((0, 0.3),),
                                               eta_schedule=((0, 0.5),), enabled=True),
                              np.random.default_rng(0), 2)
                plan = mcmc_plan(params["opacity"].reshape(-1).cpu().numpy(), None,
                                 np.random.default_rng(1))
                opt.relocate_rows(plan)
                opt.noise_perturb(1e-4, NoiseConfig(enabled=True), 3, 1)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
