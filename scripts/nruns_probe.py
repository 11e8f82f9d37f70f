import numpy as np, torch
from paper_2601_16736_b200 import synthetic as S, records as R
from paper_2601_16736_b200.optimizer import AdamWGS
for n, fused in [(4133, True), (4133, False), (100_000, True), (100_000, False), (6_000_000, True)]:
    cfg = S.WorkloadConfig(n=n, p_vis=0.5, seed=3)
    host = S.make_params(cfg)
    _, params = R.pack({k: torch.from_numpy(v).cuda() for k, v in host.items()})
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5, fused_compaction=fused)
    vis = S.visibility(cfg, 0)
    _, g = R.pack({k: torch.from_numpy(x).cuda() for k, x in S.step_grads(cfg, 0, vis).items()})
    opt.step(torch.from_numpy(vis).cuda(), cfg.n_pixels, grads=g)
    st = opt.last_stats()
    print(n, fused, opt._last_ctx[1] is None, st["n_visible"], st["n_runs"])
