import cProfile, pstats, sys, torch
sys.path.insert(0, ".")
from paper_2601_16736_b200 import records as R, synthetic as S
from paper_2601_16736_b200.optimizer import AdamWGS
dev = torch.device("cuda", 0)
cfg = S.WorkloadConfig(n=10_000, p_vis=0.3, seed=1)
_, params = R.pack(S.make_params_device(cfg, dev)); _, grads = R.pack(S.grads_device(cfg, 0, dev))
vis = S.visibility_device(cfg, 0, dev)
opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5, errors="defer")
for _ in range(20): opt.step(vis, cfg.n_pixels, grads=grads)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(300): opt.step(vis, cfg.n_pixels, grads=grads)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
