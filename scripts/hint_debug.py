import sys, torch
sys.path.insert(0, ".")
from paper_2601_16736_b200 import records as R, synthetic as S
from paper_2601_16736_b200.optimizer import AdamWGS
dev = torch.device("cuda:0")
cfg = S.WorkloadConfig(n=100_000, p_vis=0.5, seed=1)
_, params = R.pack(S.make_params_device(cfg, dev))
_, grads = R.pack(S.grads_device(cfg, 0, dev))
opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
vis = S.visibility_device(cfg, 0, dev)
orig = opt.engine.step_masked
def sm(*a, **k):
    print("step_masked low", k.get("low_visibility"), "coherent", k.get("coherent"), "balance", k.get("balance_tail"))
    return orig(*a, **k)
opt.engine.step_masked = sm
for i in range(3):
    opt.step(vis, cfg.n_pixels, grads=grads)
    opt.check_errors()
    print("vis_frac", opt._vis_frac, "vis_run", opt._vis_run, opt.last_stats())
