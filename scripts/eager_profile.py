"""cProfile of eager AdamWGS.step at c1 (host overhead breakdown)."""

import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402

dev = torch.device("cuda:0")
cfg = S.WorkloadConfig(n=100_000, p_vis=0.5, seed=1)
_, params = R.pack(S.make_params_device(cfg, dev))
_, grads = R.pack(S.grads_device(cfg, 0, dev))
opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5)
vis = S.visibility_device(cfg, 0, dev)
for _ in range(50):
    opt.step(vis, cfg.n_pixels, grads=grads)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    opt.step(vis, cfg.n_pixels, grads=grads)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
