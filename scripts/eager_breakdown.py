"""Host time per eager step split into the deferred-check pieces (c1)."""

import sys
import time
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
acc = {"_poll": 0.0, "_enqueue_check": 0.0}
cnt = {"_poll": 0, "_enqueue_check": 0, "blocking": 0}
orig_poll, orig_enq = opt._poll, opt._enqueue_check


def poll(block, limit=None):
    t = time.perf_counter()
    if block:
        cnt["blocking"] += 1
    r = orig_poll(block, limit)
    acc["_poll"] += time.perf_counter() - t
    cnt["_poll"] += 1
    return r


def enq():
    t = time.perf_counter()
    r = orig_enq()
    acc["_enqueue_check"] += time.perf_counter() - t
    cnt["_enqueue_check"] += 1
    return r


opt._poll, opt._enqueue_check = poll, enq
for _ in range(50):
    opt.step(vis, cfg.n_pixels, grads=grads)
opt.check_errors()
torch.cuda.synchronize()
for k in acc:
    acc[k] = 0.0
cnt.update({"_poll": 0, "_enqueue_check": 0, "blocking": 0})
K = 2000
t0 = time.perf_counter()
for _ in range(K):
    opt.step(vis, cfg.n_pixels, grads=grads)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"per step: total {(t1 - t0) / K * 1e6:.1f} us, _poll {acc['_poll'] / K * 1e6:.1f} us "
      f"({cnt['_poll']} calls, {cnt['blocking']} blocking), _enqueue_check "
      f"{acc['_enqueue_check'] / K * 1e6:.1f} us")
