"""Host cost of an eager AdamWGS.step (the drop-in call a training loop
makes): steps issued back to back without graphs, wall time per step vs the
device time per step, on small and mid clouds.

    python scripts/eager_overhead.py
"""

import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402


def run(n, p, k=200, **kw):
    dev = torch.device("cuda:0")
    cfg = S.WorkloadConfig(n=n, p_vis=p, seed=1)
    _, params = R.pack(S.make_params_device(cfg, dev))
    _, grads = R.pack(S.grads_device(cfg, 0, dev))
    opt = AdamWGS(S.param_groups(params), mode="adamw-gs", lambda_o=1e-3, lambda_s=1e-5, **kw)
    vis = S.visibility_device(cfg, 0, dev)
    for _ in range(20):
        opt.step(vis, cfg.n_pixels, grads=grads)
    opt.check_errors()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(k):
        opt.step(vis, cfg.n_pixels, grads=grads)
    t_issue = time.perf_counter() - t0
    b.record()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t0
    opt.check_errors()
    dev_ms = a.elapsed_time(b) / k
    print(f"n={n:>9} p={p}: host issue {t_issue / k * 1e6:7.1f} us/step, wall {t_wall / k * 1e6:7.1f} "
          f"us/step, device {dev_ms * 1e3:7.1f} us/step  {kw}")


if __name__ == "__main__":
    for n, p in ((100_000, 0.5), (1_000_000, 0.3), (6_000_000, 0.3)):
        run(n, p)
    run(100_000, 0.5, errors="ignore")
