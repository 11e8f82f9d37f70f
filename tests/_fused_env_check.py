"""Subprocess body of tests/test_gpu_fused_variants.py: with the library's
measurement switches in the environment (read once per process), the fused
step equals K1 + K2 bit for bit on one cloud.  argv: n kind mode p"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_16736_b200 import records as R  # noqa: E402
from paper_2601_16736_b200 import synthetic as S  # noqa: E402
from paper_2601_16736_b200.optimizer import AdamWGS  # noqa: E402


def main(n, kind, mode, p):
    dev = torch.device("cuda:0")
    cfg = S.WorkloadConfig(n=n, p_vis=p, seed=n % 97 + 1)
    base = S.make_params_device(cfg, dev)  # device-generated: big clouds in seconds
    outs = []
    for fused in (True, False):
        _, params = R.pack({k: v.clone() for k, v in base.items()})
        lo, ls = (1e-3, 1e-5)
        opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=lo, lambda_s=ls,
                      fused_compaction=fused)
        stats = []
        for s in range(2):
            vis = S.visibility_device(cfg, s, dev)
            m = (torch.where(vis, torch.arange(n, device=dev, dtype=torch.int32) % 7 + 1, 0)
                 .to(torch.int32).contiguous() if kind == "radii" else vis)
            _, g = R.pack(S.grads_device(cfg, s, dev, vis))
            opt.step(m, cfg.n_pixels, grads=g)
            assert (opt._last_ctx[1] is None) == fused, "path"
            stats.append(opt.last_stats())
        opt.check_errors()
        outs.append(({k: q.cpu().numpy() for k, q in params.items()},
                     opt.state.record.cpu().numpy(), stats))
    (pa, ra, sa), (pb, rb, sb) = outs
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k
    assert np.array_equal(ra.view(np.int32), rb.view(np.int32))
    for x, y in zip(sa, sb):
        for f in x:
            if f != "n_runs" and not f.startswith("sum_"):
                assert x[f] == y[f], f
    print("ok")


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2], sys.argv[3], float(sys.argv[4]))
