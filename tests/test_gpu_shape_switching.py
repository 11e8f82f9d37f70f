"""Kernel-shape switching over many steps (marked gpu).

The optimizer picks the fused step's shape per step from the statistics of
earlier steps (visible fraction, run length): the streaming loader on tiles
or per-CTA slices, with or without the bias warp, the 3-CTA sparse shape,
the dynamic tail (whose claim counter the last CTA re-arms), the two-phase
kernel (whose grid barrier re-arms) and the index path for coherent masks.
Here the visibility changes every step (1% .. 60%, i.i.d. or in coherent
blocks), so consecutive launches switch shapes in every order; the final
parameters, moments and clocks must equal a run on the index path (K1 + K2)
bit for bit, and every step's visible count must match the mask's.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _masks(n, steps, seed):
    rng = np.random.default_rng(seed)
    out = []
    for s in range(steps):
        p = float(rng.choice([0.01, 0.03, 0.1, 0.3, 0.6]))
        if rng.random() < 0.3:  # coherent blocks of 64 rows
            nb = -(-n // 64)
            m = np.repeat(rng.random(nb) < p, 64)[:n]
        else:
            m = rng.random(n) < p
        out.append(m)
    return out


@pytest.mark.parametrize("n,mode", [(300_007, "adamw-gs"), (2_000_003, "adamw-gs"),
                                    (1_000_003, "sparse-adam"), (6_000_011, "adamw-const"),
                                    (20_000_003, "adamw-gs")])
def test_shape_switching_equals_index_path(n, mode):
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS
    steps = 40 if n < 5_000_000 else 16 if n < 10_000_000 else 10
    cfg = S.WorkloadConfig(n=n, p_vis=0.3, seed=n % 83 + 1)
    base = S.make_params_device(cfg, torch.device(DEV))
    masks = [torch.from_numpy(m).to(DEV) for m in _masks(n, steps, n % 7)]
    outs = []
    for fused in (True, False):
        _, params = R.pack({k: v.clone() for k, v in base.items()})
        opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=1e-3, lambda_s=1e-5,
                      fused_compaction=fused)
        grec, grads = R.pack({k: torch.zeros_like(v) for k, v in base.items()})
        for s in range(steps):
            for k, x in S.grads_device(cfg, s, torch.device(DEV), masks[s]).items():
                grads[k].copy_(x)
            opt.step(masks[s], cfg.n_pixels, grads=grads)
            if s % 3 == 2:  # the statistics (and layout hints) are read now and then
                st = opt.last_stats()
                assert st["n_visible"] == int(masks[s].sum().item())
        opt.check_errors()
        torch.cuda.synchronize()
        outs.append(({k: p.cpu().numpy() for k, p in params.items()},
                     opt.state.record.cpu().numpy()))
    (pa, ra), (pb, rb) = outs
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k
    assert np.array_equal(ra.view(np.int32), rb.view(np.int32))
