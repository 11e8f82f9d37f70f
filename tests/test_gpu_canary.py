"""Out-of-bounds write canaries for the device kernels (marked gpu).

compute-sanitizer cannot run on this GPU pool, so the
bounds of every writing kernel are checked directly: the parameter, gradient
and moment records live in the middle of buffers filled with a NaN bit
pattern, the records' pad columns hold the same pattern, and after steps on
every path (streaming fused on per-CTA mask slices and on tiles dealt
grid-stride, two-phase, the bias-warp and 3-CTA sparse shapes, the index
path, the strict check) and the operations around the step (RSR, reset,
AIU, position noise, MCMC relocation) every canary word must be unchanged:
the 2-D TMA boxes end at the 480-byte moment span and the 256-byte
parameter row, and no kernel writes a row outside [0, n).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
CANARY = 0x7FC0DEAD  # a quiet-NaN bit pattern no kernel produces
PAD_ROWS = 67


def _canary_rows(n, width):
    buf = torch.full((n + 2 * PAD_ROWS, width), CANARY, dtype=torch.int32, device=DEV)
    return buf, buf.view(torch.float32)[PAD_ROWS:PAD_ROWS + n]


def _check(buf, n, used_cols, what):
    b = buf.cpu().numpy()
    assert (b[:PAD_ROWS] == CANARY).all(), f"{what}: rows before the record written"
    assert (b[PAD_ROWS + n:] == CANARY).all(), f"{what}: rows after the record written"
    assert (b[PAD_ROWS:PAD_ROWS + n, used_cols:] == CANARY).all(), f"{what}: pad columns written"


def _setup(n, p, mode, fused, check="fused", lo=1e-3, ls=1e-5):
    from paper_2601_16736_b200 import records as R
    from paper_2601_16736_b200 import synthetic as S
    from paper_2601_16736_b200.optimizer import AdamWGS, MomentState
    cfg = S.WorkloadConfig(n=n, p_vis=p, seed=n % 89 + 2)
    host = S.make_params_device(cfg, DEV)  # device-generated (big clouds)
    shapes = {k: tuple(v.shape[1:]) for k, v in host.items()}
    pbuf, prec = _canary_rows(n, 64)
    params = R.views(prec, shapes)
    for k, v in host.items():
        params[k].copy_(v)
    del host
    gbuf, grec = _canary_rows(n, 64)
    grads = R.views(grec, shapes)
    opt = AdamWGS(S.param_groups(params), mode=mode, lambda_o=lo, lambda_s=ls, check=check,
                  fused_compaction=fused)
    assert opt.state.record is not None and opt.state.record.shape[1] == 128
    mbuf, mrec = _canary_rows(n, 128)
    mrec[:, :120].zero_()
    opt.state = MomentState.from_record(mrec, opt.state.spec, 0)
    assert opt.state.record.data_ptr() == mrec.data_ptr()
    return cfg, None, opt, grads, (pbuf, gbuf, mbuf)


def _steps(cfg, opt, grads, k=3, radii=False):
    from paper_2601_16736_b200 import synthetic as S
    for s in range(k):
        vis = S.visibility_device(cfg, s, DEV)
        for name, x in S.grads_device(cfg, s, DEV, vis).items():
            grads[name].copy_(x.view(grads[name].shape))
        m = torch.where(vis, 3, 0).to(torch.int32).contiguous() if radii else vis
        opt.step(m, cfg.n_pixels, grads=grads)
    opt.check_errors()


def _verify(n, bufs):
    pbuf, gbuf, mbuf = bufs
    torch.cuda.synchronize()
    _check(pbuf, n, 59, "parameter record")
    _check(gbuf, n, 59, "gradient record")
    _check(mbuf, n, 120, "moment record")
    # and the steps did run on these buffers: clocks (column 118) advanced
    clocks = mbuf[PAD_ROWS:PAD_ROWS + n, 118]
    assert int((clocks > 0).sum()) > 0


@pytest.mark.parametrize("n,p,mode,fused,check,radii", [
    (300_007, 0.3, "adamw-gs", True, "fused", False),        # per-CTA mask slices
    (300_007, 0.3, "sparse-adam", True, "fused", True),      # two-phase (coupled N_v), radii
    (300_007, 0.3, "adamw-gs", False, "fused", False),       # K1 + K2, short list (bias warp)
    (300_007, 0.3, "adamw-const", False, "strict", False),   # strict pre-check + K2
    (5_000_011, 0.3, "adamw-gs", True, "fused", False),      # tiles dealt grid-stride
    (5_000_011, 0.3, "adamw-gs", False, "fused", False),     # K1 + K2, long list
    (20_000_003, 0.02, "adamw-gs", True, "fused", False),    # sparse: bias warp, 3 CTAs/SM
    (20_000_003, 0.3, "adamw-gs", True, "fused", False),     # dynamic tail (from step 2 on)
])
def test_step_paths_write_only_their_rows(n, p, mode, fused, check, radii):
    cfg, _, opt, grads, bufs = _setup(n, p, mode, fused, check)
    _steps(cfg, opt, grads, radii=radii)
    assert (opt._last_ctx[1] is None) == fused
    _verify(n, bufs)


def test_operations_around_the_step_write_only_their_rows():
    from paper_2601_16736_b200.noise import NoiseConfig
    from paper_2601_16736_b200.sampling import AiuConfig, StSSchedule, stream, stss_sample
    n = 300_007
    cfg, _, opt, grads, bufs = _setup(n, 0.3, "adamw-gs", True)
    _steps(cfg, opt, grads)
    picked = stss_sample(StSSchedule(((0, 0.25),), 3), 3, n, stream(0, "stss", 3))
    opt.rsr_apply(picked, 0.2, 0.04)
    opt.reset_rows(np.array([0, 1, n // 2, n - 2, n - 1]))
    vis = torch.from_numpy(np.random.default_rng(4).random(n) < 0.3).to(DEV)
    aiu = AiuConfig(start=0, end=100, prob_schedule=((0, 0.3),), eta_schedule=((0, 0.5),),
                    enabled=True)
    opt.aiu_apply(vis, aiu, np.random.default_rng(7), 5)
    alive = torch.ones(n, dtype=torch.bool, device=DEV)
    opt.noise_perturb(1e-4, NoiseConfig(enabled=True), 11, 5, alive=alive)
    alive_np = np.random.default_rng(5).random(n) > 0.05
    opt.mcmc_relocate(np.random.default_rng(9), alive=alive_np)
    _steps(cfg, opt, grads, k=1)
    _verify(n, bufs)
