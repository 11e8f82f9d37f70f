"""The reference's own training loop drives the B200 step (marked gpu).

tests/golden/trace_tiny.npz holds every optimizer call the unmodified
reference run_training makes on the TINY configuration of
R/pkg/tests/test_pipeline.py (real renderer gradients and visibility,
densification and relocation boundaries, RSR, AIU, noise) in four modes.
Each call is replayed through paper_2601_16736_b200.reference_api on CUDA
tensors.  Where the loop changed nothing between two calls, the GPU state
is carried over (a chained run) instead of reloading the recorded input, so
errors accumulate as in a real run.  Clocks and AIU picks are exact;
parameters and moments within 1e-6 normwise of the float64 reference (the
north star's fp32 contract, tests/_golden.py:normwise)."""

import numpy as np
import pytest
import torch

from _golden import normwise
from _trace import GROUPS, WIDTH, Trace

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TOL = 1e-6
TR = Trace()


def _cfg(run):
    from paper_2601_16736_b200.reference_api import OptimizerConfig
    o = TR.meta["runs"][run]["optimizer"]
    return OptimizerConfig(**o)


def _load_p(i):
    return {g: torch.tensor(TR.arr(i, f"in_p_{g}").reshape(-1, WIDTH[g]), dtype=torch.float32,
                            device=DEV) for g in GROUPS}


def _load_st(i, like):
    from paper_2601_16736_b200.optimizer import MomentState
    n = TR.arr(i, "in_t").shape[0]
    st = MomentState.zeros_like({g: torch.zeros((n, WIDTH[g]), device=DEV) for g in GROUPS},
                                "rows")
    for g in GROUPS:
        st.m[g].copy_(torch.from_numpy(TR.arr(i, f"in_m_{g}").reshape(-1, WIDTH[g])))
        st.v[g].copy_(torch.from_numpy(TR.arr(i, f"in_v_{g}").reshape(-1, WIDTH[g])))
    st.clock.copy_(torch.from_numpy(TR.arr(i, "in_t").astype(np.int32)))
    return st


def _eq(i, a, j, b):
    if not (TR.has(i, a) and TR.has(j, b)):
        return False
    x, y = TR.arr(i, a), TR.arr(j, b)
    return x.shape == y.shape and np.array_equal(x, y)


def _p_carried(i, j):
    """Call j's parameters are exactly what call i left (nothing in between)."""
    return all(_eq(i, f"out_p_{g}", j, f"in_p_{g}") for g in GROUPS)


def _st_carried(i, j):
    return all(_eq(i, f"out_{x}_{g}", j, f"in_{x}_{g}") for g in GROUPS for x in ("m", "v")) \
        and _eq(i, "out_t", j, "in_t")


@pytest.mark.parametrize("run", ["gs", "sparse", "coupled", "mcmc"])
def test_reference_loop_replayed_on_gpu(run):
    from paper_2601_16736_b200 import reference_api as RA
    from paper_2601_16736_b200.sampling import AiuConfig
    a, b = TR.meta["runs"][run]["calls"]
    cfg = _cfg(run)
    p = st = None
    chained = longest = 0
    prev = last_p = None
    worst = 0.0
    for i in range(a, b):
        c = TR.calls[i]
        fn = c["fn"]
        has_p = TR.has(i, "in_p_mu")
        keep_s = st is not None and prev is not None and _st_carried(prev, i)
        keep_p = (not has_p) or (p is not None and last_p is not None and _p_carried(last_p, i))
        if keep_s and keep_p:
            chained += 1
        else:
            chained = 0
            if not keep_s:
                st = _load_st(i, p)
            if has_p and not keep_p:
                p = _load_p(i)
        st.global_t = c.get("global_t", st.global_t)
        if fn in ("rsr_apply", "reset_rows"):
            idx = TR.arr(i, "idx")
            if fn == "rsr_apply":
                RA.rsr_apply(st, idx, c["alpha1"], c["alpha2"])
            else:
                RA.reset_rows(st, idx)
        elif fn == "aiu_apply":
            pd = dict(p, alive=torch.from_numpy(TR.arr(i, "in_alive")).to(DEV))
            rng = np.random.Generator(np.random.Philox())
            rs = c["rng_state"]
            rng.bit_generator.state = {**rs, "state": {
                "counter": np.array(rs["state"]["counter"], np.uint64),
                "key": np.array(rs["state"]["key"], np.uint64)},
                "buffer": np.array(rs["buffer"], np.uint64)}
            aiu = AiuConfig(start=c["aiu"]["start"], end=c["aiu"]["end"],
                            prob_schedule=tuple(map(tuple, c["aiu"]["prob"])),
                            eta_schedule=tuple(map(tuple, c["aiu"]["eta"])), enabled=True)
            picked = RA.aiu_apply(st, pd, torch.from_numpy(TR.arr(i, "vis")).to(DEV), cfg, aiu,
                                  rng, c["iteration"])
            assert np.array_equal(picked, TR.arr(i, "picked")), i
        else:
            g = {k: torch.tensor(TR.arr(i, f"in_g_{k}").reshape(-1, WIDTH[k]),
                                 dtype=torch.float32, device=DEV) for k in GROUPS}
            vis = torch.from_numpy(TR.arr(i, "vis")).to(DEV) if TR.has(i, "vis") else None
            mls = c["mu_lr_scale"]
            if fn == "dar_step":
                RA.dar_step(st, p, g, vis, cfg, c["n_pixels"], mls, lambda_o=c.get("lambda_o"),
                            lambda_s=c.get("lambda_s"))
            elif fn == "sparse_adam_step":
                RA.sparse_adam_step(st, p, g, vis, cfg, mls)
            elif fn == "adamw_const_step":
                RA.adamw_const_step(st, p, g, vis, cfg, clip=c["clip"], mu_lr_scale=mls)
            else:
                RA.adam_step_sync(st, p, g, cfg, mls)
                assert st.global_t == c["global_t_out"]
        # compare with the reference's outputs of this call
        assert np.array_equal(st.clock.cpu().numpy(), TR.arr(i, "out_t").astype(np.int32)), i
        for k in GROUPS:
            for name, got in (("m", st.m[k]), ("v", st.v[k])):
                want = TR.arr(i, f"out_{name}_{k}").reshape(-1, WIDTH[k])
                e = normwise(got.cpu().numpy(), want)
                worst = max(worst, e)
                assert e <= TOL, (i, fn, name, k, e, chained)
            if TR.has(i, f"out_p_{k}"):
                want = TR.arr(i, f"out_p_{k}").reshape(-1, WIDTH[k])
                e = normwise(p[k].cpu().numpy(), want)
                worst = max(worst, e)
                assert e <= TOL, (i, fn, "param", k, e, chained)
        longest = max(longest, chained)
        prev = i
        if TR.has(i, "out_p_mu"):
            last_p = i
    print(f"{run}: {b - a} calls, longest chained run {longest + 1}, worst normwise {worst:.2e}")


