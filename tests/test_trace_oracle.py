"""The oracle against the reference's own training loop (CPU).

Every optimizer call that the unmodified reference run_training makes on the
TINY configuration (tests/golden/trace_tiny.npz: real renderer gradients,
visibility masks, densification / relocation boundaries, RSR, AIU) is
replayed through the oracle's float64 restatement on the recorded inputs:
the outputs must equal the reference's bit for bit."""

import numpy as np
import pytest

from _trace import LAYOUT, Trace
from oracle import adamw_gs_oracle as O

TR = Trace()


@pytest.mark.parametrize("i", range(len(TR.calls)))
def test_oracle_replays_reference_call(i):
    c = TR.calls[i]
    fn, run = c["fn"], c["run"]
    hp = TR.hyper(run)
    m, v, t = TR.state(i)
    if fn in ("rsr_apply", "reset_rows"):
        idx = TR.arr(i, "idx")
        if fn == "rsr_apply":
            O.rsr_apply_f64(LAYOUT, m, v, idx, c["alpha1"], c["alpha2"])
        else:
            O.reset_rows_f64(LAYOUT, m, v, t, idx)
        p = None
    elif fn == "aiu_apply":
        p = TR.params(i)
        rng = np.random.Generator(np.random.Philox())
        rng.bit_generator.state = {**c["rng_state"], "state": {
            "counter": np.array(c["rng_state"]["state"]["counter"], np.uint64),
            "key": np.array(c["rng_state"]["state"]["key"], np.uint64)},
            "buffer": np.array(c["rng_state"]["buffer"], np.uint64)}
        from paper_2601_16736_b200.sampling import AiuConfig
        aiu = AiuConfig(start=c["aiu"]["start"], end=c["aiu"]["end"],
                        prob_schedule=tuple(map(tuple, c["aiu"]["prob"])),
                        eta_schedule=tuple(map(tuple, c["aiu"]["eta"])), enabled=True)
        it = c["iteration"]
        picked = O.aiu_apply_f64(LAYOUT, p, m, v, t, TR.arr(i, "vis"), TR.arr(i, "in_alive"),
                                 hp.lr, hp.beta1, hp.beta2, hp.eps, aiu.prob_at(it),
                                 aiu.eta_at(it), rng)
        assert np.array_equal(picked, TR.arr(i, "picked"))
    else:
        p, g = TR.params(i), TR.grads(i)
        vis = TR.arr(i, "vis") if TR.has(i, "vis") else None
        mls = c["mu_lr_scale"]
        if fn == "dar_step":
            O.dar_step_f64(LAYOUT, p, g, m, v, t, vis, hp, c["n_pixels"], mls,
                           lambda_o=c.get("lambda_o"), lambda_s=c.get("lambda_s"))
        elif fn == "sparse_adam_step":
            O.sparse_adam_step_f64(LAYOUT, p, g, m, v, t, vis, hp, mls)
        elif fn == "adamw_const_step":
            O.adamw_const_step_f64(LAYOUT, p, g, m, v, t, vis, hp, clip=c["clip"], mu_lr_scale=mls)
        else:
            gt = O.adam_step_sync_f64(LAYOUT, p, g, m, v, t, c["global_t"], hp, mls)
            if gt is not None:
                assert gt == c["global_t_out"]
    mo, vo, to = TR.state(i, "out")
    assert np.array_equal(t, to)
    for k in m:
        assert np.array_equal(m[k], mo[k]), (fn, k)
        assert np.array_equal(v[k], vo[k]), (fn, k)
    if p is not None:
        po = TR.params(i, "out")
        for k in p:
            assert np.array_equal(p[k], po[k]), (fn, k)
