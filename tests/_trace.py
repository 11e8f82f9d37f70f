"""Loader for tests/golden/trace_tiny.npz (written by tests/golden/make_trace.py
from the unmodified reference's run_training): every optimizer call of the
reference loop with its inputs and outputs."""

from __future__ import annotations

import json

import numpy as np

from _golden import GOLDEN
from oracle.adamw_gs_oracle import LAYOUT_REF2D, Hyper

GROUPS = ("mu", "kappa", "rot", "tau", "color")
WIDTH = {"mu": 2, "kappa": 2, "rot": 1, "tau": 1, "color": 3}


class Trace:
    def __init__(self):
        self.z = np.load(GOLDEN / "trace_tiny.npz")
        self.meta = json.loads(str(self.z["meta"]))
        self.calls = self.meta["calls"]

    def hyper(self, run) -> Hyper:
        o = self.meta["runs"][run]["optimizer"]
        return Hyper(lr={"mu": o["lr_mu"], "kappa": o["lr_kappa"], "rot": o["lr_rot"],
                         "tau": o["lr_tau"], "color": o["lr_color"]},
                     beta1=o["beta1"], beta2=o["beta2"], eps=o["eps"], lambda_o=o["lambda_o"],
                     lambda_s=o["lambda_s"], ct_opacity=o["ct_opacity"], ct_scale=o["ct_scale"],
                     round_n_pixels=o["round_n_pixels"])

    def arr(self, i, key):
        return self.z[f"c{i}_{key}"]

    def has(self, i, key):
        return f"c{i}_{key}" in self.z

    def params(self, i, side="in"):
        return {g: self.arr(i, f"{side}_p_{g}").astype(np.float64).reshape(-1, WIDTH[g])
                for g in GROUPS}

    def state(self, i, side="in"):
        m = {g: self.arr(i, f"{side}_m_{g}").astype(np.float64).reshape(-1, WIDTH[g])
             for g in GROUPS}
        v = {g: self.arr(i, f"{side}_v_{g}").astype(np.float64).reshape(-1, WIDTH[g])
             for g in GROUPS}
        return m, v, self.arr(i, f"{side}_t").astype(np.int64).copy()

    def grads(self, i):
        return {g: self.arr(i, f"in_g_{g}").astype(np.float64).reshape(-1, WIDTH[g])
                for g in GROUPS}


LAYOUT = LAYOUT_REF2D
