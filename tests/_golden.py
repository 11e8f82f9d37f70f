"""Loader for the committed golden vectors (tests/golden/*.npz).

The vectors were written by ``tests/golden/make_golden.py`` from the
unmodified reference optimizer; this module only reads them.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from oracle.adamw_gs_oracle import LAYOUT_REF2D, LAYOUT_SH3, Hyper

GOLDEN = Path(__file__).resolve().parent / "golden"

STEP_CASES = ("sh3_dar", "sh3_dar_clip", "sh3_sparse", "sh3_const", "sh3_const_clip",
              "ref2d_sparse_coupled", "ref2d_sync_coupled")


class Case:
    def __init__(self, name: str):
        z = np.load(GOLDEN / f"{name}.npz")
        self.name = name
        self.meta = json.loads(str(z["meta"]))
        self.z = z
        self.layout = LAYOUT_SH3 if self.meta["layout"] == "sh3" else LAYOUT_REF2D
        self.n = int(self.meta["n"])
        self.steps = int(self.meta["steps"])
        self.vis = z["vis"]
        self.mode = self.meta["mode"]

    def hyper(self) -> Hyper:
        m = self.meta
        return Hyper(lr=dict(m["lr"]), beta1=m["beta1"], beta2=m["beta2"], eps=m["eps"],
                     lambda_o=m["lambda_o"], lambda_s=m["lambda_s"],
                     ct_opacity=m.get("ct_opacity", 10.0), ct_scale=m.get("ct_scale", 10.0))

    def init(self, dtype=np.float64):
        return {g.name: self.z[f"init_{g.name}"].astype(dtype).copy() for g in self.layout}

    def grads(self, s, dtype=np.float64):
        return {g.name: self.z[f"grads_{g.name}"][s].astype(dtype).copy() for g in self.layout}

    def expected(self):
        out = {g.name: self.z[f"out_{g.name}"] for g in self.layout}
        m = {g.name: self.z[f"m_{g.name}"] for g in self.layout}
        v = {g.name: self.z[f"v_{g.name}"] for g in self.layout}
        return out, m, v, self.z["t"]


def normwise(a, ref):
    """max|a - ref| / max|ref| (SURVEY §7.3(1) tier i)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max()
    if den == 0.0:
        return float(np.abs(a).max())
    return float(np.abs(a - ref).max() / den)
