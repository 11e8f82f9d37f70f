"""CPU tests of the row-interleaved record helpers (records.py) and the row
stride rule the engine applies to parameter / gradient tensors."""

import pytest
import torch

from paper_2601_16736_b200 import records as R
from paper_2601_16736_b200.engine import ConfigError, row_stride


def _attrs(n=7):
    g = torch.Generator().manual_seed(0)
    return {"xyz": torch.randn(n, 3, generator=g), "f_dc": torch.randn(n, 3, generator=g),
            "f_rest": torch.randn(n, 15, 3, generator=g), "opacity": torch.randn(n, 1, generator=g),
            "scaling": torch.randn(n, 3, generator=g), "rotation": torch.randn(n, 4, generator=g)}


def test_pack_layout_and_views():
    a = _attrs()
    rec, v = R.pack(a)
    assert rec.shape == (7, 64) and rec.is_contiguous()   # 64-byte-granule rows
    assert R.pack(a, align=4)[0].shape == (7, 60)          # compact rows
    off = 0
    for k, t in a.items():
        w = t[0].numel()
        assert torch.equal(v[k], t) and v[k].shape == t.shape
        assert torch.equal(rec[:, off:off + w].reshape(t.shape), t)
        assert row_stride(k, v[k], 7, w) == 64
        off += w
    assert torch.all(rec[:, 59:] == 0)  # pad


def test_autograd_fills_record_grad_and_base_grad_view():
    rec, v = R.pack(_attrs(), requires_grad=True)
    loss = (v["xyz"] ** 2).sum() + 3.0 * v["f_rest"].sum()
    loss.backward()
    assert rec.grad.shape == rec.shape
    assert torch.equal(R.base_grad_view(v["xyz"]), 2 * v["xyz"].detach())
    assert torch.equal(R.base_grad_view(v["f_rest"]), torch.full((7, 15, 3), 3.0))
    assert torch.equal(R.base_grad_view(v["opacity"]), torch.zeros(7, 1))
    assert R.base_grad_view(torch.zeros(7, 3)) is None


def test_adopt_rehomes_parameters_and_autograd_fills_the_record():
    a = _attrs()
    params = {k: torch.nn.Parameter(t.clone()) for k, t in a.items()}
    ids = {k: id(p) for k, p in params.items()}
    params["opacity"].grad = torch.full((7, 1), 0.5)   # an existing gradient is kept
    rec, grec = R.adopt(params)
    assert rec.shape == (7, 64) and grec.shape == (7, 64)
    base, gbase = rec.data_ptr(), grec.data_ptr()
    for k, p in params.items():
        assert id(p) == ids[k] and p.is_leaf and p.requires_grad
        assert torch.equal(p.detach(), a[k]) and p.stride(0) == 64
        assert base <= p.data_ptr() < base + rec.numel() * 4
        assert p.grad.stride(0) == 64 and gbase <= p.grad.data_ptr() < gbase + grec.numel() * 4
    assert torch.all(grec[:, 51] == 0.5)
    loss = (params["xyz"] ** 2).sum() + 3.0 * params["f_rest"].sum() + params["opacity"].sum()
    loss.backward()
    g = R.views_like(grec, params)
    assert params["xyz"].grad.data_ptr() == g["xyz"].data_ptr()   # accumulated in place
    assert torch.equal(g["xyz"], 2 * a["xyz"])
    assert torch.equal(g["f_rest"], torch.full((7, 15, 3), 3.0))
    assert torch.equal(g["opacity"], torch.full((7, 1), 1.5))
    assert torch.equal(g["rotation"], torch.zeros(7, 4))
    with torch.no_grad():                                        # in-place updates land in the record
        params["scaling"].add_(1.0)
    assert torch.equal(R.views_like(rec, params)["scaling"], a["scaling"] + 1.0)
    with pytest.raises(ConfigError):
        R.adopt({"x": params["xyz"] * 2})


def test_views_like_matches_offsets():
    a = _attrs()
    _, v = R.pack(a)
    other = torch.arange(7 * 64, dtype=torch.float32).view(7, 64)
    w = R.views_like(other, v)
    assert w["opacity"][2, 0] == other[2, 51]
    assert torch.equal(w["rotation"][1], other[1, 55:59])


def test_row_stride_rules():
    assert row_stride("c", torch.zeros(5, 3), 5, 3) == 3
    assert row_stride("v", torch.zeros(5, 8)[:, 2:5], 5, 3) == 8
    with pytest.raises(ConfigError):
        row_stride("t", torch.zeros(3, 5).t(), 5, 3)           # column-major rows
    with pytest.raises(ConfigError):
        row_stride("s", torch.zeros(5, 6)[:, ::2], 5, 3)       # gaps inside a row
    with pytest.raises(ConfigError):
        row_stride("n", torch.zeros(4, 3), 5, 3)               # wrong row count
    with pytest.raises(ConfigError):
        R.pack({"a": torch.zeros(3, 2), "b": torch.zeros(4, 2)})


def test_record_of_packed_adopted_and_plain():
    a = _attrs()
    rec, v = R.pack(a)
    assert R.record_of(v) is rec
    params = {k: torch.nn.Parameter(t.clone()) for k, t in a.items()}
    arec, _ = R.adopt(params, grads=False)
    got = R.record_of(params)
    assert got is not None and got.shape == arec.shape and got.data_ptr() == arec.data_ptr()
    assert torch.equal(got, arec)
    sel = R.views_like(got.detach().index_select(0, torch.tensor([4, 0])), params)
    assert torch.equal(sel["f_rest"], a["f_rest"][[4, 0]])
    assert R.record_of(a) is None                                  # separate tensors
    assert R.record_of(dict(reversed(list(v.items())))) is None    # offsets out of dict order
    assert R.record_of({"xyz": v["xyz"], "opacity": v["opacity"]}) is None   # a gap
