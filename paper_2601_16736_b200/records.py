"""Row-interleaved parameter and gradient records.

The reference keeps one array per attribute (``GaussianParams``,
``src/primitives.py:95-112``; ``ParamGrads``, ``src/gradients.py:18-47``).
With ~30% of rows visible per step, the step's gathers then touch each
attribute's HBM separately. A 12-byte xyz row or a 4-byte opacity costs a
whole 32/64-byte DRAM granule, shared with invisible neighbours. The partial
writes are read-modify-written.

A record stores the attributes of one row contiguously: SH-3 is 59 floats,
padded to 64 (256 B, whole 64-byte DRAM granules). The attributes stay ordinary
tensors, as views of the record with the same shapes, so the renderer, the
optimizer API and the checkpoint code see per-attribute tensors. The step
kernel reads a visible row with one run of 16-byte copies.

Gradients follow naturally from autograd. Make the record the leaf
parameter and take the attribute views from it; backward then fills
``record.grad`` with the same interleaving. :meth:`AdamWGS.step` picks up
``view._base.grad`` by itself, or the caller passes :func:`views_like` of a
gradient record, e.g. a pinned host buffer that the step kernel reads
zero-copy.
"""

from __future__ import annotations

import torch

from .engine import ConfigError


def record_width(widths, align: int = 16) -> int:
    """Floats per record row: the attribute widths summed, rounded up to
    ``align``.  16 (default) pads rows to whole 64-byte DRAM granules (SH-3:
    59 -> 64 floats, 256 B), so a row never straddles an extra granule: the
    step kernel is 5% faster on random visibility, 5% slower on index-coherent
    visibility (profiles/r01/record_alignment_probe.txt).  4 is the compact
    minimum (16-byte rows for the kernels' 16-byte copies)."""
    p = int(sum(widths))
    return (p + align - 1) // align * align


def _width(t: torch.Tensor) -> int:
    w = 1
    for d in t.shape[1:]:
        w *= int(d)
    return w


def _tail_strides(tail: tuple) -> tuple:
    out, acc = [], 1
    for d in reversed(tail):
        out.append(acc)
        acc *= int(d)
    return tuple(reversed(out))


def views(record: torch.Tensor, shapes: dict[str, tuple]) -> dict[str, torch.Tensor]:
    """Per-attribute views of a ``(n, PL)`` record. ``shapes`` gives each
    attribute's per-row shape; attributes are packed in dict order."""
    if record.dim() != 2 or not record.is_contiguous():
        raise ConfigError("a record must be a contiguous (n, row_width) tensor")
    n, pl = record.shape
    out, off = {}, 0
    for name, rs in shapes.items():
        rs = tuple(int(d) for d in rs)
        w = 1
        for d in rs:
            w *= d
        if off + w > pl:
            raise ConfigError(f"record row of {pl} floats is too narrow for {name}")
        v = record[:, off:off + w]
        out[name] = v.view(n, *rs) if rs else v.view(n)
        off += w
    return out


def pack(tensors: dict[str, torch.Tensor], align: int = 16, pin_memory: bool = False,
         requires_grad: bool = False) -> tuple[torch.Tensor, dict[str, torch.Tensor]]:
    """Copy per-attribute tensors (same row count, dict order = record order)
    into one new record; return ``(record, views)``. The views keep the
    input shapes; with ``requires_grad`` the record is a leaf whose ``.grad``
    has the same layout."""
    if not tensors:
        raise ConfigError("nothing to pack")
    first = next(iter(tensors.values()))
    n = int(first.shape[0])
    shapes = {}
    for name, t in tensors.items():
        if t.dim() == 0 or int(t.shape[0]) != n:
            raise ConfigError(f"{name}: every attribute needs the same row count {n}")
        if t.dtype != torch.float32:
            raise ConfigError(f"{name}: records hold fp32 attributes")
        shapes[name] = tuple(t.shape[1:])
    pl = record_width([_width(t) for t in tensors.values()], align)
    record = torch.zeros((n, pl), dtype=torch.float32, device=first.device,
                         pin_memory=pin_memory and first.device.type == "cpu")
    vs = views(record, shapes)
    with torch.no_grad():
        for name, t in tensors.items():
            vs[name].copy_(t)
    if requires_grad:
        record.requires_grad_(True)
        vs = views(record, shapes)
    return record, vs


def adopt(params: dict[str, torch.Tensor], align: int = 16,
          grads: bool = True) -> tuple[torch.Tensor, torch.Tensor | None]:
    """Re-home existing per-attribute leaf parameters into one record, in
    place: each ``Parameter`` keeps its identity (model code, param groups,
    hooks and checkpoints still hold the same objects) but its ``.data``
    becomes the attribute view of a new record. With ``grads`` each ``.grad``
    becomes the same view of a zeroed gradient record (an existing gradient
    is copied in); autograd accumulates into a defined ``.grad`` in place, so
    backward keeps filling the record (PyTorch warns once that such a strided
    ``.grad`` breaks its layout contract; the layout is intended). Clear it
    with ``AdamWGS.zero_grad()``, which zeroes record views in place, or
    ``grad_record.zero_()``: setting gradients to None detaches them from the
    record, and the step then falls back to per-attribute gathers. Returns
    ``(record, grad_record)``.

    This is the one-line switch from the reference's per-attribute arrays
    (``src/primitives.py:95-112``, ``src/gradients.py:18-47``) to the record
    layout the step kernel reads fastest (c3: 0.58 -> 0.78 of copy peak,
    profiles/r01/bench_c3_attr.json vs bench_c3.json)."""
    if not params:
        raise ConfigError("nothing to adopt")
    for name, p in params.items():
        if not p.is_leaf:
            raise ConfigError(f"{name}: only leaf tensors can be adopted into a record")
    record, vs = pack({k: p.detach() for k, p in params.items()}, align)
    grad_record = None
    if grads:
        grad_record = torch.zeros_like(record)
        gvs = views_like(grad_record, vs)
    with torch.no_grad():
        for name, p in params.items():
            old = p.grad
            p.data = vs[name]
            if grads:
                if old is not None:
                    gvs[name].copy_(old)
                p.grad = gvs[name]
    return record, grad_record


def views_like(record: torch.Tensor, like: dict[str, torch.Tensor]) -> dict[str, torch.Tensor]:
    """Views of another record (a gradient record, a host staging buffer)
    with the attribute shapes of ``like`` (e.g. the views :func:`pack`
    returned)."""
    return views(record, {k: tuple(v.shape[1:]) for k, v in like.items()})


def record_of(tensors: dict[str, torch.Tensor]) -> torch.Tensor | None:
    """The ``(n, row_width)`` record the attribute tensors are views of, or
    None: views from :func:`pack` (a common ``_base``) and parameters
    re-homed by :func:`adopt` (one storage, one row stride). The attributes
    must sit at the offsets :func:`views` gives them in dict order, so that
    :func:`views_like` of a gathered record maps back to the same names."""
    ts = list(tensors.values())
    if not ts or any(t.dim() < 1 or t.dtype != torch.float32 for t in ts):
        return None
    first = ts[0]
    n, rs = int(first.shape[0]), first.stride(0)
    base = first._base
    if base is not None and all(t._base is base for t in ts):
        if base.dim() != 2 or not base.is_contiguous() or base.shape[0] != n:
            return None
    else:
        st = first.untyped_storage()
        if any(t.untyped_storage().data_ptr() != st.data_ptr() or t.stride(0) != rs or
               int(t.shape[0]) != n for t in ts):
            return None
        off0 = first.storage_offset()
        if (off0 + n * rs) * first.element_size() > st.nbytes():
            return None
        base = torch.empty(0, dtype=first.dtype, device=first.device).set_(st, off0, (n, rs),
                                                                           (rs, 1))
    off = 0
    for t in ts:
        if t.stride(0) != rs or t.storage_offset() - base.storage_offset() != off or \
                t.stride()[1:] != _tail_strides(tuple(t.shape[1:])):
            return None
        off += _width(t)
    return base if off <= base.shape[1] else None


def base_grad_view(p: torch.Tensor) -> torch.Tensor | None:
    """The gradient of an attribute view ``p`` of a leaf record: the same
    view of ``p._base.grad``. None if ``p`` is not such a view or the record
    has no gradient."""
    base = getattr(p, "_base", None)
    if base is None or base.grad is None:
        return None
    g = base.grad
    if g.shape != base.shape or g.stride() != base.stride() or g.dtype != p.dtype:
        return None
    rel = p.storage_offset() - base.storage_offset()
    return g.as_strided(p.shape, p.stride(), g.storage_offset() + rel)
