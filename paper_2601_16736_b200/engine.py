"""Device-side step engine: owns the scratch buffers of one row range and
drives the C ABI (include/adamw_gs.h) on the current CUDA stream.

Everything here is plumbing around the four kernel families; no arithmetic
of the optimizer runs in Python or PyTorch.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

ACTIVE_OPACITY_THRESHOLD = 1.0 / 255.0   # primitives.py:33


class ConfigError(ValueError):
    """Invalid optimizer configuration (optimizer.py:58)."""


class GradientError(RuntimeError):
    """A step hit a non-finite gradient (optimizer.py:62-67); ``ids`` lists the rows."""

    def __init__(self, ids):
        self.ids = np.asarray(ids)
        super().__init__(f"non-finite gradient on primitives {self.ids.tolist()[:16]}")


class DomainError(ValueError):
    """tau non-finite or kappa > 80 on a visible row (primitives.py:40-48,78-84)."""

    def __init__(self, msg, ids=()):
        self.ids = np.asarray(ids)
        super().__init__(msg)


def round_pixel_count(n_pixels: int, enabled: bool = True) -> float:
    """N_I' — keep the most significant digit of N_I, divide by ten (optimizer.py:168-178)."""
    if n_pixels <= 0:
        raise ConfigError("pixel count must be positive")
    if not enabled:
        return float(n_pixels)
    p = 10 ** math.floor(math.log10(n_pixels))
    return (n_pixels // p) * p / 10.0


def _sigmoid_f64(t: float) -> float:
    """primitives.py:51-59 on one float64."""
    if t >= 0:
        return 1.0 / (1.0 + math.exp(-t))
    e = math.exp(t)
    return e / (1.0 + e)


def active_logit_threshold() -> float:
    """Largest fp32 tau with float64 sigmoid(tau) <= 1/255.

    ``classify_active`` (primitives.py:228-238) compares the float64 sigmoid
    with 1/255; for fp32 tau this is exactly ``tau > T`` with this T, so the
    kernels count active rows with one fp32 compare.
    """
    t = np.float32(math.log(ACTIVE_OPACITY_THRESHOLD / (1.0 - ACTIVE_OPACITY_THRESHOLD)))
    up, down = np.float32(np.inf), np.float32(-np.inf)
    while _sigmoid_f64(float(t)) > ACTIVE_OPACITY_THRESHOLD:
        t = np.nextafter(t, down)
    while _sigmoid_f64(float(np.nextafter(t, up))) <= ACTIVE_OPACITY_THRESHOLD:
        t = np.nextafter(t, up)
    return float(t)


def bias_lut_exact_len(beta1: float, beta2: float) -> int:
    """Entries t = 0 .. L-1 after which both fp32 factors 1/(1-beta^t) are
    exactly 1.0f (beta^t < 2^-26), so a kernel clamping t to L-1 is exact."""
    b = max(beta1, beta2)
    if b <= 0.0:
        return 2
    return max(2, int(math.ceil(math.log(2.0 ** -26) / math.log(b))) + 2)


def bias_lut(beta1: float, beta2: float, length: int | None = None) -> np.ndarray:
    """fp32 factors 1/(1-beta^t) rounded once from float64, t in [0, length).

    Denominators as in ``_corrected`` (optimizer.py:202-203).  The kernels
    read entry t for a clock t (clamped to the last entry): exact as long as
    the table covers every clock in use or reaches bias_lut_exact_len
    (StepEngine.ensure_lut keeps that true; oracle.step_fp32 computes the
    same float64 formula)."""
    n = bias_lut_exact_len(beta1, beta2) if length is None else max(2, int(length))
    t = np.arange(n, dtype=np.float64)
    with np.errstate(divide="ignore"):
        c1 = 1.0 / (1.0 - np.power(beta1, t))
        c2 = 1.0 / (1.0 - np.power(beta2, t))
    c1[0] = c2[0] = 1.0
    return np.ascontiguousarray(np.stack([c1.astype(np.float32), c2.astype(np.float32)], axis=1))


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _strides(t: torch.Tensor | None):
    return None if t is None else t.stride()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
# NVTX ranges around the kernel launches (K1 compaction, K2 step, K3 state
# scatters, K4 statistics) for nsys / ncu --nvtx, with GS_NVTX=1 (host cost
# ~1 us per range, which small clouds' eager steps feel)
if os.environ.get("GS_NVTX", "0") not in ("", "0"):
    _nvtx_push = torch.cuda.nvtx.range_push
    _nvtx_pop = torch.cuda.nvtx.range_pop
else:
    def _nvtx_push(name):
        pass

    def _nvtx_pop():
        pass


def _stream_handle(device: torch.device) -> int:
    if _raw_stream is not None:  # the current stream's handle without a Stream object
        return _raw_stream(device.index if device.index is not None else
                           torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class GroupBinding:
    """One attribute group as the kernels see it: [rows, width] fp32 views."""

    name: str
    role: int
    lr: float
    param: torch.Tensor
    grad: torch.Tensor | None
    exp_avg: torch.Tensor | None
    exp_avg_sq: torch.Tensor | None
    w: int = 0  # width when neither param nor per-group state is given

    @property
    def width(self) -> int:
        t = self.param if self.param is not None else self.exp_avg
        if t is None:
            return int(self.w)
        return max(1, t.shape[1:].numel()) if t.dim() > 1 else 1


def row_stride(name, t: torch.Tensor, n_rows: int, width: int) -> int:
    """Row stride (elements) of a tensor whose rows are each one dense run of
    ``width`` values: a contiguous tensor (stride == width) or a view of a
    row-interleaved record (stride > width)."""
    if t.dim() == 0 or t.shape[0] != n_rows or t.numel() != n_rows * width:
        raise ConfigError(f"{name} has shape {tuple(t.shape)}, expected {n_rows} rows x {width}")
    expect = 1
    for d in range(t.dim() - 1, 0, -1):
        if t.shape[d] != 1 and t.stride(d) != expect:
            raise ConfigError(f"{name}: the values of one row must be contiguous")
        expect *= t.shape[d]
    # one row: its stride is unconstrained by the shape (keep a record view's)
    rs = t.stride(0) if (n_rows > 1 or t.stride(0) >= width) else width
    if rs < width:
        raise ConfigError(f"{name}: row stride {rs} is below the row width {width}")
    return int(rs)


def _check_tensor(name, t: torch.Tensor, n_rows: int, width: int, device, dtype=torch.float32,
                  strided: bool = False) -> int:
    if t.device != device:
        raise ConfigError(f"{name} is on {t.device}, expected {device}")
    if t.dtype != dtype:
        raise ConfigError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if strided:
        return row_stride(name, t, n_rows, width)
    if not t.is_contiguous():
        raise ConfigError(f"{name} must be contiguous")
    if t.shape[0] != n_rows or t.numel() != n_rows * width:
        raise ConfigError(f"{name} has shape {tuple(t.shape)}, expected {n_rows} rows x {width}")
    return width


class StepEngine:
    """Scratch buffers + C-ABI launches for one optimizer of ``n_rows`` rows."""

    def __init__(self, n_rows: int, device: torch.device, beta1: float, beta2: float):
        if not torch.cuda.is_available():
            raise L.ExtensionMissing("CUDA device required: the step has no CPU fallback")
        self.lib = L.load()
        self.device = torch.device(device)
        self.n_rows = int(n_rows)
        self.beta1, self.beta2 = float(beta1), float(beta2)
        dev = self.device
        with torch.cuda.device(dev):
            n = max(self.n_rows, 1)
            self.idx = torch.empty(n, dtype=torch.int32, device=dev)
            self.count = torch.zeros(1, dtype=torch.int32, device=dev)
            self.compact_ws = torch.zeros(int(self.lib.gs_compact_workspace_bytes(n)),
                                          dtype=torch.uint8, device=dev)
            self.step_ws = torch.zeros(int(self.lib.gs_step_workspace_bytes()), dtype=torch.uint8,
                                       device=dev)
            # the base step workspace + the two-phase fused kernel's counts and id list
            self.rows_ws = torch.zeros(int(self.lib.gs_step_rows_masked_workspace_bytes(n)),
                                       dtype=torch.uint8, device=dev)
            self.stats = torch.zeros(L.GS_STEP_STATS, dtype=torch.float64, device=dev)
            self.abort = torch.zeros(1, dtype=torch.int32, device=dev)
            # the bias LUT grows with the clocks in use (ensure_lut), up to the
            # exact length past which both factors are 1.0f
            self.lut_exact_len = bias_lut_exact_len(self.beta1, self.beta2)
            self.lut = torch.from_numpy(
                bias_lut(self.beta1, self.beta2, min(self.lut_exact_len, 1 << 14))).to(dev)
            self._old_luts = []
            self.stats_ws = torch.zeros(int(self.lib.gs_stats_workspace_bytes(L.GS_MAX_GROUPS)),
                                        dtype=torch.uint8, device=dev)
            self.stats_all_out = torch.zeros(2 + 5 * L.GS_MAX_GROUPS, dtype=torch.float64,
                                             device=dev)
            self._bad_rows = None
            self._rows_tmp = None
            self._sel = None  # secondary compaction buffers (AIU), lazily
        self.active_logit = active_logit_threshold()
        self.launches = 0  # C-ABI kernel launches issued (bench accounting)
        self._group_cache_key = None
        self._group_cache = None
        self._record_ok = None
        self._cfg_key = None
        self._cfg = None
        self._launched = C.c_int32(0)
        self._omb1 = float(np.float32(1.0 - self.beta1))
        self._omb2 = float(np.float32(1.0 - self.beta2))
        self._eps32 = {}

    def ensure_lut(self, t_max: int):
        """Make the bias LUT exact for every clock <= t_max (it doubles, up to
        the exact length).  Earlier tables stay alive: a captured CUDA graph
        keeps reading the table it was captured with, so capture first
        extends the table to its exact length (AdamWGS.capture)."""
        if t_max < self.lut.shape[0] or self.lut.shape[0] >= self.lut_exact_len:
            return
        n = min(self.lut_exact_len, max(2 * self.lut.shape[0], int(t_max) + 1))
        self._old_luts.append(self.lut)
        self.lut = torch.from_numpy(bias_lut(self.beta1, self.beta2, n)).to(self.device)
        self._cfg_key = None  # the cached configuration holds the table pointer

    # ------------------------------------------------------------------ groups
    def group_array(self, groups: list[GroupBinding], need_grad: bool = True):
        # cache key: pointers and row strides (every step rebuilds the
        # bindings; the array is rebuilt only when a tensor moved)
        key = [need_grad]
        for g in groups:
            p, gr = g.param, g.grad
            key += (g.role, g.lr, p.data_ptr() if p is not None else 0,
                    p.stride() if p is not None else None,
                    gr.data_ptr() if gr is not None else 0,
                    gr.stride() if gr is not None else None,
                    gr.is_cuda if gr is not None else None,
                    g.exp_avg.data_ptr() if g.exp_avg is not None else 0,
                    g.exp_avg_sq.data_ptr() if g.exp_avg_sq is not None else 0)
        if key == self._group_cache_key:
            return self._group_cache
        if not 1 <= len(groups) <= L.GS_MAX_GROUPS:
            raise ConfigError(f"between 1 and {L.GS_MAX_GROUPS} attribute groups are supported")
        arr = (L.GsGroup * len(groups))()
        for i, g in enumerate(groups):
            w = g.width
            ps = gs = 0
            if g.param is not None:
                ps = _check_tensor(f"{g.name}.param", g.param, self.n_rows, w, self.device,
                                   strided=True)
            elif need_grad:
                raise ConfigError(f"group {g.name} has no parameter tensor")
            if g.exp_avg is not None:  # per-group state (the row-record layout passes None)
                _check_tensor(f"{g.name}.exp_avg", g.exp_avg, self.n_rows, w, self.device)
                _check_tensor(f"{g.name}.exp_avg_sq", g.exp_avg_sq, self.n_rows, w, self.device)
            grad_ptr = _ptr(g.grad)
            if need_grad:
                if g.grad is None:
                    raise ConfigError(f"group {g.name} has no gradient")
                if g.grad.device.type == "cpu":
                    grad_ptr, gs = self._host_mapped(f"{g.name}.grad", g.grad, w)
                else:
                    gs = _check_tensor(f"{g.name}.grad", g.grad, self.n_rows, w, self.device,
                                       strided=True)
            arr[i] = L.GsGroup(_ptr(g.param), grad_ptr, _ptr(g.exp_avg), _ptr(g.exp_avg_sq),
                               w, g.role, float(np.float32(g.lr)), ps, gs)
        self._group_cache_key, self._group_cache = key, arr
        return arr

    def _host_mapped(self, name: str, t: torch.Tensor, width: int) -> tuple[int, int]:
        """Pinned host gradients are read zero-copy by the step kernel: only
        the visible rows' bytes cross PCIe (``gs_host_device_pointer``)."""
        if not t.is_pinned():
            raise ConfigError(f"{name} is in pageable host memory; pass a CUDA tensor or a "
                              "pinned (page-locked) host tensor")
        rs = _check_tensor(name, t, self.n_rows, width, t.device, strided=True)
        dptr = L.C.c_void_p()
        L.check(self.lib.gs_host_device_pointer(t.data_ptr(), L.C.byref(dptr)),
                "gs_host_device_pointer")
        return int(dptr.value), rs

    # ------------------------------------------------------------- compaction
    def compact(self, vis: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        """K1: visibility mask (bool/uint8) or radii (int32 > 0) -> (idx, count)."""
        if vis.device != self.device:
            raise ConfigError(f"visibility is on {vis.device}, expected {self.device}")
        if vis.dim() != 1 or vis.shape[0] != self.n_rows:
            raise ConfigError(f"visibility must have shape ({self.n_rows},), got {tuple(vis.shape)}")
        if not vis.is_contiguous():
            raise ConfigError("visibility must be contiguous")
        s = _stream_handle(self.device)
        ws, wsb = self.compact_ws.data_ptr(), self.compact_ws.numel()
        if vis.dtype not in (torch.bool, torch.uint8, torch.int32):
            raise ConfigError(f"visibility dtype {vis.dtype} not supported (bool/uint8 mask or "
                              "int32 radii)")
        _nvtx_push("gs.K1.compact")
        if vis.dtype == torch.int32:
            rc = self.lib.gs_compact_i32(vis.data_ptr(), self.n_rows, self.idx.data_ptr(),
                                         self.count.data_ptr(), ws, wsb, s)
        else:
            rc = self.lib.gs_compact_u8(vis.data_ptr(), self.n_rows, self.idx.data_ptr(),
                                        self.count.data_ptr(), ws, wsb, s)
        _nvtx_pop()
        L.check(rc, "gs_compact")
        self.launches += 2 if self.n_rows > 0 else 0  # count + write passes
        return self.idx, self.count

    def count_visible(self, vis: torch.Tensor) -> torch.Tensor:
        """N_v on the device (K1's count pass only; no index list)."""
        if vis.device != self.device or vis.dim() != 1 or vis.shape[0] != self.n_rows or \
                not vis.is_contiguous() or vis.dtype not in (torch.bool, torch.uint8, torch.int32):
            raise ConfigError("visibility must be a contiguous bool/uint8/int32 row vector")
        is_radii = vis.dtype == torch.int32
        _nvtx_push("gs.K1.count")
        rc = self.lib.gs_count_visible(None if is_radii else vis.data_ptr(),
                                       vis.data_ptr() if is_radii else None, self.n_rows,
                                       self.count.data_ptr(), self.compact_ws.data_ptr(),
                                       self.compact_ws.numel(), _stream_handle(self.device))
        _nvtx_pop()
        L.check(rc, "gs_count_visible")
        self.launches += 1 if self.n_rows > 0 else 0
        return self.count

    def compact_select(self, mask: torch.Tensor, alive: torch.Tensor | None = None,
                       invert: bool = False) -> tuple[torch.Tensor, torch.Tensor]:
        """Rows with mask != 0 (or == 0 when ``invert``), alive only; into a
        second index buffer so the step's visible list is not clobbered."""
        if mask.dtype not in (torch.bool, torch.uint8) or mask.numel() != self.n_rows:
            raise ConfigError("selection mask must be a bool/uint8 row mask")
        if alive is not None and (alive.dtype not in (torch.bool, torch.uint8)
                                  or alive.numel() != self.n_rows):
            raise ConfigError("alive must be a bool/uint8 row mask")
        if self._sel is None:
            n = max(self.n_rows, 1)
            self._sel = (torch.empty(n, dtype=torch.int32, device=self.device),
                         torch.zeros(1, dtype=torch.int32, device=self.device),
                         torch.zeros(int(self.lib.gs_compact_workspace_bytes(n)),
                                     dtype=torch.uint8, device=self.device))
        idx, cnt, ws = self._sel
        mask = mask.contiguous()
        alive = alive.contiguous() if alive is not None else None
        rc = self.lib.gs_compact_select_u8(mask.data_ptr(), _ptr(alive), int(bool(invert)),
                                           self.n_rows, idx.data_ptr(), cnt.data_ptr(),
                                           ws.data_ptr(), ws.numel(), _stream_handle(self.device))
        L.check(rc, "gs_compact_select_u8")
        self.launches += 2 if self.n_rows > 0 else 0
        return idx, cnt

    def compact_positions(self, mask: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        """K1 on an arbitrary-length uint8 mask (scratch buffers sized on demand)."""
        n = int(mask.numel())
        buf = getattr(self, "_pos", None)
        if buf is None or buf[0].numel() < n:
            cap = max(n, 1)
            buf = (torch.empty(cap, dtype=torch.int32, device=self.device),
                   torch.zeros(1, dtype=torch.int32, device=self.device),
                   torch.zeros(int(self.lib.gs_compact_workspace_bytes(cap)), dtype=torch.uint8,
                               device=self.device))
            self._pos = buf
        idx, cnt, ws = buf
        rc = self.lib.gs_compact_u8(mask.contiguous().data_ptr(), n, idx.data_ptr(),
                                    cnt.data_ptr(), ws.data_ptr(), ws.numel(),
                                    _stream_handle(self.device))
        L.check(rc, "gs_compact_u8")
        self.launches += 2 if n > 0 else 0
        return idx, cnt

    def aiu(self, groups: list[GroupBinding], record: torch.Tensor, inv_idx: torch.Tensor,
            jlist: torch.Tensor, k_dev: torch.Tensor, max_k: int, eta: float, eps: float):
        """Artificial implicit updates on picked rows (optimizer.py:425-450);
        returns the picked rows (device int32 [max_k])."""
        self._check_record(record, groups)
        arr = (L.GsGroup * len(groups))()
        for i, g in enumerate(groups):
            ps = _check_tensor(f"{g.name}.param", g.param, self.n_rows, g.width, self.device,
                               strided=True)
            # optimizer.py:449: lr * eta (no mu_lr_scale), rounded once
            arr[i] = L.GsGroup(_ptr(g.param), None, None, None, g.width, g.role,
                               float(np.float32(g.lr * eta)), ps, 0)
        picked = torch.empty(max(max_k, 1), dtype=torch.int32, device=self.device)
        rc = self.lib.gs_aiu_apply_rows(arr, len(groups), record.data_ptr(), record.stride(0),
                                        inv_idx.data_ptr(), jlist.data_ptr(), k_dev.data_ptr(),
                                        int(max_k), self.lut.data_ptr(), self.lut.shape[0],
                                        float(np.float32(eps)), picked.data_ptr(),
                                        _stream_handle(self.device))
        L.check(rc, "gs_aiu_apply_rows")
        self.launches += 1 if max_k else 0
        return picked[:max_k]

    def _build_cfg(self, mode, check, eps, lambda_opacity, lambda_scale, clip_opacity,
                   clip_scale, n_pixels_rounded, global_t, n_visible_dev, n_visible_host,
                   densify):
        cfg = L.GsStepCfg()
        cfg.mode = L.MODE_IDS[mode]
        cfg.check = L.CHECK_STRICT if check == "strict" else L.CHECK_FUSED
        cfg.one_minus_beta1 = self._omb1
        cfg.one_minus_beta2 = self._omb2
        e32 = self._eps32.get(eps)
        if e32 is None:
            e32 = self._eps32[eps] = float(np.float32(eps))
        cfg.eps = e32
        cfg.active_logit = self.active_logit
        cfg.lambda_opacity = float(lambda_opacity)
        cfg.lambda_scale = float(lambda_scale)
        cfg.clip_opacity = float(clip_opacity)
        cfg.clip_scale = float(clip_scale)
        cfg.n_pixels_rounded = float(n_pixels_rounded)
        cfg.bias_lut = self.lut.data_ptr()
        cfg.lut_len = self.lut.shape[0]
        cfg.global_t = int(global_t)
        cfg.beta1, cfg.beta2 = self.beta1, self.beta2
        cfg.n_visible_norm = _ptr(n_visible_dev)
        cfg.n_visible_host = float(n_visible_host)
        cfg.abort_flag = self.abort.data_ptr()
        cfg.densify_group = -1
        if densify is not None:
            accum, dcount, dscale, dgroup = densify
            _check_tensor("densify accum", accum, self.n_rows, 1, self.device, torch.float32)
            _check_tensor("densify count", dcount, self.n_rows, 1, self.device, torch.int32)
            cfg.densify_accum = accum.data_ptr()
            cfg.densify_count = dcount.data_ptr()
            cfg.densify_scale = float(np.float32(dscale))
            cfg.densify_group = int(dgroup)
        return cfg

    # ------------------------------------------------------------------ step
    def step(self, groups: list[GroupBinding], mode: str, clock: torch.Tensor, *,
             rows: torch.Tensor | None, count: torch.Tensor | None, eps: float,
             lambda_opacity: float = 0.0, lambda_scale: float = 0.0, clip_opacity: float = 10.0,
             clip_scale: float = 10.0, n_pixels_rounded: float = 0.0, global_t: int = 0,
             n_visible_dev: torch.Tensor | None = None, n_visible_host: float = 0.0,
             check: str = "fused", record: torch.Tensor | None = None,
             densify: tuple | None = None, abort_hook=None,
             densify_rows: tuple | None = None) -> torch.Tensor:
        """K2 (plus the strict pre-check when ``check == "strict"``).

        ``record`` given: row-record state (gs_step_rows), ``clock`` ignored;
        otherwise per-group m / v tensors and the int32 ``clock``.
        ``abort_hook(flag)``: called between the strict pre-check and the
        step with the device abort flag (index-sharded runs all-reduce it so
        every shard aborts together).  ``densify_rows``: (rows, count) of the
        visible rows for the dense mode, whose kernels step every row: the
        densification statistics then observe only those rows
        (gs_densify_rows) instead of being fused into the step.
        """
        if mode not in L.MODE_IDS:
            raise ConfigError(f"unknown mode {mode!r}; expected one of {tuple(L.MODE_IDS)}")
        if record is None:
            _check_tensor("clock", clock, self.n_rows, 1, self.device, torch.int32)
        else:
            self._check_record(record, groups)
        garr = self.group_array(groups)
        s = _stream_handle(self.device)
        fused_densify = None if (densify_rows is not None and mode == "coupled-adam") else densify
        dkey = None if fused_densify is None else (densify[0].data_ptr(), densify[1].data_ptr(),
                                                   float(densify[2]), int(densify[3]))
        ckey = (mode, check, eps, float(lambda_opacity), float(lambda_scale),
                float(clip_opacity), float(clip_scale), float(n_pixels_rounded), int(global_t),
                _ptr(n_visible_dev), float(n_visible_host), dkey)
        if ckey == self._cfg_key:  # same scalars as the last step: reuse the struct
            cfg = self._cfg
        else:
            cfg = self._build_cfg(mode, check, eps, lambda_opacity, lambda_scale, clip_opacity,
                                  clip_scale, n_pixels_rounded, global_t, n_visible_dev,
                                  n_visible_host, fused_densify)
            self._cfg_key, self._cfg = ckey, cfg
        _nvtx_push("gs.K2.step")
        try:
            self._launch_step(groups, garr, cfg, mode, check, clock, rows, count, record,
                              lambda_opacity, lambda_scale, s, abort_hook)
        finally:
            _nvtx_pop()
        if densify_rows is not None and densify is not None and mode == "coupled-adam":
            self._densify_listed(garr, densify, *densify_rows, strict=check == "strict")
        return self.stats

    def _launch_step(self, groups, garr, cfg, mode, check, clock, rows, count, record,
                     lambda_opacity, lambda_scale, s, abort_hook):
        if check == "strict":
            # the penalty's activation domain is checked where the penalty
            # applies: listed rows, or every row for the dense coupled mode
            drows, dcount = (self.all_rows() if mode == "coupled-adam" else (rows, count))
            rc = self.lib.gs_check_grads(garr, len(groups), self.n_rows, _ptr(drows),
                                         _ptr(dcount), float(lambda_opacity),
                                         float(lambda_scale), None, self.abort.data_ptr(), s)
            L.check(rc, "gs_check_grads")
            if abort_hook is not None:
                abort_hook(self.abort)
        if record is None:
            rc = self.lib.gs_step(garr, len(groups), C.byref(cfg), _ptr(rows), _ptr(count),
                                  self.n_rows, clock.data_ptr(), self.stats.data_ptr(),
                                  self.step_ws.data_ptr(), self.step_ws.numel(), s)
            L.check(rc, "gs_step")
        else:
            rc = self.lib.gs_step_rows(garr, len(groups), C.byref(cfg), _ptr(rows), _ptr(count),
                                       self.n_rows, record.data_ptr(), record.stride(0),
                                       self.stats.data_ptr(), self.rows_ws.data_ptr(),
                                       self.rows_ws.numel(), s)
            L.check(rc, "gs_step_rows")
        self.launches += 2 if check == "strict" else 1

    def step_masked(self, groups: list[GroupBinding], mode: str, vis: torch.Tensor, *, eps: float,
                    lambda_opacity: float = 0.0, lambda_scale: float = 0.0,
                    clip_opacity: float = 10.0, clip_scale: float = 10.0,
                    n_pixels_rounded: float = 0.0, record: torch.Tensor,
                    densify: tuple | None = None, low_visibility: bool = False,
                    coherent: bool = False, balance_tail: bool = False,
                    n_visible_dev: torch.Tensor | None = None) -> torch.Tensor | None:
        """Fused K1 + K2 (gs_step_rows_masked): the step of the mask's visible
        rows with the compaction done inside the step kernel.  Returns the
        statistics, or None when the layout does not take this path (the
        caller then compacts and calls :meth:`step`).  The index list
        (``idx`` / ``count``) is not produced."""
        if vis.device != self.device or vis.dim() != 1 or vis.shape[0] != self.n_rows or \
                not vis.is_contiguous() or vis.dtype not in (torch.bool, torch.uint8, torch.int32):
            return None
        self._check_record(record, groups)
        garr = self.group_array(groups)
        ckey = (mode, "fused", eps, float(lambda_opacity), float(lambda_scale),
                float(clip_opacity), float(clip_scale), float(n_pixels_rounded), 0,
                _ptr(n_visible_dev), 0.0,
                None if densify is None else (densify[0].data_ptr(), densify[1].data_ptr(),
                                              float(densify[2]), int(densify[3])))
        if ckey == self._cfg_key:
            cfg = self._cfg
        else:
            cfg = self._build_cfg(mode, "fused", eps, lambda_opacity, lambda_scale, clip_opacity,
                                  clip_scale, n_pixels_rounded, 0, n_visible_dev, 0.0, densify)
            self._cfg_key, self._cfg = ckey, cfg
        launched = self._launched
        is_radii = vis.dtype == torch.int32
        _nvtx_push("gs.K1K2.step_masked")
        rc = self.lib.gs_step_rows_masked(garr, len(groups), C.byref(cfg),
                                          None if is_radii else vis.data_ptr(),
                                          vis.data_ptr() if is_radii else None, self.n_rows,
                                          record.data_ptr(), record.stride(0),
                                          self.stats.data_ptr(), self.rows_ws.data_ptr(),
                                          self.rows_ws.numel(),
                                          (L.GS_MASKED_LOW_VISIBILITY if low_visibility else 0)
                                          | (L.GS_MASKED_COHERENT if coherent else 0)
                                          | (L.GS_MASKED_BALANCE_TAIL if balance_tail else 0),
                                          C.byref(launched), _stream_handle(self.device))
        _nvtx_pop()
        L.check(rc, "gs_step_rows_masked")
        if not launched.value:
            return None
        self.launches += 1
        return self.stats

    def _densify_listed(self, garr, densify, rows, count, strict: bool):
        """DensifyStats.observe (pipeline.py:77-82) on the listed rows only
        (a no-op when the strict pre-check aborted the step)."""
        accum, dcount, dscale, dgroup = densify
        g = garr[dgroup]
        gs = g.grad_stride if g.grad_stride else g.width
        rc = self.lib.gs_densify_rows(g.grad, gs, g.width, rows.data_ptr(), count.data_ptr(),
                                      self.n_rows, accum.data_ptr(), dcount.data_ptr(),
                                      float(np.float32(dscale)),
                                      self.abort.data_ptr() if strict else None,
                                      _stream_handle(self.device))
        L.check(rc, "gs_densify_rows")
        self.launches += 1

    def _check_record(self, record: torch.Tensor, groups):
        key = (record.data_ptr(), record.shape, record.stride(), record.dtype,
               tuple(g.param.shape if g.param is not None else g.w for g in groups))
        if key == self._record_ok:
            return
        p = sum(g.width for g in groups)
        if (record.device != self.device or record.dtype != torch.float32 or record.dim() != 2
                or record.shape[0] != self.n_rows or record.stride(1) != 1
                or record.shape[1] < 2 * (p + 1)):
            raise ConfigError(f"state record must be fp32 [{self.n_rows}, >= {2 * (p + 1)}] "
                              f"with unit column stride, got {tuple(record.shape)}")
        self._record_ok = key

    def relocate(self, groups: list[GroupBinding], record: torch.Tensor, opacity_group: int,
                 dead: torch.Tensor, targets: torch.Tensor, tau_new: torch.Tensor):
        """MCMC relocation row movement (gs_relocate_rows, pipeline.py:221-228)."""
        self._check_record(record, groups)
        arr = (L.GsGroup * len(groups))()
        for i, g in enumerate(groups):
            ps = _check_tensor(f"{g.name}.param", g.param, self.n_rows, g.width, self.device,
                               strided=True)
            arr[i] = L.GsGroup(_ptr(g.param), None, None, None, g.width, g.role, 0.0, ps, 0)
        k = int(dead.numel())
        for name, t, dt in (("dead", dead, torch.int32), ("targets", targets, torch.int32),
                            ("tau_new", tau_new, torch.float32)):
            if t.device != self.device or t.dtype != dt or t.numel() != k or not t.is_contiguous():
                raise ConfigError(f"{name} must be a contiguous {dt} CUDA tensor of {k} entries")
        rc = self.lib.gs_relocate_rows(arr, len(groups), int(opacity_group), dead.data_ptr(),
                                       targets.data_ptr(), tau_new.data_ptr(), k,
                                       record.data_ptr(), record.stride(0),
                                       _stream_handle(self.device))
        L.check(rc, "gs_relocate_rows")
        self.launches += 1 if k else 0

    def all_rows(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Identity index list (dense mode domain checks, error ids)."""
        if getattr(self, "_all_rows", None) is None:
            self._all_rows = torch.arange(self.n_rows, dtype=torch.int32, device=self.device)
            self._all_count = torch.tensor([self.n_rows], dtype=torch.int32, device=self.device)
        return self._all_rows, self._all_count

    # ----------------------------------------------------------- error ids
    def bad_rows(self, groups: list[GroupBinding], rows=None, count=None, lambda_opacity=0.0,
                 lambda_scale=0.0) -> tuple[np.ndarray, np.ndarray]:
        """Row ids with a non-finite gradient (all rows, gradients.py:50-58) and
        visible row ids outside the activation domain (error path only)."""
        garr = self.group_array(groups)
        if self._bad_rows is None:
            self._bad_rows = torch.zeros((self.n_rows + 3) // 4 * 4, dtype=torch.uint8,
                                         device=self.device)
        flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        rc = self.lib.gs_check_grads(garr, len(groups), self.n_rows, _ptr(rows), _ptr(count),
                                     float(lambda_opacity), float(lambda_scale),
                                     self._bad_rows.data_ptr(), flag.data_ptr(),
                                     _stream_handle(self.device))
        L.check(rc, "gs_check_grads")
        bits = self._bad_rows[: self.n_rows].cpu().numpy()
        return np.flatnonzero(bits & 1), np.flatnonzero(bits & 2)

    # --------------------------------------------------------- RSR / reset
    def _rows_device(self, indices) -> tuple[torch.Tensor, int]:
        """Row ids for K3 with NumPy fancy-index semantics: a boolean mask
        selects its true rows, negative ids count from the end, out-of-range
        ids raise IndexError, and a repeated id acts once (``m[idx] *= a``
        assigns each selected row once).  Returns sorted distinct int32 ids
        on the device.  Inside CUDA-graph capture a device tensor cannot be
        inspected: it is taken as given (the kernels skip ids outside the
        rows; the caller owns distinctness)."""
        n = self.n_rows
        if isinstance(indices, torch.Tensor) and indices.device.type == "cuda" \
                and indices.dtype != torch.bool:
            if indices.dtype.is_floating_point or indices.dtype.is_complex:
                raise IndexError("row indices must be integers or a boolean mask")
            t = indices.reshape(-1)
            if torch.cuda.is_current_stream_capturing():
                t = t.to(device=self.device, dtype=torch.int32).contiguous()
                return t, int(t.numel())
            t = t.to(device=self.device, dtype=torch.int64)
            if t.numel():
                t = torch.where(t < 0, t + n, t)
                lo, hi, mono = torch.stack([t.min(), t.max(),
                                            (t[1:] > t[:-1]).all().to(torch.int64)]).tolist()
                if lo < 0 or hi >= n:
                    raise IndexError(f"row index out of range for {n} rows")
                if not mono:
                    t = torch.unique(t, sorted=True)
            t = t.to(torch.int32).contiguous()
            return t, int(t.numel())
        if isinstance(indices, torch.Tensor):
            indices = indices.detach().cpu().numpy()
        arr = np.asarray(indices)
        if arr.dtype == np.bool_:
            if arr.ndim != 1 or arr.size != n:
                raise IndexError(f"boolean index of shape {arr.shape} does not match {n} rows")
            arr = np.flatnonzero(arr)
        elif arr.size and not np.issubdtype(arr.dtype, np.integer):
            raise IndexError("row indices must be integers or a boolean mask")
        arr = arr.astype(np.int64).reshape(-1)
        if arr.size:
            arr = np.where(arr < 0, arr + n, arr)
            if arr.min() < 0 or arr.max() >= n:
                raise IndexError(f"row index out of range for {n} rows")
            if not np.all(arr[1:] > arr[:-1]):
                arr = np.unique(arr)
        t = torch.from_numpy(arr.astype(np.int32)).to(self.device, non_blocking=False)
        return t, int(t.numel())

    def rsr_apply(self, groups: list[GroupBinding], indices, alpha1: float, alpha2: float,
                  record: torch.Tensor | None = None):
        if not (0.0 <= alpha1 < 1.0 and 0.0 <= alpha2 < 1.0):
            raise ConfigError("RSR factors must lie in [0, 1)")
        rows, k = self._rows_device(indices)
        s = _stream_handle(self.device)
        _nvtx_push("gs.K3.rsr")
        if record is not None:
            self._check_record(record, groups)
            rc = self.lib.gs_rsr_apply_rows(record.data_ptr(), record.stride(0),
                                            sum(g.width for g in groups),
                                            rows.data_ptr() if k else None, k, self.n_rows,
                                            float(alpha1), float(alpha2), s)
        else:
            garr = self.group_array(groups, need_grad=False)
            rc = self.lib.gs_rsr_apply(garr, len(groups), rows.data_ptr() if k else None, k,
                                       self.n_rows, float(alpha1), float(alpha2), s)
        _nvtx_pop()
        L.check(rc, "gs_rsr_apply")
        self.launches += 1 if k else 0
        self._rows_tmp = rows  # keep alive until the kernel has consumed it

    def reset_rows(self, groups: list[GroupBinding], clock: torch.Tensor | None, indices,
                   record: torch.Tensor | None = None):
        rows, k = self._rows_device(indices)
        s = _stream_handle(self.device)
        _nvtx_push("gs.K3.reset")
        if record is not None:
            self._check_record(record, groups)
            rc = self.lib.gs_reset_rows_rows(record.data_ptr(), record.stride(0),
                                             sum(g.width for g in groups),
                                             rows.data_ptr() if k else None, k, self.n_rows, s)
        else:
            garr = self.group_array(groups, need_grad=False)
            rc = self.lib.gs_reset_rows(garr, len(groups), clock.data_ptr(),
                                        rows.data_ptr() if k else None, k, self.n_rows, s)
        _nvtx_pop()
        L.check(rc, "gs_reset_rows")
        self.launches += 1 if k else 0
        self._rows_tmp = rows

    # ---------------------------------------------------------- statistics
    def stats_all(self, groups: list[GroupBinding], alive: torch.Tensor | None = None,
                  record: torch.Tensor | None = None):
        garr = self.group_array(groups, need_grad=False)
        if alive is not None:
            if alive.dtype not in (torch.bool, torch.uint8) or alive.numel() != self.n_rows:
                raise ConfigError("alive must be a bool/uint8 mask over the rows")
            alive = alive.contiguous()
        s = _stream_handle(self.device)
        _nvtx_push("gs.K4.stats")
        if record is not None:
            self._check_record(record, groups)
            rc = self.lib.gs_stats_all_rows(garr, len(groups), self.n_rows, record.data_ptr(),
                                            record.stride(0), _ptr(alive),
                                            float(self.active_logit),
                                            self.stats_all_out.data_ptr(),
                                            self.stats_ws.data_ptr(), self.stats_ws.numel(), s)
        else:
            rc = self.lib.gs_stats_all(garr, len(groups), self.n_rows, _ptr(alive),
                                       float(self.active_logit), self.stats_all_out.data_ptr(),
                                       self.stats_ws.data_ptr(), self.stats_ws.numel(), s)
        _nvtx_pop()
        L.check(rc, "gs_stats_all")
        return self.stats_all_out[: 2 + 5 * len(groups)]
