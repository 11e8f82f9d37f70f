"""ctypes binding of the C ABI in include/adamw_gs.h.

The shared library is built in-tree (``_build.py``) and loaded from
``paper_2601_16736_b200/libadamw_gs_b200.so``.  There is no fallback: a
missing or stale library raises ``ExtensionMissing``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libadamw_gs_b200.so"

GS_ABI_VERSION = 4
GS_MAX_GROUPS = 8
GS_MASKED_LOW_VISIBILITY = 1
GS_MASKED_COHERENT = 2
GS_MASKED_BALANCE_TAIL = 4

GS_OK = 0

ROLE_PLAIN, ROLE_POSITION, ROLE_OPACITY, ROLE_SCALE = 0, 1, 2, 3

MODE_IDS = {"coupled-adam": 0, "sparse-adam": 1, "adamw-const": 2, "adamw-const-clip": 3,
            "adamw-gs": 4}
CHECK_FUSED, CHECK_STRICT = 0, 1

STAT_FIELDS = ("n_visible", "n_stepped", "n_bad_grad", "n_bad_domain", "n_active_pre",
               "n_active_post", "n_clip_opacity", "n_clip_scale", "sum_extra_opacity",
               "sum_extra_scale", "n_runs")
GS_STEP_STATS = len(STAT_FIELDS)
# n_runs is a layout hint (how index-coherent the visible rows were), not a
# reference statistic: it depends on the kernel's chunking
HINT_FIELDS = ("n_runs",)


class ExtensionMissing(RuntimeError):
    """The CUDA extension is not built / not loadable: no CPU fallback exists."""


class GsGroup(C.Structure):
    _fields_ = [("param", C.c_void_p), ("grad", C.c_void_p), ("exp_avg", C.c_void_p),
                ("exp_avg_sq", C.c_void_p), ("width", C.c_int64), ("role", C.c_int32),
                ("lr", C.c_float), ("param_stride", C.c_int64), ("grad_stride", C.c_int64)]


class GsStepCfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("check", C.c_int32), ("one_minus_beta1", C.c_float),
                ("one_minus_beta2", C.c_float), ("eps", C.c_float), ("active_logit", C.c_float),
                ("lambda_opacity", C.c_double), ("lambda_scale", C.c_double),
                ("clip_opacity", C.c_double), ("clip_scale", C.c_double),
                ("n_pixels_rounded", C.c_double), ("bias_lut", C.c_void_p),
                ("lut_len", C.c_int32), ("global_t", C.c_int32), ("beta1", C.c_double),
                ("beta2", C.c_double), ("n_visible_norm", C.c_void_p),
                ("n_visible_host", C.c_double), ("abort_flag", C.c_void_p),
                ("densify_accum", C.c_void_p), ("densify_count", C.c_void_p),
                ("densify_scale", C.c_float), ("densify_group", C.c_int32)]


# name -> (restype, argtypes); exactly the symbols declared in include/adamw_gs.h
SIGNATURES = {
    "gs_abi_version": (C.c_int32, []),
    "gs_last_error": (C.c_char_p, []),
    "gs_device_sm_count": (C.c_int32, []),
    "gs_host_device_pointer": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "gs_compact_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "gs_compact_u8": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_size_t, C.c_void_p]),
    "gs_compact_i32": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_size_t, C.c_void_p]),
    "gs_step_workspace_bytes": (C.c_size_t, []),
    "gs_step": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.POINTER(GsStepCfg), C.c_void_p,
                          C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                          C.c_void_p]),
    "gs_check_grads": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.c_int64, C.c_void_p,
                                 C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    "gs_rsr_apply": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.c_void_p, C.c_int64, C.c_int64,
                               C.c_double, C.c_double, C.c_void_p]),
    "gs_reset_rows": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_int64, C.c_int64, C.c_void_p]),
    "gs_stats_workspace_bytes": (C.c_size_t, [C.c_int32]),
    "gs_compact_select_u8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "gs_aiu_apply_rows": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.c_void_p, C.c_int64,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                    C.c_int32, C.c_float, C.c_void_p, C.c_void_p]),
    "gs_relocate_rows": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                   C.c_void_p]),
    "gs_noise_perturb": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int64, C.c_int32, C.c_float, C.c_float, C.c_float,
                                   C.c_float, C.c_uint64, C.c_uint32, C.c_void_p, C.c_int32,
                                   C.c_void_p, C.c_void_p]),
    "gs_step_rows_workspace_bytes": (C.c_size_t, []),
    "gs_step_rows_masked_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "gs_mirror_to_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                    C.c_size_t, C.c_void_p]),
    "gs_set_rows_variant": (C.c_int32, [C.c_int32]),
    "gs_set_fixed_variant": (C.c_int32, [C.c_int32]),
    "gs_step_rows": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.POINTER(GsStepCfg), C.c_void_p,
                               C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                               C.c_void_p, C.c_size_t, C.c_void_p]),
    "gs_rsr_apply_rows": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                    C.c_int64, C.c_double, C.c_double, C.c_void_p]),
    "gs_reset_rows_rows": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                     C.c_int64, C.c_void_p]),
    "gs_densify_rows": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_int64, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p,
                                  C.c_void_p]),
    "gs_build_flags": (C.c_int32, []),
    "gs_count_visible": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                   C.c_size_t, C.c_void_p]),
    "gs_philox_bernoulli": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int64,
                                      C.c_int64, C.c_double, C.c_void_p, C.c_void_p]),
    "gs_step_rows_masked": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.POINTER(GsStepCfg),
                                      C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32,
                                      C.c_void_p, C.c_void_p]),
    "gs_stats_all_rows": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.c_int64, C.c_void_p,
                                    C.c_int64, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p,
                                    C.c_size_t, C.c_void_p]),
    "gs_stats_all": (C.c_int, [C.POINTER(GsGroup), C.c_int32, C.c_int64, C.c_void_p, C.c_float,
                               C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
}

_lib = None


def load(path: os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raise if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ExtensionMissing(
            f"{p} not found: build it with `python -m paper_2601_16736_b200._build` "
            "(there is no CPU fallback)")
    try:
        lib = C.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise ExtensionMissing(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.gs_abi_version() != GS_ABI_VERSION:
        raise ExtensionMissing(f"ABI mismatch: library {lib.gs_abi_version()} != {GS_ABI_VERSION}")
    if path is None:
        _lib = lib
    return lib


class GsError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


def check(rc: int, what: str) -> None:
    if rc != GS_OK:
        msg = load().gs_last_error().decode(errors="replace")
        raise GsError(f"{what} failed (status {rc}): {msg}")
