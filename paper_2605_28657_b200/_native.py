"""ctypes binding of the C-ABI in ``include/ringflow_b200.h``.

The library is the product path: there is no fallback.  If the in-tree library is
missing this module tries to build it (nvcc is in the image); if that fails, or the
CUDA device is absent when a compute entry point is used, it raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import build as _build

RF_OK = 0
RF_STATUS_NOISE_SHORT = 0x1
RF_STATUS_NOISE_LONG = 0x2
RF_STATUS_NONFINITE = 0x4

RF_MAX_COND = 4
RF_NUM_CURVES = 7
CURVE_INDEX = {
    "sde_denoise_curve": 0,
    "guidance_curve": 1,
    "velocity_scale": 2,
    "ode_noise_curve": 3,
    "apg_momentum": 4,
    "cfg_rescale_curve": 5,
    "x0_target_strength": 6,
}
RF_SOLVER_SDE, RF_SOLVER_ODE = 0, 1
RF_NEG_NONE, RF_NEG_UNCOND, RF_NEG_RESIDUAL, RF_NEG_PREV = 0, 1, 2, 3
RF_ROWF_MOMENTUM_INIT = 0x1
RF_ROWF_WRITE_RESIDUAL = 0x2
RF_ROWF_WRITE_PREV = 0x4
RF_ROWF_ODE_MORPH = 0x8
RF_ROWF_COND_V = 0x10
RF_ROWF_UNCOND_V = 0x20
RF_ROWF_NO_STEP = 0x40
RF_ROWF_V_F32 = 0x80
RF_ROWF_STYLE_V = 0x100

c_dptr = ctypes.c_void_p


class RfDraw(ctypes.Structure):
    _fields_ = [("k0", ctypes.c_uint64), ("k1", ctypes.c_uint64), ("n", ctypes.c_int64),
                ("out", c_dptr)]


class RfRow(ctypes.Structure):
    _fields_ = [
        ("x", c_dptr),
        ("noise_model", c_dptr),
        ("noise_step", c_dptr),
        ("source", c_dptr),
        ("x0_target", c_dptr),
        ("curves", c_dptr * RF_NUM_CURVES),
        ("cond_x0", c_dptr * RF_MAX_COND),
        ("cond_w", c_dptr * RF_MAX_COND),
        ("uncond_x0", c_dptr),
        ("momentum", c_dptr),
        ("residual", c_dptr),
        ("prev_positive", c_dptr),
        ("v_out", c_dptr),
        ("t_curr", ctypes.c_double),
        ("t_next", ctypes.c_double),
        ("jitter_t", ctypes.c_double),
        ("n_cond", ctypes.c_int32),
        ("solver", ctypes.c_int32),
        ("neg_kind", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class RfAdmit(ctypes.Structure):
    _fields_ = [("x", c_dptr), ("noise", c_dptr), ("source", c_dptr), ("denoise", ctypes.c_double)]


class RfEmit(ctypes.Structure):
    _fields_ = [("latent", c_dptr), ("record", c_dptr)]


# every symbol declared in include/ringflow_b200.h
EXPORTS = (
    "rf_abi_version", "rf_last_error", "rf_device_sm_count",
    "rf_normal_workspace_bytes", "rf_normal_fill", "rf_uniform_fill",
    "rf_tick_solve", "rf_x0_compose", "rf_admit_init", "rf_emit_stats", "rf_reduce_workspace_elems",
    "rf_decode_workspace_bytes", "rf_decode_window", "rf_decode_tc_packed_bytes", "rf_decode_tc_pack",
    "rf_decode_window_tc", "rf_encode_frames", "rf_mse", "rf_gemm_bf16",
    "rf_dit_workspace_bytes", "rf_dit_create", "rf_dit_destroy", "rf_dit_forward",
    "rf_dit_output", "rf_attention_tc_bf16", "rf_attention_tc_bf16_kernel",
)

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    pass


def library_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load (building first if needed) the sm_100a library; raises if unavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if not os.path.exists(path) or (build_if_missing and not _build.up_to_date()):
            if not build_if_missing and not os.path.exists(path):
                raise NativeError(f"CUDA extension missing: {path}")
            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - exercised only without nvcc
                if not os.path.exists(path):
                    raise NativeError(f"CUDA extension missing and build failed: {exc}") from exc
        lib = ctypes.CDLL(path)
        _declare(lib)
        if lib.rf_abi_version() != 1:
            raise NativeError("ringflow_b200 ABI version mismatch")
        _lib = lib
        return lib


def _declare(lib):
    i32, i64, vp, u32p = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
    lib.rf_abi_version.restype = i32
    lib.rf_last_error.restype = ctypes.c_char_p
    lib.rf_device_sm_count.restype = i32
    lib.rf_normal_workspace_bytes.restype = i64
    lib.rf_normal_workspace_bytes.argtypes = [ctypes.POINTER(RfDraw), i32]
    lib.rf_normal_fill.restype = i32
    lib.rf_normal_fill.argtypes = [ctypes.POINTER(RfDraw), i32, vp, i64, u32p, vp]
    lib.rf_uniform_fill.restype = i32
    lib.rf_uniform_fill.argtypes = [ctypes.POINTER(RfDraw), i32, vp]
    lib.rf_tick_solve.restype = i32
    lib.rf_tick_solve.argtypes = [ctypes.POINTER(RfRow), i32, i64, i64, vp, vp]
    lib.rf_x0_compose.restype = i32
    lib.rf_x0_compose.argtypes = [vp, vp, vp, ctypes.c_double, vp, ctypes.c_double, vp, i64, vp]
    lib.rf_admit_init.restype = i32
    lib.rf_admit_init.argtypes = [ctypes.POINTER(RfAdmit), i32, i64, vp]
    lib.rf_emit_stats.restype = i32
    lib.rf_emit_stats.argtypes = [ctypes.POINTER(RfEmit), i32, i64, vp, vp, vp, vp, u32p, vp, i64, vp]
    lib.rf_reduce_workspace_elems.restype = i64
    lib.rf_reduce_workspace_elems.argtypes = [i64]
    lib.rf_decode_workspace_bytes.restype = i64
    lib.rf_decode_workspace_bytes.argtypes = [i64, i64]
    lib.rf_decode_window.restype = i32
    lib.rf_decode_window.argtypes = [vp, i64, i64, vp, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                     vp, i64, i64, i64, i64, ctypes.c_int32, vp, vp, i64, vp]
    lib.rf_decode_tc_packed_bytes.restype = i64
    lib.rf_decode_tc_packed_bytes.argtypes = [i64, i64, i32]
    lib.rf_decode_tc_pack.restype = i32
    lib.rf_decode_tc_pack.argtypes = [vp, i32, i64, vp, i64, vp, i64, vp]
    lib.rf_decode_window_tc.restype = i32
    lib.rf_decode_window_tc.argtypes = [vp, i64, i64, vp, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                        i64, i64, i64, i64, ctypes.c_int32, vp, vp]
    lib.rf_encode_frames.restype = i32
    lib.rf_encode_frames.argtypes = [vp, i64, i64, vp, i64, vp, vp]
    lib.rf_gemm_bf16.restype = i32
    lib.rf_gemm_bf16.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, ctypes.c_int32, vp, i64,
                                 ctypes.c_int32, ctypes.c_float, ctypes.c_int32, vp]
    lib.rf_mse.restype = i32
    lib.rf_mse.argtypes = [vp, vp, i64, vp, vp, i64, vp]


def check(rc: int, what: str = "") -> None:
    if rc != RF_OK:
        msg = _lib.rf_last_error().decode() if _lib is not None else "?"
        raise NativeError(f"{what or 'ringflow_b200'} failed (rc={rc}): {msg}")
