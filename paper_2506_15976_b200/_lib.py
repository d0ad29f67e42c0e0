"""ctypes binding of ``liblbscan_b200.so`` (the C ABI in include/lbscan_b200.h).

The product path has no CPU fallback: if the library is missing or fails to
load, every entry point raises.  Tensors cross the ABI as raw device pointers,
element strides and the caller's CUDA stream handle.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ShapeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LBSCAN_B200_LIB", os.path.join(HERE, "liblbscan_b200.so"))

LBS_OK, LBS_ERR_INVALID, LBS_ERR_CUDA, LBS_ERR_UNSUPPORTED = 0, 1, 2, 3
LBS_F32, LBS_BF16, LBS_F16, LBS_F64 = 0, 1, 2, 3

FLAG_REVERSE = 1 << 0
FLAG_SOFTPLUS = 1 << 1
FLAG_LB = 1 << 2
FLAG_LINEAR = 1 << 3
FLAG_ACCUM = 1 << 5
FLAG_NO_TMA = 1 << 6  # testing: cp.async staging instead of TMA (bitwise-equal results)
CONV_SILU = 1 << 4

ABI_VERSION = 2  # include/lbscan_b200.h LBS_ABI_VERSION
I64 = C.c_int64
I64x3 = C.c_int64 * 3
VP = C.c_void_p


class ScanFwdArgs(C.Structure):
    _fields_ = [
        ("batch", I64), ("seqlen", I64), ("dim", I64), ("dstate", I64), ("window", I64),
        ("io_dtype", C.c_int32), ("bc_dtype", C.c_int32), ("flags", C.c_uint32), ("seg_hint", C.c_int32),
        ("u", VP), ("u_stride", I64x3),
        ("delta", VP), ("delta_stride", I64x3),
        ("A", VP),
        ("B", VP), ("B_stride", I64x3),
        ("C", VP), ("C_stride", I64x3),
        ("D", VP), ("delta_bias", VP),
        ("z", VP), ("z_stride", I64x3),
        ("out", VP), ("out_stride", I64x3),
        ("last_state", VP),
        ("checkpoints", VP), ("ckpt_len", I64),
    ]


class ScanBwdArgs(C.Structure):
    _fields_ = [
        ("fwd", ScanFwdArgs),
        ("dout", VP), ("dout_stride", I64x3),
        ("du", VP), ("du_stride", I64x3),
        ("ddelta", VP), ("ddelta_stride", I64x3),
        ("dz", VP), ("dz_stride", I64x3),
        ("dA", VP), ("dD", VP), ("ddelta_bias", VP),
        ("dB", VP), ("dB_stride", I64x3),
        ("dC", VP), ("dC_stride", I64x3),
    ]


class PrediscretizedArgs(C.Structure):
    _fields_ = [
        ("batch", I64), ("seqlen", I64), ("dim", I64), ("dstate", I64), ("window", I64),
        ("flags", C.c_uint32), ("dtype", C.c_int32),
        ("abar", VP), ("bx", VP), ("c", VP), ("dx", VP), ("y", VP), ("h_final", VP),
    ]


class ConvArgs(C.Structure):
    _fields_ = [
        ("batch", I64), ("seqlen", I64), ("dim", I64), ("width", I64),
        ("io_dtype", C.c_int32), ("flags", C.c_uint32),
        ("x", VP), ("x_stride", I64x3),
        ("weight", VP), ("bias", VP),
        ("out", VP), ("out_stride", I64x3),
        ("dout", VP), ("dout_stride", I64x3),
        ("dx", VP), ("dx_stride", I64x3),
        ("dweight", VP), ("dbias", VP),
    ]


class NormArgs(C.Structure):
    _fields_ = [
        ("rows", I64), ("dim", I64), ("io_dtype", C.c_int32), ("eps", C.c_float),
        ("x", VP), ("x_row_stride", I64), ("scale", VP), ("out", VP), ("out_row_stride", I64),
        ("out_dtype", C.c_int32),
    ]


class NormBwdArgs(C.Structure):
    _fields_ = [
        ("rows", I64), ("dim", I64), ("io_dtype", C.c_int32), ("eps", C.c_float),
        ("x", VP), ("x_row_stride", I64), ("scale", VP), ("dout", VP), ("dout_row_stride", I64),
        ("dx", VP), ("dx_row_stride", I64), ("dscale", VP), ("dres", VP), ("dres_row_stride", I64),
    ]


# every symbol include/lbscan_b200.h declares (tests check the export table)
EXPORTS = (
    "lbs_abi_version", "lbs_last_error", "lbs_select_tile_len",
    "lbs_scan_ckpt_len", "lbs_scan_ckpt_bytes",
    "lbs_scan_fwd_workspace_bytes", "lbs_scan_fwd",
    "lbs_scan_bwd_workspace_bytes", "lbs_scan_bwd",
    "lbs_prediscretized_fwd", "lbs_rms_norm_fwd", "lbs_rms_norm_bwd_workspace_bytes", "lbs_rms_norm_bwd",
    "lbs_causal_conv1d_bwd_workspace_bytes", "lbs_causal_conv1d_fwd", "lbs_causal_conv1d_bwd",
)

_lib = None


def lib():
    """Load (once) and return the ctypes library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"lbscan_b200 CUDA library not found at {LIB_PATH}; build it with "
            "`python -m paper_2506_15976_b200.build` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.lbs_abi_version.restype = C.c_int
    L.lbs_last_error.restype = C.c_char_p
    L.lbs_select_tile_len.restype = I64
    L.lbs_select_tile_len.argtypes = [I64]
    L.lbs_scan_ckpt_len.restype = I64
    L.lbs_scan_ckpt_len.argtypes = [I64, I64]
    L.lbs_scan_ckpt_bytes.restype = C.c_size_t
    L.lbs_scan_ckpt_bytes.argtypes = [C.POINTER(ScanFwdArgs)]
    L.lbs_scan_fwd_workspace_bytes.restype = C.c_size_t
    L.lbs_scan_fwd_workspace_bytes.argtypes = [C.POINTER(ScanFwdArgs)]
    L.lbs_scan_fwd.restype = C.c_int
    L.lbs_scan_fwd.argtypes = [C.POINTER(ScanFwdArgs), VP, C.c_size_t, VP]
    L.lbs_scan_bwd_workspace_bytes.restype = C.c_size_t
    L.lbs_scan_bwd_workspace_bytes.argtypes = [C.POINTER(ScanBwdArgs)]
    L.lbs_scan_bwd.restype = C.c_int
    L.lbs_scan_bwd.argtypes = [C.POINTER(ScanBwdArgs), VP, C.c_size_t, VP]
    L.lbs_prediscretized_fwd.restype = C.c_int
    L.lbs_prediscretized_fwd.argtypes = [C.POINTER(PrediscretizedArgs), VP]
    L.lbs_rms_norm_fwd.restype = C.c_int
    L.lbs_rms_norm_fwd.argtypes = [C.POINTER(NormArgs), VP]
    L.lbs_rms_norm_bwd_workspace_bytes.restype = C.c_size_t
    L.lbs_rms_norm_bwd_workspace_bytes.argtypes = [C.POINTER(NormBwdArgs)]
    L.lbs_rms_norm_bwd.restype = C.c_int
    L.lbs_rms_norm_bwd.argtypes = [C.POINTER(NormBwdArgs), VP, C.c_size_t, VP]
    L.lbs_causal_conv1d_fwd.restype = C.c_int
    L.lbs_causal_conv1d_fwd.argtypes = [C.POINTER(ConvArgs), VP]
    L.lbs_causal_conv1d_bwd_workspace_bytes.restype = C.c_size_t
    L.lbs_causal_conv1d_bwd_workspace_bytes.argtypes = [C.POINTER(ConvArgs)]
    L.lbs_causal_conv1d_bwd.restype = C.c_int
    L.lbs_causal_conv1d_bwd.argtypes = [C.POINTER(ConvArgs), VP, C.c_size_t, VP]
    if L.lbs_abi_version() != ABI_VERSION:
        raise RuntimeError("liblbscan_b200.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    """Map a C status to the reference's exceptions (core.py:24-29)."""
    if rc == LBS_OK:
        return
    msg = lib().lbs_last_error().decode(errors="replace")
    if rc == LBS_ERR_INVALID:
        raise ShapeError(f"{what}: {msg}")
    if rc == LBS_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")
