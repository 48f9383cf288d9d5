"""ctypes binding of libconvb200.so (include/convb200.h).

Status codes are mapped onto the reference exception types so callers see the same
failures the reference raises (descriptor.py:23-24, algos.py:35-36, harness.py:138-147).
The product path has no CPU fallback: if the library or a GPU is missing, every entry
point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .descriptor import ConvDescriptor, InvalidDescriptorError

# CB_LIB_PATH (diagnostics only): load another build of the library for A/B runs
LIB_PATH = Path(os.environ["CB_LIB_PATH"]) if os.environ.get("CB_LIB_PATH") else \
    Path(__file__).resolve().parent / "libconvb200.so"

CB_OK, CB_ERR_INVALID, CB_ERR_UNSUPPORTED, CB_ERR_WORKSPACE, CB_ERR_MISALIGNED, CB_ERR_CUDA = range(6)

VARIANTS = {"tc3xtf32": 0, "ffma": 1, "tc3xbf16": 2}
TC_VARIANTS = ("tc3xtf32", "tc3xbf16")

# Every symbol include/convb200.h declares (tests check the .so exports all of them).
EXPORTS = (
    "cb_version", "cb_last_error_string", "cb_device_sm_count", "cb_launch_count",
    "cb_event_create", "cb_event_destroy", "cb_event_record", "cb_event_elapsed_ns",
    "cb_output_shape", "cb_env_fingerprint",
    "cb_workspace_bytes", "cb_im2col_f32", "cb_sconv_plan", "cb_sconv_range",
    "cb_sconv_pack_f32", "cb_plan_tiles",
    "cb_split_kdim", "cb_weight_split", "cb_gemm", "cb_conv_gemm_cols", "cb_sconv_gemm",
    "cb_unpack_f32", "cb_fused_layout_query", "cb_fused_reduction_map", "cb_fused_plan_tiles",
    "cb_fused_pack_weights",
    "cb_fused_pack_input", "cb_conv_fused_packed", "cb_conv_fused",
)


class UnsupportedDescriptorError(ValueError):
    """The selected algorithm cannot execute this descriptor (algos.py:35-36)."""


class ConvB200Error(RuntimeError):
    """A CUDA-side failure reported by libconvb200."""


class CbConvDesc(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int32) for name in (
        "batch", "in_channels", "in_h", "in_w", "out_channels", "k_h", "k_w",
        "stride_h", "stride_w", "pad_h", "pad_w", "dil_h", "dil_w", "groups", "has_bias")]


class CbSlicePlan(ctypes.Structure):
    _fields_ = [("band_rows", ctypes.c_int32), ("num_slices", ctypes.c_int32)]


class CbTilePlan(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("variant", "block_m", "block_n", "block_k", "stages", "splits")] + \
               [(n, ctypes.c_int64) for n in ("m_tiles", "n_tiles", "k_blocks", "ctas")]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class CbFusedLayout(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("path", "chunk_channels", "chunk_bytes", "k_blocks",
                                             "weight_rows", "weight_cols")] + \
               [("workspace_bytes", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_DESC = ctypes.POINTER(CbConvDesc)
_PLAN = ctypes.POINTER(CbSlicePlan)

_SIGNATURES = {
    "cb_version": ([], ctypes.c_int),
    "cb_last_error_string": ([], ctypes.c_char_p),
    "cb_device_sm_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cb_launch_count": ([], ctypes.c_uint64),
    "cb_event_create": ([ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "cb_event_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "cb_event_record": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "cb_event_elapsed_ns": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)],
                            ctypes.c_int),
    "cb_output_shape": ([_DESC, ctypes.POINTER(_I32), ctypes.POINTER(_I32)], ctypes.c_int),
    "cb_workspace_bytes": ([_DESC, ctypes.c_int, _PLAN, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "cb_im2col_f32": ([_DESC, _P, _P, _P], ctypes.c_int),
    "cb_sconv_plan": ([_DESC, _I32, _PLAN], ctypes.c_int),
    "cb_sconv_range": ([_DESC, _PLAN, _I32, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64)],
                       ctypes.c_int),
    "cb_sconv_pack_f32": ([_DESC, _PLAN, _I32, _I32, _P, _P, _P], ctypes.c_int),
    "cb_plan_tiles": ([ctypes.c_int, _DESC, _I64, ctypes.POINTER(CbTilePlan)], ctypes.c_int),
    "cb_split_kdim": ([_I32], _I32),
    "cb_weight_split": ([ctypes.c_int, _I32, _I32, _P, _P, _P, _P], ctypes.c_int),
    "cb_gemm": ([ctypes.c_int, _I32, _I32, _I32, _P, _P, _P, _P, _I64, _P, _I64, ctypes.c_int, _P],
                ctypes.c_int),
    "cb_conv_gemm_cols": ([ctypes.c_int, _DESC, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "cb_sconv_gemm": ([ctypes.c_int, _DESC, _PLAN, _I32, _I32, _P, _P, _P, _P, _P, _P],
                      ctypes.c_int),
    "cb_unpack_f32": ([_DESC, _PLAN, _I32, _I32, _P, _P, _P, _P], ctypes.c_int),
    "cb_env_fingerprint": ([], ctypes.c_uint64),
    "cb_fused_layout_query": ([ctypes.c_int, _DESC, ctypes.POINTER(CbFusedLayout)], ctypes.c_int),
    "cb_fused_reduction_map": ([ctypes.c_int, _DESC, _I32, ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "cb_fused_plan_tiles": ([ctypes.c_int, _DESC, ctypes.POINTER(CbTilePlan)], ctypes.c_int),
    "cb_fused_pack_weights": ([ctypes.c_int, _DESC, _P, _P, _P, _P], ctypes.c_int),
    "cb_fused_pack_input": ([ctypes.c_int, _DESC, _P, _P, ctypes.c_size_t, _P], ctypes.c_int),
    "cb_conv_fused_packed": ([ctypes.c_int, _DESC, _P, _P, ctypes.c_size_t, _P, _P, _P, _P, _P, _P],
                             ctypes.c_int),
    "cb_conv_fused": ([ctypes.c_int, _DESC, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P],
                      ctypes.c_int),
}

_lib = None
_lock = threading.Lock()


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library.  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise ConvB200Error(
                f"{p} is missing: build it with `python -m paper_2407_10730_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, (argtypes, restype) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = restype
        if path is None:
            _lib = lib
        return lib


def check(rc: int) -> None:
    """Raise the reference-equivalent exception for a non-zero status."""
    if rc == CB_OK:
        return
    msg = (load().cb_last_error_string() or b"").decode(errors="replace")
    if rc == CB_ERR_INVALID:
        raise InvalidDescriptorError(msg)
    if rc == CB_ERR_UNSUPPORTED:
        raise UnsupportedDescriptorError(msg)
    if rc == CB_ERR_WORKSPACE:
        raise MemoryError(msg)
    if rc == CB_ERR_MISALIGNED:
        raise ValueError(f"misaligned buffer: {msg}")
    raise ConvB200Error(msg or f"libconvb200 status {rc}")


def cdesc(d: ConvDescriptor) -> CbConvDesc:
    return CbConvDesc(d.batch, d.in_channels, d.in_h, d.in_w, d.out_channels, d.k_h, d.k_w,
                      d.stride_h, d.stride_w, d.pad_h, d.pad_w, d.dil_h, d.dil_w, d.groups,
                      1 if d.has_bias else 0)


def split_kdim(kdim: int) -> int:
    return int(load().cb_split_kdim(kdim))


def variant_id(name: str) -> int:
    try:
        return VARIANTS[name]
    except KeyError:
        raise ValueError(f"unknown variant {name!r}; choose from {sorted(VARIANTS)}") from None
