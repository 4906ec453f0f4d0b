"""ctypes binding of libpackkv_b200.so (the C ABI in include/packkv_b200.h).

This is the only place the package touches native code.  There is no CPU
fallback: if the library is missing or no CUDA device is present, every
compute call raises.  Pointers passed across the boundary are device pointers
of torch tensors; every call is enqueued on torch's current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_float, c_int32, c_int64, c_void_p

from . import errors as E

LIB_NAME = "libpackkv_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

PKV_OK, PKV_E_SHAPE, PKV_E_NONFINITE, PKV_E_WIDTH, PKV_E_MALFORMED = 0, 1, 2, 3, 4
PKV_E_INDEX, PKV_E_ARG, PKV_E_CUDA, PKV_E_CAPACITY = 5, 6, 7, 8
FLAG_NONFINITE, FLAG_WIDTH, FLAG_MALFORMED, FLAG_CAPACITY, FLAG_SHAPE = 1, 2, 4, 8, 16
PATH_NONE, PATH_FAST, PATH_GENERIC, PATH_SINGLE = 0, 1, 2, 3
REPACK = {"none": 0, "greedy": 1, "v_median": 2}
REPACK_EXTERNAL = 3


class CapacityError(E.PackKVError):
    """Arena or block table too small (the store grows and retries)."""


class NativeError(RuntimeError):
    """CUDA launch/runtime failure inside libpackkv_b200."""


class Layer(ctypes.Structure):
    """Mirror of pkv_layer_t (include/packkv_b200.h)."""
    _fields_ = [
        ("batch", c_int32), ("heads", c_int32), ("head_dim", c_int32), ("block", c_int32),
        ("pack_size", c_int32), ("buffer", c_int32), ("max_blocks", c_int32), ("reserved", c_int32),
        ("arena", c_void_p), ("arena_capacity", c_int64), ("tail", c_void_p), ("blk_off", c_void_p),
        ("blk_len", c_void_p), ("perm", c_void_p), ("nblk", c_void_p), ("nres", c_void_p),
        ("stage", c_void_p), ("err", c_void_p),
    ]


_SIGS = {
    "pkv_last_error": (ctypes.c_char_p, []),
    "pkv_version": (c_int32, []),
    "pkv_last_path": (c_int32, []),
    "pkv_quantize": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_float, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pkv_check_finite": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p]),
    "pkv_copy_scaled": (c_int32, [c_void_p, c_void_p, c_int64, c_float, c_void_p]),
    "pkv_dequantize": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "pkv_encode_sizes": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    "pkv_encode": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p,
                             c_void_p, c_void_p, c_void_p]),
    "pkv_decode": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                             c_void_p]),
    "pkv_decode_pack_at": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    "pkv_compress_scratch_bytes": (c_int64, [POINTER(Layer), c_int32]),
    "pkv_compress_scratch_bytes_ex": (c_int64, [POINTER(Layer), c_int32, c_int32]),
    "pkv_stage_token": (c_int32, [POINTER(Layer), c_void_p, c_void_p, c_void_p]),
    "pkv_compress_codes": (c_int32, [POINTER(Layer), c_void_p, c_void_p, c_int32, c_int32, c_float, c_float, c_void_p,
                                     c_void_p, c_void_p]),
    "pkv_repack_plan": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p,
                                  c_void_p]),
    "pkv_compress_tokens": (c_int32, [POINTER(Layer), c_void_p, c_void_p, c_int32, c_int32, c_int32, c_float, c_float,
                                      c_int32, c_void_p, c_int64, c_void_p]),
    "pkv_flush_scratch_bytes": (c_int64, [POINTER(Layer)]),
    "pkv_flush_staged": (c_int32, [POINTER(Layer), c_float, c_float, c_void_p, c_int64, c_void_p]),
    "pkv_fused_k_scores": (c_int32, [POINTER(Layer), c_int32, c_void_p, c_int32, c_void_p, c_int64, c_void_p]),
    "pkv_fused_v_scratch_bytes": (c_int64, [POINTER(Layer), c_int32, c_int32]),
    "pkv_fused_v_output": (c_int32, [POINTER(Layer), c_int32, c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_int64,
                                     c_void_p]),
    "pkv_decode_store": (c_int32, [POINTER(Layer), c_int32, c_void_p, c_void_p, c_void_p]),
    "pkv_attention_scratch_bytes": (c_int64, [POINTER(Layer), c_int32, c_int32]),
    "pkv_attention_decode": (c_int32, [POINTER(Layer), c_int32, c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_void_p,
                                       c_int64, c_void_p]),
    "pkv_append_flush": (c_int32, [POINTER(Layer), c_void_p, c_void_p, c_float, c_float, c_void_p, c_int64, c_void_p]),
    "pkv_append_flush_masked": (c_int32, [POINTER(Layer), c_void_p, c_void_p, c_void_p, c_float, c_float, c_void_p,
                                          c_int64, c_void_p]),
}

_lib = None


def exported_symbols():
    return list(_SIGS)


def load(require_cuda: bool = False):
    """Load the library (once).  Raises loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make`). "
                "There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("packkv_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    return _lib


_cuda_ok = False


def lib():
    global _cuda_ok
    if _cuda_ok:
        return _lib
    out = load(require_cuda=True)
    _cuda_ok = True
    return out


def last_error() -> str:
    return load().pkv_last_error().decode(errors="replace")


def check(status: int, what: str = ""):
    if status == PKV_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == PKV_E_SHAPE:
        raise E.ShapeMismatchError(msg)
    if status == PKV_E_NONFINITE:
        raise E.NonFiniteValueError(msg)
    if status == PKV_E_WIDTH:
        raise E.WidthOverflowError(msg)
    if status == PKV_E_MALFORMED:
        raise E.MalformedBlockError(msg)
    if status == PKV_E_INDEX:
        raise IndexError(msg)
    if status == PKV_E_ARG:
        raise ValueError(msg)
    if status == PKV_E_CAPACITY:
        raise CapacityError(msg)
    raise NativeError(msg)


def raise_flags(flags: int, what: str = ""):
    """Map device-side PKV_FLAG_* bits onto packkv.errors classes."""
    if not flags:
        return
    if flags & FLAG_NONFINITE:
        raise E.NonFiniteValueError(f"{what}: NaN or infinity in fp16 input")
    if flags & FLAG_WIDTH:
        raise E.WidthOverflowError(f"{what}: pack range needs more than 15 bits or scale overflows f16")
    if flags & FLAG_MALFORMED:
        raise E.MalformedBlockError(f"{what}: block header or length invalid")
    if flags & FLAG_CAPACITY:
        raise CapacityError(f"{what}: arena capacity exceeded")
    if flags & FLAG_SHAPE:
        raise E.ShapeMismatchError(f"{what}: score / weight row stride shorter than the token count")


def last_path() -> int:
    """PATH_FAST / PATH_GENERIC / PATH_SINGLE: kernel family of this thread's last fused call."""
    return int(load().pkv_last_path())


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def stream() -> int:
    """The current CUDA stream of the current device, as a raw handle.  Uses
    torch's C accessor (torch.cuda.current_stream() builds a Python Stream
    object and re-validates the device: ~10 us per call on the append path)."""
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(torch._C._cuda_getDevice()))
    return int(torch.cuda.current_stream().cuda_stream)
