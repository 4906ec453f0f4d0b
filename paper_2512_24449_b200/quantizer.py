"""Token-wise error-bounded quantizer on the GPU.

Same operations as the reference module ``quantizer``: ``quantize_token_wise``
(SPEC.md:111-119), ``dequantize`` and ``max_abs_error``
(SPEC.md:129-137).  Inputs are fp16 torch tensors ``[rows, cols]`` (one head's
slice) or ``[n, rows, cols]`` (n independent slices); the arithmetic runs in
``pkv_quantize`` / ``pkv_dequantize`` (csrc/codec.cu) with f32 IEEE division
and round-half-away-from-zero, bit-identical to the CPU oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N
from . import errors as E

KIND_K, KIND_V = 0, 1


@dataclass
class QuantParams:
    """SPEC.md:96-101."""
    rel_quant_scale: float

    @property
    def rel_error_bound(self) -> float:
        return self.rel_quant_scale / 2


@dataclass
class QuantBlock:
    """SPEC.md:102-108.  q: uint16 codes [..., rows, cols]; scale/zp: f32 [..., rows]."""
    q: torch.Tensor
    scale: torch.Tensor
    zp: torch.Tensor
    kind: int = KIND_K
    rel: float = 0.1

    @property
    def rows(self) -> int:
        return self.q.shape[-2]

    @property
    def cols(self) -> int:
        return self.q.shape[-1]


def as_half_cuda(x, device=None) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    dev = torch.device(device) if device is not None else (x.device if x.is_cuda else torch.device("cuda"))
    if x.dtype != torch.float16:
        x = x.to(torch.float16)
    return x.to(dev).contiguous()


def _flags(t: torch.Tensor, what: str):
    N.raise_flags(int(t.item()), what)


def quantize_token_wise(x, rel_quant_scale: float, kind: int = KIND_K) -> QuantBlock:
    """per row: scale = rel*(max-min), q = round((x-min)/scale)."""
    x = as_half_cuda(x)
    if x.dim() not in (2, 3):
        raise E.ShapeMismatchError("quantize_token_wise expects [rows, cols] or [n, rows, cols]")
    if not (0.0 < rel_quant_scale <= 1.0):
        raise ValueError("rel_quant_scale must be in (0, 1]")
    lead = x.shape[:-2]
    n = int(x.shape[0]) if x.dim() == 3 else 1
    rows, cols = int(x.shape[-2]), int(x.shape[-1])
    q = torch.empty(x.shape, dtype=torch.uint16, device=x.device)
    params = torch.empty(lead + (rows, 2), dtype=torch.float32, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    N.check(N.lib().pkv_quantize(N.ptr(x), n, rows, cols, float(rel_quant_scale), N.ptr(q), N.ptr(params),
                                 N.ptr(err), N.stream()), "quantize_token_wise")
    flags = int(err.item())
    if flags & N.FLAG_NONFINITE:
        raise E.NonFiniteValueError("non-finite value in quantizer input")
    if flags & N.FLAG_WIDTH:
        raise E.WidthOverflowError("quantized value >= 2^16 (rel_quant_scale too small)")
    return QuantBlock(q, params[..., 0], params[..., 1], kind, float(rel_quant_scale))


def dequantize(q, scale=None, zp=None) -> torch.Tensor:
    """q*scale + zp in f32 (mul then add).  Accepts a QuantBlock."""
    if isinstance(q, QuantBlock):
        q, scale, zp = q.q, q.scale, q.zp
    q = q.to(torch.uint16).contiguous() if q.dtype != torch.uint16 else q.contiguous()
    rows, cols = int(q.shape[-2]), int(q.shape[-1])
    n = int(q.numel() // (rows * cols)) if rows * cols else 0
    params = torch.stack([scale.to(torch.float32), zp.to(torch.float32)], dim=-1).contiguous()
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    N.check(N.lib().pkv_dequantize(N.ptr(q), N.ptr(params), n, rows, cols, N.ptr(out), N.stream()), "dequantize")
    return out


def max_abs_error(x, rel_quant_scale: float) -> float:
    """SPEC.md:129-137."""
    x = as_half_cuda(x)
    qb = quantize_token_wise(x, rel_quant_scale)
    d = dequantize(qb)
    if d.numel() == 0:
        return 0.0
    return float((x.float() - d).abs().max().item())
