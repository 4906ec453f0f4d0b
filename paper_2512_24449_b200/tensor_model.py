"""Tensor containers' file format and synthetic KV inputs.

``read_dump`` / ``write_dump`` implement the "PKKV" KV-dump file
(layout :82): magic | version u16 = 1 | layers u16 | heads u16
| head_dim u16 | tokens u32 | per (layer, head) K then V, tokens x head_dim raw
little-endian f16, no padding.  Arrays are [layers, heads, tokens, head_dim].

``gauss_outlier`` is the bench workload of BASELINE.md §3: N(0,1) fp16 with
4/128 K outlier channels per (layer, kv-head) at +-8 + N(0, 2) (fixed sign per
channel) and 1/128 such V channel.  Deterministic for a fixed seed (torch's
CUDA generator), generated directly in HBM so large configs need no host copy.
"""
from __future__ import annotations

import struct

import numpy as np
import torch

from . import errors as E

_DUMP = struct.Struct("<4sHHHHI")


def write_dump(k, v, path) -> None:
    """k, v [layers, heads, tokens, head_dim] fp16 (numpy or torch)."""
    k = np.asarray(k.cpu() if isinstance(k, torch.Tensor) else k, dtype=np.float16)
    v = np.asarray(v.cpu() if isinstance(v, torch.Tensor) else v, dtype=np.float16)
    if k.shape != v.shape or k.ndim != 4:
        raise E.ShapeMismatchError("k and v must both be [layers, heads, tokens, head_dim]")
    if not (np.isfinite(k.astype(np.float32)).all() and np.isfinite(v.astype(np.float32)).all()):
        raise E.NonFiniteValueError("non-finite value in dump")
    L, H, T, D = k.shape
    body = np.stack([k, v], axis=2).astype("<f2")         # [L, H, 2, T, D]: K then V per (layer, head)
    with open(path, "wb") as f:
        f.write(_DUMP.pack(b"PKKV", 1, L, H, D, T))
        f.write(body.tobytes())


def read_dump(path):
    """SPEC.md:40-48 -> (k, v) fp16 numpy [layers, heads, tokens, head_dim].
    BadMagicError / TruncatedDumpError / NonFiniteValueError / DumpFormatError."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"PKKV":
        raise E.BadMagicError(f"{path}: not a PKKV dump")
    if len(data) < _DUMP.size:
        raise E.TruncatedDumpError(f"{path}: header truncated")
    _, ver, L, H, D, T = _DUMP.unpack_from(data)
    if ver != 1:
        raise E.DumpFormatError(f"{path}: unsupported version {ver}")
    need = _DUMP.size + 2 * 2 * L * H * T * D
    if len(data) < need:
        raise E.TruncatedDumpError(f"{path}: payload truncated ({len(data)} < {need} bytes)")
    if len(data) > need:
        raise E.DumpFormatError(f"{path}: {len(data) - need} trailing bytes")
    body = np.frombuffer(data, "<f2", offset=_DUMP.size).reshape(L, H, 2, T, D)
    if not np.isfinite(body.astype(np.float32)).all():
        raise E.NonFiniteValueError(f"{path}: non-finite value")
    return body[:, :, 0].astype(np.float16), body[:, :, 1].astype(np.float16)


def gauss_outlier(shape, head_dim_axis: int = -1, n_outlier: int = 4, amp: float = 8.0, sigma: float = 2.0,
                  seed: int = 0, device="cuda", heads_axis: int = -2) -> torch.Tensor:
    """fp16 tensor of `shape` (..., H, D): per kv head a fixed set of outlier channels."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    D = shape[head_dim_axis]
    H = shape[heads_axis]
    if n_outlier:
        # per kv head a fixed set of channels (the CPU generator's draws, head by
        # head), applied in one broadcast op instead of a launch chain per head
        gc = torch.Generator(device="cpu")
        gc.manual_seed(seed + 1)
        mask = torch.zeros((H, D), dtype=torch.bool)
        sgn = torch.zeros((H, D), dtype=torch.float32)
        for h in range(H):
            ch = torch.randperm(D, generator=gc)[:n_outlier]
            sign = (torch.randint(0, 2, (n_outlier,), generator=gc) * 2 - 1).float()
            mask[h, ch] = True
            sgn[h, ch] = sign
        bshape = [1] * len(shape)
        bshape[heads_axis] = H
        bshape[head_dim_axis] = D
        mask = mask.view(bshape).to(device)
        sgn = sgn.view(bshape).to(device)
        x = torch.where(mask, sgn * amp + sigma * x, x)
    return x.to(torch.float16)


SYNTH_MODES = ("uniform", "channel-banded", "token-scaled", "gauss-outlier")


def generate_synthetic(mode: str, seed: int, layers: int, heads: int, head_dim: int, tokens: int,
                       amplitude: float = 1.0, device="cuda"):
    """(K, V) fp16 [layers, heads, tokens, head_dim], generated in HBM
    with torch's CUDA generator (same seed + profile => byte-identical output):

    * uniform         U(-a, a);
    * channel-banded  a per-(layer, head, channel) offset U(-4a, 4a) + 0.25a N(0, 1):
                      adjacent tokens of a column are correlated (Fig. 4);
    * token-scaled    per-token scale U(0.1, 2)a times N(0, 1);
    * gauss-outlier   the bench distribution (gauss_outlier).
    """
    if mode not in SYNTH_MODES:
        raise ValueError(f"unknown synthetic mode {mode!r}; one of {SYNTH_MODES}")
    if min(layers, heads, head_dim) < 1 or tokens < 0:
        raise ValueError("counts must be >= 1 (tokens >= 0)")
    shape = (layers, heads, tokens, head_dim)
    if mode == "gauss-outlier":
        k = gauss_outlier((layers, tokens, heads, head_dim), n_outlier=max(1, head_dim * 4 // 128), seed=seed,
                          device=device, heads_axis=-2)
        v = gauss_outlier((layers, tokens, heads, head_dim), n_outlier=max(1, head_dim // 128), seed=seed + 7,
                          device=device, heads_axis=-2)
        return k.permute(0, 2, 1, 3).contiguous(), v.permute(0, 2, 1, 3).contiguous()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    a = float(amplitude)
    out = []
    for _ in range(2):
        if mode == "uniform":
            x = (torch.rand(shape, generator=g, device=device) * 2 - 1) * a
        elif mode == "channel-banded":
            off = (torch.rand((layers, heads, 1, head_dim), generator=g, device=device) * 8 - 4) * a
            x = off + 0.25 * a * torch.randn(shape, generator=g, device=device)
        else:
            sc = (0.1 + 1.9 * torch.rand((layers, heads, tokens, 1), generator=g, device=device)) * a
            x = sc * torch.randn(shape, generator=g, device=device)
        out.append(x.to(torch.float16))
    return out[0], out[1]
