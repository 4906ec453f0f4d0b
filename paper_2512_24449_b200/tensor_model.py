"""Synthetic KV inputs generated on the device.

``gauss_outlier`` is the bench workload of BASELINE.md §3: N(0,1) fp16 with
4/128 K outlier channels per (layer, kv-head) at +-8 + N(0, 2) (fixed sign per
channel) and 1/128 such V channel.  Deterministic for a fixed seed (torch's
CUDA generator), generated directly in HBM so large configs need no host copy.
"""
from __future__ import annotations

import torch


def gauss_outlier(shape, head_dim_axis: int = -1, n_outlier: int = 4, amp: float = 8.0, sigma: float = 2.0,
                  seed: int = 0, device="cuda", heads_axis: int = -2) -> torch.Tensor:
    """fp16 tensor of `shape` (..., H, D): per kv head a fixed set of outlier channels."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    D = shape[head_dim_axis]
    H = shape[heads_axis]
    if n_outlier:
        gc = torch.Generator(device="cpu")
        gc.manual_seed(seed + 1)
        for h in range(H):
            ch = torch.randperm(D, generator=gc)[:n_outlier]
            sign = (torch.randint(0, 2, (n_outlier,), generator=gc) * 2 - 1).float()
            idx = [slice(None)] * len(shape)
            idx[heads_axis] = h
            sub = x[tuple(idx)]                      # (..., D) view
            sub[..., ch.to(device)] = sign.to(device) * amp + sigma * sub[..., ch.to(device)]
    return x.to(torch.float16)
