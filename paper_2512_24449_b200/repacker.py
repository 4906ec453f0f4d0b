"""Encode-aware token repacking, the plans on the GPU.

``repack_greedy`` (Algorithm 1) and ``repack_v_median``
 run the same device kernel the compressor uses
(csrc/store.cu ``store_plan_kernel`` through ``pkv_repack_plan``), so a plan
computed here is the permutation the store applies to the same codes.  The
vectors are laid out as the kernel's codes: the K part as "kind 0" and the V
part as "kind 1", each split into head-sized pieces.  ``pack_cost`` /
``plan_cost`` are the SPEC's integer cost model (host arithmetic on code ranges,
like ``bitpack_codec.compression_ratio``).  ``oracle_optimal`` (an exhaustive
test-only search) lives in the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import errors as E

META_BITS = 20  # 4-bit width + 16-bit minimum per pack


@dataclass
class RepackPlan:
    """SPEC.md:181-186."""
    permutation: np.ndarray
    strategy: str
    cost_bits: int


def _as_int(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.int64)


def _bit_length(r: np.ndarray) -> np.ndarray:
    r = np.asarray(r, dtype=np.int64)
    out = np.zeros(r.shape, dtype=np.int64)
    m = r > 0
    out[m] = np.frexp(r[m].astype(np.float64))[1]  # exact for ranges < 2^53
    return out


def pack_cost(group) -> int:
    """sum_d (|g| * w_d + META_BITS), w_d = ceil(log2(range_d + 1))."""
    g = _as_int(group)
    if g.ndim == 1:
        g = g[None, :]
    if g.shape[0] == 0:
        raise ValueError("pack_cost of an empty group")
    return int(np.sum(g.shape[0] * _bit_length(g.max(axis=0) - g.min(axis=0)) + META_BITS))


def plan_cost(vectors, perm, k: int) -> int:
    """Total pack_cost of consecutive groups of k in permuted order."""
    v = _as_int(vectors)[np.asarray(perm, dtype=np.int64)]
    return sum(pack_cost(v[i:i + k]) for i in range(0, v.shape[0], k))


def repack_none(vectors, k: int) -> RepackPlan:
    n = _as_int(vectors).shape[0]
    perm = np.arange(n, dtype=np.int64)
    return RepackPlan(perm, "none", plan_cost(vectors, perm, k) if n else 0)


def _layout(k_part: np.ndarray, v_part: np.ndarray):
    """[n, Dk] / [n, Dv] codes -> the kernel's [1 set][1 seq][2 kinds][H][n][Dh] u16
    (zero padding: a zero column changes neither the costs nor the distances)."""
    n = k_part.shape[0]
    D = max(k_part.shape[1], v_part.shape[1], 1)
    Dh = D if D <= 1024 else 128
    H = -(-D // Dh)
    codes = np.zeros((1, 1, 2, H, n, Dh), dtype=np.uint16)
    for kind, part in ((0, k_part), (1, v_part)):
        flat = np.zeros((n, H * Dh), dtype=np.uint16)
        flat[:, :part.shape[1]] = part
        codes[0, 0, kind] = flat.reshape(n, H, Dh).transpose(1, 0, 2)
    return codes, H, Dh


def _device_plan(k_part: np.ndarray, v_part: np.ndarray, k: int, strategy: int) -> np.ndarray:
    n = k_part.shape[0]
    if not (1 <= n <= 64):
        raise ValueError(f"plans cover 1..64 vectors (a store block-set), got {n}")
    if k not in (2, 4, 8, 16, 32):
        raise ValueError("pack_size must be one of 2, 4, 8, 16, 32")
    for part in (k_part, v_part):
        if part.size and (part.min() < 0 or part.max() > 65535):
            raise E.WidthOverflowError("repack vectors must be u16 quantized codes")
    codes, H, Dh = _layout(k_part, v_part)
    dev = torch.device("cuda", torch.cuda.current_device())
    c = torch.from_numpy(codes.view(np.int16)).to(dev)
    perm = torch.empty((1, 1, n), dtype=torch.uint8, device=dev)
    N.check(N.lib().pkv_repack_plan(N.ptr(c), 1, 1, H, Dh, n, k, strategy, N.ptr(perm), N.stream()),
            "repack_plan")
    return perm.view(-1).cpu().numpy().astype(np.int64)


def repack_greedy(vectors, k: int) -> RepackPlan:
    """SPEC.md:198-207 on the GPU: vectors [n <= 64, D] non-negative codes (the
    concatenated K and V parts of each token)."""
    X = _as_int(vectors)
    if X.ndim != 2:
        raise E.ShapeMismatchError("vectors must be [n, d]")
    half = (X.shape[1] + 1) // 2
    perm = _device_plan(X[:, :half], X[:, half:], k, N.REPACK["greedy"])
    return RepackPlan(perm, "greedy", plan_cost(X, perm, k))


def repack_v_median(vectors, v_parts, k: int) -> RepackPlan:
    """SPEC.md:208-216 on the GPU: stable ascending sort by the lower median of
    each token's V part."""
    X = _as_int(vectors)
    V = _as_int(v_parts)
    if V.ndim != 2 or V.shape[0] != X.shape[0]:
        raise E.ShapeMismatchError("v_parts must be [n, d_v] with the vectors' n")
    if V.shape[1] > 1024 and V.shape[1] % 128:
        raise ValueError("a V part longer than 1024 must be a multiple of 128 (heads x head_dim)")
    perm = _device_plan(np.zeros_like(V), V, k, N.REPACK["v_median"])
    return RepackPlan(perm, "v_median", plan_cost(X, perm, k))
