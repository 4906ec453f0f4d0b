"""Decode-step attention over the compressed store.

attention_decode composes fused_k_scores -> 1/sqrt(d) -> stable softmax ->
fused_v_output; scores stay in block/permuted order, which
single-query attention is invariant to (proof box).
"""
from __future__ import annotations

import math

import torch

from . import errors as E
from .fused_kernels import fused_k_scores_batched, fused_v_output_batched, _as_f32
from .kv_store import CompressedStore


def attention_decode_batched(store: CompressedStore, layer: int, q) -> torch.Tensor:
    """q [B, Hq, D] -> out [B, Hq, D]."""
    s = fused_k_scores_batched(store, layer, q)
    a = torch.softmax(s * (1.0 / math.sqrt(store.head_dim)), dim=-1)
    return fused_v_output_batched(store, layer, a)


def attention_decode(store: CompressedStore, layer: int, head: int, q) -> torch.Tensor:
    """SPEC.md:520-528 (batch 1, one head)."""
    if not (0 <= head < store.heads):
        raise IndexError("head out of range")
    q = _as_f32(q, store.device)
    if q.shape != (store.head_dim,):
        raise E.ShapeMismatchError("|q| must equal head_dim")
    qa = torch.zeros((1, store.heads, store.head_dim), dtype=torch.float32, device=store.device)
    qa[0, head] = q
    return attention_decode_batched(store, layer, qa)[0, head]


def attention_reference(K, V, q) -> torch.Tensor:
    """direct f64 softmax(Kq/sqrt(d))^T V."""
    K = torch.as_tensor(K).double()
    V = torch.as_tensor(V).double()
    q = torch.as_tensor(q).double().to(K.device)
    if K.shape != V.shape or K.shape[1] != q.shape[0]:
        raise E.ShapeMismatchError("K, V, q dimensions disagree")
    return torch.softmax(K @ q / math.sqrt(K.shape[1]), 0) @ V
