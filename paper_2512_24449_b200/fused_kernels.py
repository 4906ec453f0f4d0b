"""Fused decompress + GEMV over the compressed store.

SPEC surface (one head, batch 1):
  fused_k_scores(store, layer, head, q) -> ScoreVector
  fused_v_output(store, layer, head, w) -> f32 [head_dim]
Batched / GQA surface used by the decode step (one launch for every
(sequence, kv-head) unit, its blocks and its residue):
  fused_k_scores_batched(store, layer, q[B, Hq, D]) -> scores [B, Hq, L]
  fused_v_output_batched(store, layer, w[B, Hq, L]) -> out [B, Hq, D]
Query head hq reads kv head hq // (Hq / H).  Scores are in block/permuted
order followed by the residue; ``token_map`` gives each
position's original token index.

``naive_*`` decode the whole store to a dense matrix on the
GPU (pkv_decode_store + dequantize) and multiply — the two-step baseline.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import errors as E
from .kv_store import CompressedStore, ctypes_ref


@dataclass
class ScoreVector:
    """SPEC.md:434-438."""
    scores: torch.Tensor
    token_map: torch.Tensor


def _as_f32(x, dev) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x))
    return x.to(device=dev, dtype=torch.float32).contiguous()


def fused_k_scores_batched(store: CompressedStore, layer: int, q, out: torch.Tensor = None) -> torch.Tensor:
    ls = store[layer]
    q = _as_f32(q, store.device)
    B, H, D = store.batch, store.heads, store.head_dim
    if q.dim() != 3 or q.shape[0] != B or q.shape[2] != D or q.shape[1] % H:
        raise E.ShapeMismatchError(f"q must be [B={B}, Hq (multiple of {H}), D={D}], got {tuple(q.shape)}")
    Hq = int(q.shape[1])
    L = ls.tokens
    if out is None:
        out = torch.empty((B, Hq, max(L, 1)), dtype=torch.float32, device=store.device)
    N.check(N.lib().pkv_fused_k_scores(ctypes_ref(ls.struct()), ls.nblk_h, N.ptr(q), Hq, N.ptr(out),
                                       int(out.shape[-1]), N.stream()), "fused_k_scores")
    return out[..., :L]


def fused_v_output_batched(store: CompressedStore, layer: int, w, out: torch.Tensor = None) -> torch.Tensor:
    ls = store[layer]
    w = _as_f32(w, store.device)
    B, H, D = store.batch, store.heads, store.head_dim
    L = ls.tokens
    if w.dim() != 3 or w.shape[0] != B or w.shape[1] % H or w.shape[2] < L:
        raise E.ShapeMismatchError(f"w must be [B={B}, Hq, >= L={L}], got {tuple(w.shape)}")
    Hq = int(w.shape[1])
    lib = N.lib()
    st = ls.struct()
    need = int(lib.pkv_fused_v_scratch_bytes(ctypes_ref(st), ls.nblk_h, Hq))
    if need < 0:
        N.check(N.PKV_E_ARG, "fused_v_output")
    if ls.v_scratch.numel() < need:
        ls.v_scratch = torch.empty(need, dtype=torch.uint8, device=store.device)
    if out is None:
        out = torch.empty((B, Hq, D), dtype=torch.float32, device=store.device)
    N.check(lib.pkv_fused_v_output(ctypes_ref(st), ls.nblk_h, N.ptr(w), Hq, int(w.shape[-1]), N.ptr(out),
                                   N.ptr(ls.v_scratch), int(ls.v_scratch.numel()), N.stream()), "fused_v_output")
    return out


def token_map(store: CompressedStore, layer: int) -> torch.Tensor:
    """[B, L] original token index of every score position."""
    ls = store[layer]
    bl = store.block
    nb = ls.nblk_h
    perm = ls.perm[:, :nb].to(torch.int64)                                   # [B, nb, 64]
    base = (torch.arange(nb, device=store.device, dtype=torch.int64) * bl)[None, :, None]
    comp = (perm + base).reshape(store.batch, nb * bl)
    res = torch.arange(nb * bl, nb * bl + ls.nres_h, device=store.device, dtype=torch.int64)
    return torch.cat([comp, res[None].expand(store.batch, -1)], dim=1)


def _head_args(store, layer, head):
    if not (0 <= head < store.heads):
        raise IndexError(f"head {head} out of range [0, {store.heads})")
    if store.batch != 1:
        raise E.ShapeMismatchError("per-head API needs batch 1; use the *_batched functions")
    store[layer]


def fused_k_scores(store: CompressedStore, layer: int, head: int, q) -> ScoreVector:
    """SPEC.md:446-454."""
    _head_args(store, layer, head)
    q = _as_f32(q, store.device)
    if q.shape != (store.head_dim,):
        raise E.ShapeMismatchError(f"|q| must equal head_dim={store.head_dim}")
    qa = torch.zeros((1, store.heads, store.head_dim), dtype=torch.float32, device=store.device)
    qa[0, head] = q
    s = fused_k_scores_batched(store, layer, qa)[0, head]
    return ScoreVector(s, token_map(store, layer)[0])


def fused_v_output(store: CompressedStore, layer: int, head: int, w) -> torch.Tensor:
    """SPEC.md:455-463."""
    _head_args(store, layer, head)
    L = store[layer].tokens
    w = _as_f32(w, store.device)
    if w.shape != (L,):
        raise E.ShapeMismatchError(f"|w| must equal total tokens ({L})")
    wa = torch.zeros((1, store.heads, max(L, 1)), dtype=torch.float32, device=store.device)
    wa[0, head, :L] = w
    return fused_v_output_batched(store, layer, wa)[0, head]


# ---------------------------------------------------------------- naive
def decode_layer(store: CompressedStore, layer: int, kind: int) -> torch.Tensor:
    """Dense dequantized matrix [B*H, L, D] f32 in score order (blocks then residue)."""
    ls = store[layer]
    U = store.batch * store.heads
    nb, bl, D = ls.nblk_h, store.block, store.head_dim
    codes = torch.zeros((U, ls.max_blocks, bl, D), dtype=torch.uint16, device=store.device)
    params = torch.zeros((U, ls.max_blocks, bl, 2), dtype=torch.float32, device=store.device)
    N.check(N.lib().pkv_decode_store(ctypes_ref(ls.struct()), kind, N.ptr(codes), N.ptr(params), N.stream()),
            "decode_store")
    N.raise_flags(int(ls.err.item()), "decode_store")
    from .quantizer import dequantize
    deq = dequantize(codes[:, :nb].reshape(U, nb * bl, D), params[:, :nb, :, 0].reshape(U, nb * bl),
                     params[:, :nb, :, 1].reshape(U, nb * bl))
    res = ls.stage[kind, :, :ls.nres_h].float()
    return torch.cat([deq, res], dim=1)


def naive_k_scores(store: CompressedStore, layer: int, head: int, q) -> torch.Tensor:
    _head_args(store, layer, head)
    K = decode_layer(store, layer, 0)[head].double()
    return K @ _as_f32(q, store.device).double()


def naive_v_output(store: CompressedStore, layer: int, head: int, w) -> torch.Tensor:
    _head_args(store, layer, head)
    V = decode_layer(store, layer, 1)[head].double()
    return _as_f32(w, store.device).double() @ V


REPORT_FIELDS = ("kind", "mode", "tokens", "bytes_logical", "bytes_physical", "wall_ns", "gbps", "peak_alloc")


def bench_throughput(store: CompressedStore, layer: int, mode: str = "fused", reps: int = 10, q_heads=None):
    """SPEC.md:472-480 ThroughputReport rows {kind, mode, tokens, bytes_logical,
    bytes_physical, wall_ns, gbps, peak_alloc}, CUDA-event timed.

    gbps is over the uncompressed-equivalent bytes.  peak_alloc
    is the transient device allocation of one call beyond the tensor it
    returns (fused: nothing context-sized -- the split-L scratch is cached in
    the store after a warm-up call; naive: the dense [B*H, L, D] matrix),
    measured with torch's allocator counters around the call."""
    if mode not in ("fused", "naive"):
        raise ValueError("mode must be 'fused' or 'naive'")
    if reps < 1:
        raise ValueError("reps >= 1")
    ls = store[layer]
    B, H, D = store.batch, store.heads, store.head_dim
    Hq = q_heads or H
    L = ls.tokens
    q = torch.randn((B, Hq, D), device=store.device)
    w = torch.softmax(torch.randn((B, Hq, L), device=store.device), -1)
    _, ln, _ = ls.tables()
    rows = []
    for kind, fn in ((0, lambda: fused_k_scores_batched(store, layer, q)),
                     (1, lambda: fused_v_output_batched(store, layer, w))):
        if mode == "naive":
            fn = (lambda kind=kind: decode_layer(store, layer, kind))
        fn()  # warm-up: scratch cached in the store, modules loaded
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        r = fn()
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base - r.numel() * r.element_size()
        del r
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e6
        logical = B * H * L * D * 2
        phys = int(ln[kind].astype(np.int64).sum()) + B * H * ls.nres_h * D * 2
        rows.append({"kind": "K" if kind == 0 else "V", "mode": mode, "tokens": L, "bytes_logical": logical,
                     "bytes_physical": phys, "wall_ns": t, "gbps": logical / t, "peak_alloc": max(0, int(peak))})
    return rows


def report_rows(rows, fmt: str = "json") -> str:
    """ThroughputReport serialised as JSON lines or CSV rows, the
    fields in REPORT_FIELDS order."""
    import csv
    import io
    import json
    if fmt == "json":
        return "\n".join(json.dumps({k: r[k] for k in REPORT_FIELDS}) for r in rows) + "\n"
    if fmt == "csv":
        buf = io.StringIO()
        wr = csv.DictWriter(buf, fieldnames=REPORT_FIELDS, lineterminator="\n")
        wr.writeheader()
        for r in rows:
            wr.writerow({k: r[k] for k in REPORT_FIELDS})
        return buf.getvalue()
    raise ValueError("fmt must be 'json' or 'csv'")
