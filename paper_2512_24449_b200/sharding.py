"""(batch, kv-head) sharding of the compressed KV cache across GPUs.

The reference has no multi-GPU code (SPEC.md:8 reduces it to a concurrency
contract; PAPER.md:888-890 runs independent instances).  Following BASELINE.json
north_star (3): every rank owns a disjoint set of (sequence, kv-head) units —
its own arena, block tables and staging — so appends and the fused K/V GEMVs
never cross devices; the only collective is one all-gather of the per-head
attention outputs per decode step (NCCL over NVLink with the "nccl" backend,
gloo on CPU in tests).

Partition rule (``plan_partition``): split kv-heads when H % N == 0 (GQA query
groups stay with their kv-head), else split the batch when B % N == 0; ragged
splits are not supported (every rank must run the same kernels on the same
shapes so the all-gather is a single fixed-size collective).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import errors as E


@dataclass(frozen=True)
class Partition:
    mode: str            # "head" or "batch"
    world: int
    rank: int
    batch: int           # global
    kv_heads: int        # global
    b0: int
    b1: int
    h0: int
    h1: int

    @property
    def local_batch(self) -> int:
        return self.b1 - self.b0

    @property
    def local_heads(self) -> int:
        return self.h1 - self.h0

    def units(self):
        """Global (b, h) units owned by this rank, b-major."""
        return [(b, h) for b in range(self.b0, self.b1) for h in range(self.h0, self.h1)]


def plan_partition(batch: int, kv_heads: int, world: int, rank: int, prefer: Optional[str] = None) -> Partition:
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    modes = [prefer] if prefer else ["head", "batch"]
    for mode in modes:
        if mode == "head" and kv_heads % world == 0:
            n = kv_heads // world
            return Partition("head", world, rank, batch, kv_heads, 0, batch, rank * n, (rank + 1) * n)
        if mode == "batch" and batch % world == 0:
            n = batch // world
            return Partition("batch", world, rank, batch, kv_heads, rank * n, (rank + 1) * n, 0, kv_heads)
    raise E.ShapeMismatchError(f"cannot shard batch={batch} x kv_heads={kv_heads} evenly over {world} ranks")


def local_slice(p: Partition, x: torch.Tensor, head_axis: int, batch_axis: int = 0, group: int = 1) -> torch.Tensor:
    """This rank's slice of a global [B, ..., H*group, ...] tensor."""
    x = x.narrow(batch_axis, p.b0, p.local_batch)
    return x.narrow(head_axis, p.h0 * group, p.local_heads * group)


def assemble(p: Partition, gathered: torch.Tensor) -> torch.Tensor:
    """[world, B_loc, Hq_loc, D] all-gathered shards -> global [B, Hq, D]."""
    if p.mode == "batch":
        return gathered.reshape(p.world * gathered.shape[1], *gathered.shape[2:])
    # head split: [world, B, Hq_loc, D] -> [B, world * Hq_loc, D]
    return gathered.permute(1, 0, 2, 3).reshape(gathered.shape[1], -1, gathered.shape[3])


class ShardedDecoder:
    """One decode step over a sharded cache: local fused K -> softmax -> fused V
    on this rank's units, then one all-gather of the per-head outputs.

    ``local_attention(q_local) -> out_local`` defaults to the CUDA path
    (attention_sim.attention_decode_batched on this rank's CompressedStore);
    tests inject other callables to exercise the partition/collective logic."""

    def __init__(self, partition: Partition, local_attention: Callable[[torch.Tensor], torch.Tensor],
                 q_heads: int, head_dim: int, group=None):
        if q_heads % partition.kv_heads:
            raise E.ShapeMismatchError("q_heads must be a multiple of kv_heads")
        self.p = partition
        self.G = q_heads // partition.kv_heads
        self.q_heads, self.head_dim = q_heads, head_dim
        self.local_attention = local_attention
        self.group = group
        self._gather = None

    def local_q(self, q: torch.Tensor) -> torch.Tensor:
        """Global q [B, Hq, D] -> this rank's [B_loc, Hq_loc, D]."""
        return local_slice(self.p, q, head_axis=1, group=self.G).contiguous()

    def step(self, q_local: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
        """out (optional, host): receives the global output.  With one rank, a pinned host
        q_local and a local attention that writes host memory itself (GraphedAttention),
        q and out move inside the decode graph (zero-copy); otherwise out is filled by an
        asynchronous copy of the gathered result."""
        if self.p.world == 1 and out is not None and getattr(self.local_attention, "supports_host_out", False) \
                and not q_local.is_cuda and q_local.is_pinned() and out.is_pinned():
            return self.local_attention(q_local, out=out.view(q_local.shape))
        out_local = self.local_attention(q_local).contiguous()
        if self.p.world == 1:
            if out is not None:
                out.view(out_local.shape).copy_(out_local, non_blocking=True)
                return out
            return out_local
        shape = (self.p.world,) + tuple(out_local.shape)
        if self._gather is None or self._gather.shape != shape or self._gather.device != out_local.device:
            self._gather = torch.empty(shape, dtype=out_local.dtype, device=out_local.device)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self._gather.view(-1, *out_local.shape[1:]), out_local, group=self.group)
        else:
            dist.all_gather(list(self._gather.unbind(0)), out_local, group=self.group)
        res = assemble(self.p, self._gather)
        if out is not None:
            out.view(res.shape).copy_(res, non_blocking=True)
            return out
        return res


def _all_gather(t: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[world, *t.shape] gathered copies of t (NCCL: one all_gather_into_tensor)."""
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out.view(-1, *t.shape[1:]) if t.dim() else out, t, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), t, group=group)
    return out


def gather_codes(codes: torch.Tensor, p: Partition, all_gather) -> torch.Tensor:
    """This rank's int16 codes [nsets, B, 2, H_loc, block, D] (kv-head split)
    -> every head's [nsets, B, 2, world * H_loc, block, D], heads in global
    order.  Exchanged as bytes (NCCL has no 16-bit integer type)."""
    nsets, B, two, Hl, blk, D = codes.shape
    g = all_gather(codes.contiguous().view(torch.uint8)).view(torch.int16)
    g = g.reshape(p.world, nsets, B, two, Hl, blk, D)
    return g.permute(1, 2, 3, 0, 4, 5, 6).reshape(nsets, B, two, p.world * Hl, blk, D).contiguous()


def compress_sharded(store, p: Partition, layer: int, k_local, v_local, all_gather=None, group=None):
    """compress_batch / append for this rank's units with repacking that
    matches a single device holding every head:
    the plan of a block-set is shared by all heads of a sequence, so under a
    kv-head split each rank quantizes the block-sets the call completes
    (pkv_compress_codes), the int codes of all heads are all-gathered (as
    bytes), every rank computes the same plan from them (pkv_repack_plan) and
    compresses with it (PKV_REPACK_EXTERNAL).  Batch splits and repack "none"
    need no exchange.  k_local / v_local: [B_loc, T, H_loc, D] fp16.
    all_gather(t) -> [world, *t.shape] defaults to torch.distributed."""
    from . import _native as N
    ls = store[layer]
    k = store._norm(k_local, True)
    v = store._norm(v_local, True)
    if store.repack == "none" or p.mode == "batch" or p.world == 1:
        ls.compress(k, v, store.check)
        return
    codes = ls.pending_codes(k, v)
    gather = all_gather or (lambda t: _all_gather(t, p.world, group))
    if codes is None:  # every rank completes the same number of block-sets (lockstep batch)
        ls.compress(k, v, store.check)
        return
    allc = gather_codes(codes, p, gather)
    nsets, B, _, Hl, blk, D = codes.shape
    perm = torch.empty((B, nsets, blk), dtype=torch.uint8, device=allc.device)
    N.check(N.lib().pkv_repack_plan(N.ptr(allc), nsets, B, p.world * Hl, D, blk, store.pack_size,
                                    N.REPACK[store.repack], N.ptr(perm), N.stream()), "repack_plan")
    ls.compress(k, v, store.check, perm=perm)


def make_local_store(p: Partition, layers: int, head_dim: int, **kw):
    """CompressedStore holding this rank's units (CUDA)."""
    from .kv_store import CompressedStore
    return CompressedStore(layers, p.local_heads, head_dim, batch=p.local_batch, **kw)


def cuda_local_attention(store, layer: int = 0, graph: bool = True):
    """This rank's decode attention on the CUDA path: replayed as one CUDA graph
    per step (attention_sim.GraphedAttention) or launched eagerly."""
    from .attention_sim import GraphedAttention, attention_decode_batched
    if graph:
        return GraphedAttention(store, layer)
    return lambda q_local: attention_decode_batched(store, layer, q_local)
