"""Appendable compressed KV store, device resident.

A ``CompressedStore`` holds ``layers`` independent sub-stores,
each for a batch of ``batch`` sequences × ``heads`` KV heads.  Per layer the
HBM layout is:

  arena     uint8 [capacity]            PackedBlocks at 16-byte aligned offsets
  blk_off   int64 [2, B*H, max_blocks]  block directory: byte offset per block
  blk_len   int32 [2, B*H, max_blocks]  exact block length (SPEC.md:330 bytes)
  perm      uint8 [B, max_blocks, 64]   shared K/V repack permutation per block-set
  nblk/nres int32 [B]                   blocks / staged residue tokens per sequence
  stage     fp16  [2, B*H, buffer, D]   uncompressed staging ring

``append_token`` / ``compress_batch`` enqueue the device
compressor (csrc/store.cu) on the current stream; the host keeps mirrors of
the token counts so no device round trip is needed to decide flushes, and an
upper bound of the arena tail so capacity is only synchronised when it may run
out.  Sequences advance in lockstep (every call appends the same tokens count
to every sequence of the batch).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import _native as N
from . import errors as E
from .bitpack_codec import header_bytes

KIND_K, KIND_V = 0, 1
REPACK_STRATEGIES = ("none", "greedy", "v_median")


def _round16(x: int) -> int:
    return (x + 15) & ~15


def max_block_bytes(rows: int, cols: int, k: int) -> int:
    return header_bytes(rows, cols, k) + (rows // k) * cols * ((k * 15 + 7) // 8)


@dataclass
class BlockDirectoryEntry:
    """SPEC.md:351-356 (plus the sequence index of a batched store)."""
    kind: int
    layer: int
    head: int
    token_start: int
    token_end: int
    byte_offset: int
    byte_len: int
    permutation: np.ndarray
    seq: int = 0


@dataclass
class ResidueHandle:
    """Terminal handle of iterate_blocks: the staged, uncompressed tokens."""
    layer: int
    token_start: int
    tokens: int
    seq: int = 0


class LayerStore:
    """One layer's device-resident sub-store (see module docstring)."""

    def __init__(self, owner: "CompressedStore", layer: int, init_blocks: int):
        self.owner = owner
        self.layer = layer
        o = owner
        dev = o.device
        U = o.batch * o.heads
        self.max_blocks = max(1, init_blocks)
        self.blk_max = _round16(max_block_bytes(o.block, o.head_dim, o.pack_size))
        cap = self._expected_bytes(self.max_blocks)
        # never read beyond the tail (blocks carry their own zero padding): no fill
        self.arena = torch.empty(cap + 16, dtype=torch.uint8, device=dev)
        self.tail = torch.zeros(1, dtype=torch.int64, device=dev)
        self.blk_off = torch.full((2, U, self.max_blocks), -1, dtype=torch.int64, device=dev)
        self.blk_len = torch.zeros((2, U, self.max_blocks), dtype=torch.int32, device=dev)
        self.perm = torch.zeros((o.batch, self.max_blocks, o.block), dtype=torch.uint8, device=dev)
        self.nblk = torch.zeros(o.batch, dtype=torch.int32, device=dev)
        self.nres = torch.zeros(o.batch, dtype=torch.int32, device=dev)
        self.stage = torch.zeros((2, U, o.buffer, o.head_dim), dtype=torch.float16, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.scratch = torch.empty(0, dtype=torch.uint8, device=dev)
        self.v_scratch = torch.empty(0, dtype=torch.uint8, device=dev)
        self.a_scratch = torch.empty(0, dtype=torch.uint8, device=dev)
        # host mirrors
        self.nblk_h = 0
        # True once the sequences' lengths diverge (GraphedDecodeLoop with an
        # active mask): nblk_h / nres_h then hold the largest counts (sizing
        # only); the device nblk[b] / nres[b] are each sequence's own
        self.ragged = False
        self.nres_h = 0
        self.tail_ub = 0
        self._struct = None

    # -- geometry ---------------------------------------------------------------
    def _expected_bytes(self, blocks: int) -> int:
        o = self.owner
        # typical compressed block ~ raw/4; start there and grow geometrically
        per = _round16(header_bytes(o.block, o.head_dim, o.pack_size) + o.block * o.head_dim // 2)
        return max(1 << 16, blocks * 2 * o.batch * o.heads * per)

    @property
    def capacity(self) -> int:
        return int(self.arena.numel()) - 16

    def struct(self) -> N.Layer:
        if self._struct is None:
            o = self.owner
            s = N.Layer()
            s.batch, s.heads, s.head_dim, s.block = o.batch, o.heads, o.head_dim, o.block
            s.pack_size, s.buffer, s.max_blocks, s.reserved = o.pack_size, o.buffer, self.max_blocks, 0
            s.arena, s.arena_capacity = N.ptr(self.arena), self.capacity
            s.tail, s.blk_off, s.blk_len = N.ptr(self.tail), N.ptr(self.blk_off), N.ptr(self.blk_len)
            s.perm, s.nblk, s.nres = N.ptr(self.perm), N.ptr(self.nblk), N.ptr(self.nres)
            s.stage, s.err = N.ptr(self.stage), N.ptr(self.err)
            self._struct = s
        return self._struct

    @property
    def tokens(self) -> int:
        return self.nblk_h * self.owner.block + self.nres_h

    # -- growth -----------------------------------------------------------------
    def _grow_tables(self, need_blocks: int):
        o = self.owner
        new = max(need_blocks, 2 * self.max_blocks)
        U = o.batch * o.heads
        off = torch.full((2, U, new), -1, dtype=torch.int64, device=o.device)
        ln = torch.zeros((2, U, new), dtype=torch.int32, device=o.device)
        pm = torch.zeros((o.batch, new, o.block), dtype=torch.uint8, device=o.device)
        off[:, :, :self.max_blocks] = self.blk_off
        ln[:, :, :self.max_blocks] = self.blk_len
        pm[:, :self.max_blocks] = self.perm
        self.blk_off, self.blk_len, self.perm, self.max_blocks = off, ln, pm, new
        self._struct = None

    def _ensure(self, nsets: int):
        o = self.owner
        if self.nblk_h + nsets > self.max_blocks:
            self._grow_tables(self.nblk_h + nsets)
        need = nsets * 2 * o.batch * o.heads * self.blk_max
        if self.tail_ub + need > self.capacity:
            self.tail_ub = int(self.tail.item())         # synchronise only when it may not fit
            if self.tail_ub + need > self.capacity:
                newcap = max(2 * self.capacity, self.tail_ub + need + self._expected_bytes(nsets))
                arena = torch.empty(newcap + 16, dtype=torch.uint8, device=o.device)
                arena[:self.tail_ub] = self.arena[:self.tail_ub]
                self.arena = arena
                self._struct = None

    # -- append -----------------------------------------------------------------
    def compress(self, k_new: torch.Tensor, v_new: torch.Tensor, check: bool, perm: Optional[torch.Tensor] = None):
        """k_new/v_new: fp16 [B, T, H, D] on the device, contiguous.  perm
        ([B, nsets, block] uint8, optional): the repack plan of the block-sets
        this call completes, computed by the caller (sharded repacking); the
        store's own strategy is used otherwise."""
        o = self.owner
        T = int(k_new.shape[1])
        if self.ragged:
            raise ValueError("ragged batch (sequences of different lengths): append through GraphedDecodeLoop")
        lib = N.lib()
        strm = N.stream()
        if check and T:
            for x in (k_new, v_new):
                N.check(lib.pkv_check_finite(N.ptr(x), x.numel(), N.ptr(self.err), strm), "append")
            N.raise_flags(int(self.err.item()), "append")
        total = self.nres_h + T
        nsets = total // o.block
        if total - nsets * o.block > o.buffer:
            raise N.CapacityError("staging overflow")
        if T == 1 and nsets == 0:
            self.stage_token(k_new, v_new, check)
            return
        repack = N.REPACK[o.repack]
        if perm is not None and nsets:
            if tuple(perm.shape) != (o.batch, nsets, o.block) or perm.dtype != torch.uint8:
                raise E.ShapeMismatchError(f"perm must be uint8 [{o.batch}, {nsets}, {o.block}]")
            repack = N.REPACK_EXTERNAL
        if nsets:
            self._ensure(nsets)
            if repack == N.REPACK_EXTERNAL:
                self.perm[:, self.nblk_h:self.nblk_h + nsets].copy_(perm)
        L = self.struct()
        if nsets:
            per_set = int(lib.pkv_compress_scratch_bytes_ex(ctypes_ref(L), 1, repack))
            chunk = max(1, min(nsets, (256 << 20) // per_set))
            need = per_set * chunk
            if self.scratch.numel() < need:
                self.scratch = torch.empty(need, dtype=torch.uint8, device=o.device)
        N.check(lib.pkv_compress_tokens(ctypes_ref(L), N.ptr(k_new), N.ptr(v_new), T, self.nres_h, self.nblk_h,
                                        float(o.rel_scale_k), float(o.rel_scale_v), repack,
                                        N.ptr(self.scratch), int(self.scratch.numel()), strm), "compress")
        self.nblk_h += nsets
        self.nres_h = total - nsets * o.block
        self.tail_ub += nsets * 2 * o.batch * o.heads * self.blk_max
        if check:
            N.raise_flags(int(self.err.item()), "compress")

    def append_masked(self, k_new: torch.Tensor, v_new: torch.Tensor, counts, check: bool = False):
        """Ragged append: sequence b appends its first counts[b] tokens of
        k_new / v_new ([B, T, H, D] fp16), one masked step per token position
        (pkv_append_flush_masked: the token staged at the device residue count,
        a completed block compressed in the same launch)."""
        o = self.owner
        counts = np.asarray(counts, dtype=np.int64)
        lib = N.lib()
        if check:
            for x in (k_new, v_new):
                N.check(lib.pkv_check_finite(N.ptr(x), x.numel(), N.ptr(self.err), N.stream()), "append")
            N.raise_flags(int(self.err.item()), "append")
        nb0, nr0 = self.seq_counts()
        n = nr0 + counts
        self._ensure(int((n // o.block).max()) + 1)
        fb = int(lib.pkv_flush_scratch_bytes(ctypes_ref(self.struct())))
        if getattr(self, "flush_scr", None) is None or self.flush_scr.numel() < fb:
            self.flush_scr = torch.zeros(fb, dtype=torch.uint8, device=o.device)  # zero before first use
        active = torch.empty(o.batch, dtype=torch.uint8, device=o.device)
        for t in range(int(counts.max(initial=0))):
            active.copy_(torch.from_numpy((counts > t).astype(np.uint8)))
            kt, vt = k_new[:, t].contiguous(), v_new[:, t].contiguous()  # alive until the launch is enqueued
            N.check(lib.pkv_append_flush_masked(ctypes_ref(self.struct()), N.ptr(kt), N.ptr(vt), N.ptr(active),
                                                float(o.rel_scale_k), float(o.rel_scale_v), N.ptr(self.flush_scr),
                                                int(self.flush_scr.numel()), N.stream()), "append_masked")
        nblk, nres = nb0 + n // o.block, n % o.block
        self.tail_ub += int((n // o.block).sum()) * 2 * o.heads * self.blk_max
        self.nblk_h, self.nres_h = int(nblk.max()), int(nres.max())
        self.ragged = self.ragged or not (np.all(nblk == nblk[0]) and np.all(nres == nres[0]))
        if check:
            N.raise_flags(int(self.err.item()), "append_masked")

    def seq_counts(self):
        """Per-sequence (blocks, staged tokens) as int64 arrays [B]: the host
        mirrors for a lockstep batch, the device counts for a ragged one."""
        o = self.owner
        if not self.ragged:
            return np.full(o.batch, self.nblk_h, np.int64), np.full(o.batch, self.nres_h, np.int64)
        return self.nblk.cpu().numpy().astype(np.int64), self.nres.cpu().numpy().astype(np.int64)

    def pending_codes(self, k_new: torch.Tensor, v_new: torch.Tensor):
        """Quantized codes of the block-sets that appending k_new/v_new
        ([B, T, H, D] fp16, device) would complete, without appending:
        the u16 codes [nsets, B, 2, H, block, D] stored in an int16 tensor
        (pkv_compress_codes), or None."""
        o = self.owner
        T = int(k_new.shape[1])
        nsets = (self.nres_h + T) // o.block
        if nsets == 0:
            return None
        codes = torch.empty((nsets, o.batch, 2, o.heads, o.block, o.head_dim), dtype=torch.int16, device=o.device)
        params = torch.empty((nsets, o.batch, 2, o.heads, o.block, 2), dtype=torch.float32, device=o.device)
        N.check(N.lib().pkv_compress_codes(ctypes_ref(self.struct()), N.ptr(k_new), N.ptr(v_new), T, self.nres_h,
                                           float(o.rel_scale_k), float(o.rel_scale_v), N.ptr(codes), N.ptr(params),
                                           N.stream()), "pending_codes")
        return codes

    def stage_token(self, k_new: torch.Tensor, v_new: torch.Tensor, check: bool = False):
        """One token per sequence that does not complete a block: staged at the
        device residue count (pkv_stage_token), so the launch is identical
        every step and can live inside a CUDA graph (GraphedDecodeStep)."""
        o = self.owner
        if self.ragged:
            raise ValueError("ragged batch (sequences of different lengths): append through GraphedDecodeLoop")
        if self.nres_h + 1 >= o.block:
            raise ValueError("this token completes a block: use compress()")
        N.check(N.lib().pkv_stage_token(ctypes_ref(self.struct()), N.ptr(k_new), N.ptr(v_new), N.stream()),
                "stage_token")
        self.nres_h += 1
        if check:
            N.raise_flags(int(self.err.item()), "stage_token")

    def width_hist(self, kind: int) -> List[int]:
        """Pack-width histogram (0..15) over the layer's blocks of one kind, read
        from the width nibbles of the blocks in HBM (Fig. 3 analog)."""
        o = self.owner
        nb = self.nblk_h
        if nb == 0:
            return [0] * 16
        P = (o.block // o.pack_size) * o.head_dim
        offs = self.blk_off[kind, :, :nb].reshape(-1)
        idx = offs[:, None] + 8 + torch.arange((P + 1) // 2, device=offs.device)[None, :]
        nib = self.arena[idx.reshape(-1)].to(torch.int64)
        w = torch.stack([nib & 15, nib >> 4], 1).reshape(offs.numel(), -1)[:, :P]
        return [int(x) for x in torch.bincount(w.reshape(-1), minlength=16).cpu().tolist()]

    def shrink_to_fit(self, headroom_bytes: int = 0):
        """Reallocate the arena to its used bytes (+ headroom): geometric growth
        leaves up to ~2x reserved; the next append grows it again if needed."""
        used = int(self.tail.item())
        cap = _round16(used + max(0, int(headroom_bytes)))
        if cap + 16 < self.arena.numel():
            arena = torch.empty(cap + 16, dtype=torch.uint8, device=self.arena.device)
            arena[:used].copy_(self.arena[:used])
            self.arena = arena
            self._struct = None
        self.tail_ub = used

    # -- introspection (synchronising; parity / debug) ----------------------------
    def tables(self):
        o = self.owner
        U = o.batch * o.heads
        nb = self.nblk_h
        off = self.blk_off[:, :, :nb].cpu().numpy()
        ln = self.blk_len[:, :, :nb].cpu().numpy()
        pm = self.perm[:, :nb].cpu().numpy()
        return off, ln, pm

    def directory(self) -> List[BlockDirectoryEntry]:
        """Directory entries in arena order (block-set, sequence, K heads, V heads)."""
        o = self.owner
        off, ln, pm = self.tables()
        ents = []
        for j in range(self.nblk_h):
            for b in range(o.batch):
                for kind in (KIND_K, KIND_V):
                    for h in range(o.heads):
                        u = b * o.heads + h
                        if off[kind, u, j] < 0:  # a ragged batch: sequence b has no block j yet
                            continue
                        ents.append(BlockDirectoryEntry(kind, self.layer, h, j * o.block, (j + 1) * o.block,
                                                        int(off[kind, u, j]), int(ln[kind, u, j]),
                                                        pm[b, j].astype(np.int64), b))
        return ents

    def block_bytes(self, e: BlockDirectoryEntry) -> bytes:
        return bytes(self.arena[e.byte_offset:e.byte_offset + e.byte_len].cpu().numpy().tobytes())

    def stream_bytes(self, seq: Optional[int] = 0) -> bytes:
        """Blocks concatenated in directory order without alignment padding
        (for one sequence this is byte-identical to the reference arena)."""
        arena = self.arena[:max(1, int(self.tail.item()))].cpu().numpy()
        out = bytearray()
        for e in self.directory():
            if seq is None or e.seq == seq:
                out += arena[e.byte_offset:e.byte_offset + e.byte_len].tobytes()
        return bytes(out)


def ctypes_ref(s):
    import ctypes
    return ctypes.byref(s)


class CompressedStore:
    """SPEC.md:357-362.  Device-resident, batched, one sub-store per layer."""

    def __init__(self, layers: int, heads: int, head_dim: int, batch: int = 1, rel_scale_k: float = 0.1,
                 rel_scale_v: float = 0.2, pack_size: int = 16, repack: str = "none", block: int = 64,
                 buffer: int = 128, device=None, max_tokens: Optional[int] = None, check: bool = True):
        if repack not in REPACK_STRATEGIES:
            raise ValueError(f"repack must be one of {REPACK_STRATEGIES}")
        if pack_size not in (2, 4, 8, 16, 32):
            raise ValueError("pack_size must be one of 2, 4, 8, 16, 32")
        if block % pack_size or block > 256:
            raise ValueError("block must be a multiple of pack_size and <= 256")
        if repack != "none" and block > 64:
            raise ValueError("repacking needs block <= 64")
        if not (0 < rel_scale_k <= 1 and 0 < rel_scale_v <= 1):
            raise ValueError("relative scales must be in (0, 1]")
        if buffer < block:
            raise ValueError("buffer must hold at least one block")
        N.lib()  # fail loudly without the CUDA library / device
        self.layers, self.heads, self.head_dim, self.batch = layers, heads, head_dim, batch
        self.rel_scale_k, self.rel_scale_v = float(rel_scale_k), float(rel_scale_v)
        self.pack_size, self.repack, self.block, self.buffer = pack_size, repack, block, buffer
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.check = check
        init_blocks = max(4, math.ceil((max_tokens or 4096) / block))
        self.layer_stores = [LayerStore(self, l, init_blocks) for l in range(layers)]

    def __getitem__(self, layer: int) -> LayerStore:
        if not (0 <= layer < self.layers):
            raise IndexError(f"layer {layer} out of range [0, {self.layers})")
        return self.layer_stores[layer]

    def total_tokens(self, layer: int) -> int:
        return self[layer].tokens

    # normalisation of inputs to [B, T, H, D] fp16 on the device
    def _norm(self, x, tokens_axis: bool) -> torch.Tensor:
        if not isinstance(x, torch.Tensor):
            x = torch.as_tensor(np.asarray(x))
        H, D, B = self.heads, self.head_dim, self.batch
        shape = tuple(x.shape)
        if tokens_axis:
            if x.dim() == 3 and B == 1 and shape[1:] == (H, D):
                x = x.unsqueeze(0)
            elif x.dim() == 2 and B == 1 and shape[1] == H * D:
                x = x.reshape(1, shape[0], H, D)
            if x.dim() != 4 or tuple(x.shape[:1]) != (B,) or tuple(x.shape[2:]) != (H, D):
                raise E.ShapeMismatchError(f"expected [B={B}, T, H={H}, D={D}] tokens, got {shape}")
        else:
            if x.numel() != B * H * D:
                raise E.ShapeMismatchError(f"expected {B}x{H}x{D} values per token, got {shape}")
            x = x.reshape(B, 1, H, D)
        if x.dtype != torch.float16:
            x = x.to(torch.float16)
        return x.to(self.device).contiguous()

    def append_token(self, layer: int, k_vec, v_vec):
        """SPEC.md:365-373."""
        ls = self[layer]
        k = self._norm(k_vec, False)
        v = self._norm(v_vec, False)
        ls.compress(k, v, self.check)

    def compress_batch(self, layer: int, k_tokens, v_tokens, lengths=None):
        """identical final state to appending token by token.

        lengths (optional, [B]): a ragged prefill -- sequence b takes its first
        lengths[b] tokens of k_tokens / v_tokens ([B, T, H, D], T >= max).  The
        common prefix is compressed in lockstep, the rest appended one step at a
        time for the sequences that still have tokens (pkv_append_flush_masked,
        default format, repack none); the store is then ragged (see
        GraphedDecodeLoop)."""
        ls = self[layer]
        k = self._norm(k_tokens, True)
        v = self._norm(v_tokens, True)
        if k.shape != v.shape:
            raise E.ShapeMismatchError("K and V batches differ in shape")
        if lengths is None:
            ls.compress(k, v, self.check)
            return
        lens = np.asarray(lengths, dtype=np.int64).reshape(-1)
        if lens.shape != (self.batch,) or (lens < 0).any() or lens.max(initial=0) > k.shape[1]:
            raise E.ShapeMismatchError(f"lengths must be {self.batch} counts <= {k.shape[1]}")
        common = int(lens.min())
        ls.compress(k[:, :common].contiguous(), v[:, :common].contiguous(), self.check)
        if common == int(lens.max()):
            return
        if self.repack != "none" or self.pack_size != 16 or self.head_dim != 128 or self.block != 64:
            raise ValueError("ragged prefill: default format with repack none only")
        ls.append_masked(k[:, common:], v[:, common:], lens - common, self.check)

    def iterate_blocks(self, layer: int, kind: int, seq: int = 0):
        """directory entries of (layer, kind) then the residue handle."""
        ls = self[layer]
        ents = [e for e in ls.directory() if e.kind == kind and e.seq == seq]
        nb, nr = ls.seq_counts()
        return ents + [ResidueHandle(layer, int(nb[seq]) * self.block, int(nr[seq]), seq)]

    def shrink_to_fit(self, headroom_bytes: int = 0):
        """Release the arena capacity reserved beyond the compressed bytes (every layer)."""
        for ls in self.layer_stores:
            ls.shrink_to_fit(headroom_bytes)

    def check_errors(self):
        for ls in self.layer_stores:
            flags = int(ls.err.item())
            if flags:
                ls.err.zero_()
                N.raise_flags(flags, f"layer {ls.layer}")

    def snapshot_stats(self, include_staging: bool = False):
        """exact byte counts and CR per (layer, kind)."""
        out = {}
        for ls in self.layer_stores:
            _, ln, _ = ls.tables()
            for kind in (KIND_K, KIND_V):
                phys = int(ln[kind].astype(np.int64).sum())
                nblocks = int(ln[kind].size)
                logical = nblocks * self.block * self.head_dim * 2
                res = ls.nres_h * self.batch * self.heads * self.head_dim * 2 if include_staging else 0
                widths = ls.width_hist(kind) if nblocks else [0] * 16
                out[(ls.layer, kind)] = {
                    "blocks": nblocks, "bytes_physical": phys + res, "bytes_logical": logical + res,
                    "cr": (logical + res) / (phys + res) if phys + res else None, "width_hist": widths,
                }
        return out


def append_token(store: CompressedStore, layer: int, k_vec, v_vec):
    store.append_token(layer, k_vec, v_vec)


def compress_batch(store: CompressedStore, layer: int, k_tokens, v_tokens):
    store.compress_batch(layer, k_tokens, v_tokens)


def iterate_blocks(store: CompressedStore, layer: int, kind: int, seq: int = 0):
    return store.iterate_blocks(layer, kind, seq)


def snapshot_stats(store: CompressedStore, include_staging: bool = False):
    return store.snapshot_stats(include_staging)


# ----------------------------------------------------------------------------
# "PKKS" store file (header + arena bytes + directory records;
# field layout in DESIGN.md §3.1).  Little-endian:
#   header  "PKKS" | version u16 = 1 | layers u16 | batch u16 | heads u16 |
#           head_dim u16 | block u16 | pack_size u16 | buffer u16 | repack u8 |
#           3 x 0 | rel_k f32 | rel_v f32                             (32 B)
#   per layer:
#           nblk u32 (block-sets per sequence) | nres u32 | arena_len u64
#           arena bytes (blocks at 16-byte aligned offsets, zero padding)
#           records (offset u64, len u32), arena order (block-set, sequence,
#             kind, head)
#           permutations u8 [batch][nblk][block]
#           staging f16 [batch][kind][head][nres][head_dim]
# Writing a store and loading it back is a bit-exact round trip; the file of
# a single-sequence store equals the oracle's (oracle/packkv_oracle.save_pkks).
# ----------------------------------------------------------------------------
import struct as _struct

_PKKS_HDR = _struct.Struct("<4sHHHHHHHHB3xff")
_PKKS_LAYER = _struct.Struct("<IIQ")
_PKKS_REC = np.dtype([("off", "<u8"), ("len", "<u4")])


def save_store(store: CompressedStore, path) -> None:
    """Serialize every layer (synchronises the device).  The PKKS format holds
    one (blocks, residue) count per layer: a ragged batch cannot be saved."""
    o = store
    if any(ls.ragged for ls in o.layer_stores):
        raise E.StoreFormatError("ragged batch: PKKS stores one block / residue count per layer")
    with open(path, "wb") as f:
        f.write(_PKKS_HDR.pack(b"PKKS", 1, o.layers, o.batch, o.heads, o.head_dim, o.block, o.pack_size, o.buffer,
                               N.REPACK[o.repack], o.rel_scale_k, o.rel_scale_v))
        U = o.batch * o.heads
        for ls in o.layer_stores:
            nb, nr = ls.nblk_h, ls.nres_h
            tail = int(ls.tail.item())
            f.write(_PKKS_LAYER.pack(nb, nr, tail))
            f.write(ls.arena[:tail].cpu().numpy().tobytes())
            off, ln, pm = ls.tables()                               # [2, U, nb], [B, nb, block]
            rec = np.empty((nb, o.batch, 2, o.heads), _PKKS_REC)
            rec["off"] = off.reshape(2, o.batch, o.heads, nb).transpose(3, 1, 0, 2)
            rec["len"] = ln.reshape(2, o.batch, o.heads, nb).transpose(3, 1, 0, 2)
            f.write(rec.tobytes())
            f.write(np.ascontiguousarray(pm).tobytes())
            stage = ls.stage[:, :, :nr].reshape(2, o.batch, o.heads, nr, o.head_dim).permute(1, 0, 2, 3, 4)
            f.write(stage.contiguous().cpu().numpy().astype("<f2").tobytes())
            assert U == o.batch * o.heads


def load_store(path, device=None, check: bool = True) -> CompressedStore:
    """Inverse of save_store: a device-resident store in the saved state.
    StoreFormatError on a malformed file."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < _PKKS_HDR.size or data[:4] != b"PKKS":
        raise E.StoreFormatError(f"{path}: not a PKKS store file")
    (_, ver, layers, batch, heads, head_dim, block, k, buffer, rep, rel_k, rel_v) = _PKKS_HDR.unpack_from(data)
    if ver != 1:
        raise E.StoreFormatError(f"{path}: unsupported version {ver}")
    names = {v: s for s, v in N.REPACK.items()}
    if rep not in names:
        raise E.StoreFormatError(f"{path}: bad repack code {rep}")
    try:
        st = CompressedStore(layers, heads, head_dim, batch=batch, rel_scale_k=rel_k, rel_scale_v=rel_v,
                             pack_size=k, repack=names[rep], block=block, buffer=buffer, device=device, check=check)
    except ValueError as e:
        raise E.StoreFormatError(f"{path}: {e}") from e
    hb = header_bytes(block, head_dim, k)
    pos = _PKKS_HDR.size

    def take(n):
        nonlocal pos
        if pos + n > len(data):
            raise E.StoreFormatError(f"{path}: truncated")
        b = data[pos:pos + n]
        pos += n
        return b

    for ls in st.layer_stores:
        nb, nr, alen = _PKKS_LAYER.unpack(take(_PKKS_LAYER.size))
        if nr > buffer or nr >= block:
            raise E.StoreFormatError(f"{path}: residue {nr} out of range")
        arena = np.frombuffer(take(alen), np.uint8)
        rec = np.frombuffer(take(nb * batch * 2 * heads * _PKKS_REC.itemsize), _PKKS_REC)
        pm = np.frombuffer(take(batch * nb * block), np.uint8).reshape(batch, nb, block)
        stage = np.frombuffer(take(batch * 2 * heads * nr * head_dim * 2), "<f2")
        offs, lens = rec["off"].astype(np.int64), rec["len"].astype(np.int64)
        if ((offs % 16) != 0).any() or (offs + lens > alen).any() or (lens < hb).any():
            raise E.StoreFormatError(f"{path}: bad directory record")
        if len(offs):
            # records may not overlap (the arena is append-only)
            order = np.argsort(offs, kind="stable")
            if (offs[order][:-1] + lens[order][:-1] > offs[order][1:]).any():
                raise E.StoreFormatError(f"{path}: overlapping directory records")
            # every record's length must equal its header plus the payload bytes its
            # width nibbles promise (the fused kernels locate payloads from the
            # nibbles alone, MalformedBlockError in decode_block)
            P = (block // k) * head_dim
            nib = arena[offs[:, None] + 8 + np.arange((P + 1) // 2)[None, :]]
            wid = np.stack([nib & 15, nib >> 4], axis=-1).reshape(len(offs), -1)[:, :P].astype(np.int64)
            expect = hb + ((k * wid + 7) // 8).sum(axis=1)
            if (expect != lens).any():
                i = int(np.nonzero(expect != lens)[0][0])
                raise E.StoreFormatError(f"{path}: block {i} length {int(lens[i])} disagrees with its widths "
                                         f"({int(expect[i])} bytes)")
        for i in range(len(offs)):                  # header geometry of every block
            o0 = int(offs[i])
            kind = (i // heads) % 2
            if (arena[o0] != kind or arena[o0 + 2] != k or int(arena[o0 + 4]) | int(arena[o0 + 5]) << 8 != block
                    or int(arena[o0 + 6]) | int(arena[o0 + 7]) << 8 != head_dim):
                raise E.StoreFormatError(f"{path}: block {i} header disagrees with the store geometry")
        if nb > ls.max_blocks:
            ls._grow_tables(nb)
        if alen + 16 > ls.arena.numel():
            ls.arena = torch.empty(alen + 16, dtype=torch.uint8, device=st.device)
        ls.arena[:alen].copy_(torch.from_numpy(arena.copy()))
        ls.tail.fill_(alen)
        o4 = torch.from_numpy(offs.reshape(nb, batch, 2, heads).transpose(2, 1, 3, 0).reshape(2, batch * heads, nb).copy())
        l4 = torch.from_numpy(lens.reshape(nb, batch, 2, heads).transpose(2, 1, 3, 0).reshape(2, batch * heads, nb)
                              .astype(np.int32).copy())
        ls.blk_off[:, :, :nb].copy_(o4)
        ls.blk_len[:, :, :nb].copy_(l4)
        ls.perm[:, :nb].copy_(torch.from_numpy(pm.copy()))
        ls.nblk.fill_(nb)
        ls.nres.fill_(nr)
        if nr:
            sv = torch.from_numpy(stage.astype(np.float16).reshape(batch, 2, heads, nr, head_dim).copy())
            ls.stage[:, :, :nr].copy_(sv.permute(1, 0, 2, 3, 4).reshape(2, batch * heads, nr, head_dim))
        ls.nblk_h, ls.nres_h, ls.tail_ub = nb, nr, alen
        ls._struct = None
    if pos != len(data):
        raise E.StoreFormatError(f"{path}: {len(data) - pos} trailing bytes")
    return st
