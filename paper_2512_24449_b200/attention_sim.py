"""Decode-step attention over the compressed store.

attention_decode composes fused_k_scores -> 1/sqrt(d) -> stable softmax ->
fused_v_output; scores stay in block/permuted order, which
single-query attention is invariant to (proof box).
"""
from __future__ import annotations

import math

import torch

from . import _native as N
from . import errors as E
from .fused_kernels import fused_k_scores_batched, fused_v_output_batched, _as_f32
from .kv_store import CompressedStore, ctypes_ref


def attention_decode_batched(store: CompressedStore, layer: int, q, score_stride: int = 0, scores=None,
                             out=None, nblocks: int = None, single_pass: bool = None,
                             prescaled: bool = False) -> torch.Tensor:
    """q [B, Hq, D] -> out [B, Hq, D].

    The 1/sqrt(d) scale is applied to the (small) query instead of the
    [B, Hq, L] scores (scores are linear in q).  For the default
    format the softmax is folded into the fused kernels (pkv_attention_decode:
    the K launch records per-slot score maxima, the V launch weights rows with
    exp(s - max) and the finalize divides by the sum), so the scores are
    written once and read once; other formats compose fused K -> softmax ->
    fused V.  score_stride (>= the token count) sizes the
    internal score rows; GraphedAttention passes room for the whole staging
    ring so one capture serves every residue length.  scores / out may be
    preallocated (graph capture without allocations).  nblocks (default: the
    layer's block count) sizes the fused launches; a larger value leaves
    headroom for blocks appended on the device later (GraphedDecodeLoop):
    blocks past a sequence's device count are skipped.

    single_pass: True runs the single pass (attn_fused_kernel: K, online
    softmax and V block by block, then a deterministic merge of the per-warp
    partials; no score row reaches HBM); False the three-launch path, which
    also fills `scores`.  Default (None): the single pass when `scores` is not
    requested and the layer is latency-bound (at most 4 items per resident warp,
    single_pass_preferred), where it measured faster (config C: 622 vs 482
    tokens/s); the three-launch path at long contexts, where its two
    kernels issue faster (config B 131 vs 140 us)."""
    q = _as_f32(q, store.device)
    if not prescaled:  # prescaled: the caller already multiplied q by 1/sqrt(d)
        q = q * (1.0 / math.sqrt(store.head_dim))
    ls = store[layer]
    B, H, D = store.batch, store.heads, store.head_dim
    if q.dim() != 3 or q.shape[0] != B or q.shape[2] != D or q.shape[1] % H:
        raise E.ShapeMismatchError(f"q must be [B={B}, Hq (multiple of {H}), D={D}], got {tuple(q.shape)}")
    Hq = int(q.shape[1])
    lib = N.lib()
    st = ls.struct()
    nb = ls.nblk_h if nblocks is None else int(nblocks)
    need = int(lib.pkv_attention_scratch_bytes(ctypes_ref(st), nb, Hq))
    if single_pass is None:
        single_pass = scores is None and single_pass_preferred(store, nb)
    if need > 0 and single_pass:
        if out is None:
            out = torch.empty((B, Hq, D), dtype=torch.float32, device=store.device)
        if ls.a_scratch.numel() < need:
            ls.a_scratch = torch.zeros(need, dtype=torch.uint8, device=store.device)  # work counter: zero before first use
        N.check(lib.pkv_attention_decode(ctypes_ref(st), nb, N.ptr(q), Hq, None, 0, N.ptr(out),
                                         N.ptr(ls.a_scratch), int(ls.a_scratch.numel()), N.stream()),
                "attention_decode")
        return out
    if need > 0:
        stride = max(ls.tokens, nb * store.block + ls.nres_h, score_stride, 1)
        stride = (stride + 3) // 4 * 4
        if scores is None or scores.shape[-1] < stride:
            scores = torch.empty((B, Hq, stride), dtype=torch.float32, device=store.device)
        stride = int(scores.shape[-1])
        if out is None:
            out = torch.empty((B, Hq, D), dtype=torch.float32, device=store.device)
        if ls.a_scratch.numel() < need:
            ls.a_scratch = torch.zeros(need, dtype=torch.uint8, device=store.device)  # work counter: zero before first use
        N.check(lib.pkv_attention_decode(ctypes_ref(st), nb, N.ptr(q), Hq, N.ptr(scores), stride, N.ptr(out),
                                         N.ptr(ls.a_scratch), int(ls.a_scratch.numel()), N.stream()),
                "attention_decode")
        return out
    s = fused_k_scores_batched(store, layer, q)
    a = torch.softmax(s, dim=-1)
    return fused_v_output_batched(store, layer, a, out=out)


# resident warps of the fused kernels on a B200 (148 SMs x 16) and the
# blocks-per-warp crossover below which the single pass is the faster path
_RESIDENT_WARPS = 148 * 16
SINGLE_PASS_MAX_ITEMS_PER_WARP = 4  # config B shape: parity at 3.6 items per warp (8K tokens), three launches 10% faster at 7.1 (16K)


def single_pass_preferred(store: CompressedStore, nblocks: int) -> bool:
    """True when one decode-attention launch is latency-bound: the layer's
    (unit, block + residue chunk) items are at most
    SINGLE_PASS_MAX_ITEMS_PER_WARP per resident warp."""
    items = store.batch * store.heads * (int(nblocks) + (store.buffer + 31) // 32)
    return items <= SINGLE_PASS_MAX_ITEMS_PER_WARP * _RESIDENT_WARPS


def ptr_of(t):
    return 0 if t is None else t.data_ptr()


class _Captured:
    """Shared machinery: static input/output buffers allocated OUTSIDE the
    capture (so capturing allocates nothing), a capture key over the state the
    recorded launches bake in (block count, device buffers, shapes)."""

    def __init__(self, store: CompressedStore, layer: int):
        self.store, self.layer = store, layer
        self._key = None
        self._graph = None
        self._scores = None
        self._out = None
        self.captures = 0

    def _state(self, q: torch.Tensor):
        ls = self.store[self.layer]
        # every device buffer the recorded launches read or write: a re-allocated
        # scratch / score / output buffer must force a re-capture, not a replay
        # against freed memory
        return (ls.nblk_h, ls.arena.data_ptr(), ls.blk_off.data_ptr(), ls.stage.data_ptr(), tuple(q.shape),
                q.device, ls.a_scratch.data_ptr(), ptr_of(self._scores), ptr_of(self._out))

    def _buffers(self, q: torch.Tensor):
        st = self.store
        # room for every residue length of the current block count
        stride = (st[self.layer].nblk_h * st.block + st.buffer + 3) // 4 * 4
        B, Hq, D = q.shape
        if self._scores is None or self._scores.shape != (B, Hq, stride):
            self._scores = torch.empty((B, Hq, stride), dtype=torch.float32, device=q.device)
        if self._out is None or self._out.shape != (B, Hq, D):
            self._out = torch.empty((B, Hq, D), dtype=torch.float32, device=q.device)

    single_pass = None  # None: single_pass_preferred; True / False force a path

    def _attend(self, q: torch.Tensor, prescaled: bool = False, out: torch.Tensor = None) -> torch.Tensor:
        sp = self.single_pass
        if sp is None:
            sp = single_pass_preferred(self.store, self.store[self.layer].nblk_h)
        return attention_decode_batched(self.store, self.layer, q, scores=self._scores,
                                        out=self._out if out is None else out, single_pass=sp, prescaled=prescaled)

    def _graphable(self, q: torch.Tensor) -> bool:
        """Only the default format's folded-softmax launches (pkv_attention_decode)
        read the residue length from the device; the generic composition (fused
        K -> softmax -> fused V) bakes the host token count into its shapes, so it
        runs eagerly."""
        ls = self.store[self.layer]
        if q.dim() != 3:
            return False
        return int(N.lib().pkv_attention_scratch_bytes(ctypes_ref(ls.struct()), ls.nblk_h, int(q.shape[1]))) > 0

    def _capture(self, record):
        """record() enqueues the step's launches; warmed up eagerly by the caller.
        Captures with CUDAGraph.capture_begin/end on a side stream rather than the
        torch.cuda.graph context manager, which also runs gc.collect() and
        empty_cache() (milliseconds) at every re-capture; the launches allocate
        nothing, and one memory pool is shared by all captures of this object."""
        dev = torch.device(self.store.device)
        if getattr(self, "_pool", None) is None:
            self._pool = torch.cuda.graph_pool_handle()
            self._side = torch.cuda.Stream(device=dev)
        cur = torch.cuda.current_stream(dev)
        self._side.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self._side):
            g.capture_begin(pool=self._pool)
            try:
                record()
            finally:
                g.capture_end()
        cur.wait_stream(self._side)
        self._graph = g
        self.captures += 1


class GraphedAttention(_Captured):
    """attention_decode_batched for one layer, captured into a CUDA graph and
    replayed: a decode step is then one graph launch (fused K, softmax, fused V
    + finalize) instead of a dozen host-driven launches.  The kernels read
    the residue length from the device (pkv_layer_t.nres), so appends that
    only stage a token replay the same graph; it is re-captured when the
    block count or the device buffers change (every 64 appended tokens, or
    when the store grows)."""

    supports_host_out = True

    def __call__(self, q: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
        """q [B, Hq, D] on the device, or pinned host f32: then the graph reads it from host
        memory itself (zero-copy over PCIe, with the 1/sqrt(d) prescale, pkv_copy_scaled)
        instead of a copy-engine transfer before the replay.  out (optional, pinned host f32
        [B, Hq, D], with a host q) receives the output inside the same graph: the attention's
        last kernel stores it to host memory directly.  The host
        buffers' addresses are part of the capture: reuse the same ones every step (static
        I/O buffers), new ones re-capture."""
        if isinstance(q, torch.Tensor) and not q.is_cuda and q.dtype == torch.float32 and q.is_pinned() \
                and q.is_contiguous() and q.dim() == 3:
            return self._host_call(q, out)
        if out is not None:
            raise E.ShapeMismatchError("out= (host output) needs a pinned host f32 q")
        q = _as_f32(q, self.store.device)
        key = self._state(q)
        if key != self._key and not self._graphable(q):
            return attention_decode_batched(self.store, self.layer, q)
        if key != self._key:
            self._q = q.clone()
            self._buffers(q)
            self._attend(self._q)  # warm-up outside capture (scratch, occupancy queries)
            self._capture(lambda: self._attend(self._q))
            self._key = self._state(q)  # after _buffers: the captured buffers' addresses
        self._q.copy_(q, non_blocking=True)
        self._graph.replay()
        return self._out

    def _host_call(self, qh: torch.Tensor, oh: torch.Tensor = None) -> torch.Tensor:
        if oh is not None and not (not oh.is_cuda and oh.is_pinned() and oh.dtype == torch.float32
                                   and oh.is_contiguous() and tuple(oh.shape) == tuple(qh.shape)):
            raise E.ShapeMismatchError(f"out must be a pinned host f32 tensor of shape {tuple(qh.shape)}")
        hkey = ("host", qh.data_ptr(), oh.data_ptr() if oh is not None else 0)
        if self._key is None or self._key[-1] != hkey or self._key[:-1] != self._state(self._q):
            qd = qh.to(self.store.device)
            if not self._graphable(qd):  # generic format: eager, copies through the copy engine
                o = attention_decode_batched(self.store, self.layer, qd)
                if oh is not None:
                    oh.copy_(o)
                    return oh
                return o
            self._q = torch.empty_like(qd)
            self._buffers(qd)
            lib, n = N.lib(), qh.numel()
            inv = 1.0 / math.sqrt(self.store.head_dim)

            def record():
                N.check(lib.pkv_copy_scaled(qh.data_ptr(), self._q.data_ptr(), n, inv, N.stream()))
                # the last kernel (finalize / merge) stores the output straight to the pinned
                # host buffer (UVA): no device-side output round trip, no copy launch
                self._attend(self._q, prescaled=True, out=oh)

            record()  # warm-up outside capture
            self._capture(record)
            self._key = self._state(self._q) + (hkey,)
        self._graph.replay()
        return oh if oh is not None else self._out


class GraphedDecodeStep(_Captured):
    """One serving decode step for one layer -- append this step's K/V token
     then attend with q over everything including it
     -- as ONE CUDA-graph replay: the staging copy
    (pkv_stage_token, positioned by the device residue count) and the fused
    attention launches.  The token that completes a 64-token block runs
    eagerly (compressor: quantize + encode + arena append, then attention)
    and the next step re-captures (the block count changed)."""

    def __call__(self, k_tok, v_tok, q: torch.Tensor) -> torch.Tensor:
        st, ls = self.store, self.store[self.layer]
        q = _as_f32(q, st.device)
        if self._key is None or self._key[0] != ls.nblk_h:
            if not self._graphable(q):  # generic formats: eager append + composition
                st.append_token(self.layer, k_tok, v_tok)
                return attention_decode_batched(st, self.layer, q)
        if ls.nres_h + 1 >= st.block:  # block completes: eager compress + attention
            st.append_token(self.layer, k_tok, v_tok)
            self._buffers(q)
            return self._attend(q)
        k = st._norm(k_tok, False)
        v = st._norm(v_tok, False)
        if st.check:  # non-finite input raises at append time
            for x in (k, v):
                N.check(N.lib().pkv_check_finite(N.ptr(x), x.numel(), N.ptr(ls.err), N.stream()), "append")
            N.raise_flags(int(ls.err.item()), "append")
        key = self._state(q)
        if key != self._key:
            if getattr(self, "_k", None) is None or self._k.shape != k.shape or self._q.shape != q.shape:
                self._k, self._v, self._q = k.clone(), v.clone(), q.clone()
            self._buffers(q)
            self._attend(self._q)  # warm-up outside capture (scratch, occupancy queries); appends nothing

            def record():
                N.check(N.lib().pkv_stage_token(ctypes_ref(ls.struct()), N.ptr(self._k), N.ptr(self._v),
                                                N.stream()), "stage_token")
                self._attend(self._q)
            self._capture(record)
            self._key = self._state(q)  # after _buffers: the captured buffers' addresses
        for dst, src in ((self._k, k), (self._v, v), (self._q, q)):
            if dst.data_ptr() != src.data_ptr():  # callers may write the inputs() in place
                dst.copy_(src, non_blocking=True)
        self._graph.replay()
        ls.nres_h += 1
        return self._out

    def inputs(self, q_heads: int):
        """Static device buffers (k [B, 1, H, D] f16, v, q [B, Hq, D] f32) the
        graph reads: a caller that writes the step's token and query into
        them and passes them back skips the three input copies."""
        st = self.store
        B, H, D = st.batch, st.heads, st.head_dim
        if getattr(self, "_k", None) is None or self._q.shape != (B, q_heads, D):
            self._k = torch.zeros((B, 1, H, D), dtype=torch.float16, device=st.device)
            self._v = torch.zeros_like(self._k)
            self._q = torch.zeros((B, q_heads, D), dtype=torch.float32, device=st.device)
            self._key = None
        return self._k, self._v, self._q


class GraphedDecodeLoop:
    """The serving decode loop over one or more layers as ONE CUDA-graph replay
    per step.  For every layer the graph holds: the step's K/V token staged at
    the device residue count (pkv_stage_token), a block completed on the device
    (pkv_flush_staged: quantize, encode and append the staged block-set at the
    device block count and arena tail when nres reaches 64), and attention
    over everything including the new token (pkv_attention_decode sized for
    `headroom` more blocks; blocks past a sequence's device count are skipped).
    No launch reads a host-side position, so the same graph replays across
    block completions (SPEC.md:365-373 append_token
    attention_decode).  It is re-captured only when the headroom is used up
    (every headroom * 64 tokens) or a buffer moves.  Default format, repack
    "none" (GraphedDecodeStep serves the others).

    Default (fused_append): the token is staged and a completed block
    compressed in ONE launch per layer (pkv_append_flush) instead of two
    (pkv_stage_token, pkv_flush_staged); fused_append = False keeps them
    separate.

    step(k, v, q): k / v [layers, B, 1, H, D] (or [layers, B, H, D]) fp16,
    q [layers, B, Hq, D] f32 -> out [layers, B, Hq, D] (a static buffer,
    overwritten by the next step).  inputs() returns the static input buffers;
    a caller that writes them in place and calls step() without arguments
    skips the copies."""

    single_pass = None  # None: single_pass_preferred; True / False force a path
    fused_append = True

    def __init__(self, store: CompressedStore, q_heads: int, layers=None, headroom: int = 16):
        self.store = store
        self.layers = list(range(store.layers)) if layers is None else list(layers)
        self.headroom = max(1, int(headroom))
        B, H, D = store.batch, store.heads, store.head_dim
        if q_heads % H:
            raise E.ShapeMismatchError(f"q_heads must be a multiple of kv heads ({H})")
        if store.repack != "none" or store.pack_size != 16 or store.head_dim != 128 or store.block != 64:
            raise ValueError("GraphedDecodeLoop: default format with repack none only (use GraphedDecodeStep)")
        n, dev = len(self.layers), store.device
        self.k = torch.zeros((n, B, 1, H, D), dtype=torch.float16, device=dev)
        self.v = torch.zeros_like(self.k)
        self.q = torch.zeros((n, B, q_heads, D), dtype=torch.float32, device=dev)
        self.out = torch.empty((n, B, q_heads, D), dtype=torch.float32, device=dev)
        # ragged decode: active[b] = 1 appends sequence b's token this step
        self.active = torch.ones(B, dtype=torch.uint8, device=dev)
        self._active_all = True
        counts = [store[l].seq_counts() for l in self.layers]
        self._seq_nblk = [c[0] for c in counts]
        self._seq_nres = [c[1] for c in counts]
        self._flush_scr = [None] * n
        self._scores = [None] * n
        self._cap = [0] * n
        self._graph = None
        self._key = None
        self._pool = None
        self._hout = None  # pinned host output buffer the graph writes, or None (self.out)
        self.captures = 0

    def inputs(self):
        return self.k, self.v, self.q

    def _state(self):
        st = []
        for l in self.layers:
            ls = self.store[l]
            st.append((ls.arena.data_ptr(), ls.blk_off.data_ptr(), ls.stage.data_ptr(), ls.a_scratch.data_ptr(),
                       ls.max_blocks))
        st.append(ptr_of(self._hout))
        return tuple(st)

    def _prepare(self):
        """Host side of a (re)capture: tables, arena and scratch for `headroom`
        more block-sets per layer, allocated before the capture."""
        o = self.store
        B, Hq = o.batch, self.q.shape[2]
        lib = N.lib()
        for i, l in enumerate(self.layers):
            ls = o[l]
            ls._ensure(self.headroom)
            self._cap[i] = ls.nblk_h + self.headroom
            if ls.max_blocks < self._cap[i]:
                ls._grow_tables(self._cap[i])
            L = ls.struct()
            fb = int(lib.pkv_flush_scratch_bytes(ctypes_ref(L)))
            if self._flush_scr[i] is None or self._flush_scr[i].numel() < fb:
                self._flush_scr[i] = torch.zeros(fb, dtype=torch.uint8, device=o.device)  # zero before first use
            need = int(lib.pkv_attention_scratch_bytes(ctypes_ref(L), self._cap[i], Hq))
            if ls.a_scratch.numel() < need:
                ls.a_scratch = torch.zeros(need, dtype=torch.uint8, device=o.device)
            stride = (self._cap[i] * o.block + o.buffer + 3) // 4 * 4
            sp = self.single_pass if self.single_pass is not None else single_pass_preferred(o, self._cap[i])
            if not sp and (self._scores[i] is None or self._scores[i].shape[-1] < stride):
                self._scores[i] = torch.empty((B, Hq, stride), dtype=torch.float32, device=o.device)
        if getattr(self, "_qs", None) is None or self._qs.shape != self.q.shape:
            self._qs = torch.empty_like(self.q)

    def _record(self, with_append: bool):
        o = self.store
        lib = N.lib()
        torch.mul(self.q, 1.0 / math.sqrt(o.head_dim), out=self._qs)  # every layer's query in one launch
        for i, l in enumerate(self.layers):
            ls = o[l]
            L = ctypes_ref(ls.struct())
            if with_append and self.fused_append:
                N.check(lib.pkv_append_flush_masked(L, N.ptr(self.k[i]), N.ptr(self.v[i]), N.ptr(self.active),
                                                    float(o.rel_scale_k), float(o.rel_scale_v),
                                                    N.ptr(self._flush_scr[i]), int(self._flush_scr[i].numel()),
                                                    N.stream()), "append_flush")
            else:
                if with_append:
                    N.check(lib.pkv_stage_token(L, N.ptr(self.k[i]), N.ptr(self.v[i]), N.stream()), "stage_token")
                N.check(lib.pkv_flush_staged(L, float(o.rel_scale_k), float(o.rel_scale_v), N.ptr(self._flush_scr[i]),
                                             int(self._flush_scr[i].numel()), N.stream()), "flush_staged")
            sp = self.single_pass
            if sp is None:
                sp = single_pass_preferred(o, self._cap[i])
            dst = self.out[i] if self._hout is None else self._hout[i]  # host: the last kernel stores there
            attention_decode_batched(o, l, self._qs[i], scores=self._scores[i], out=dst, nblocks=self._cap[i],
                                     single_pass=sp, prescaled=True)

    def _capture(self):
        dev = torch.device(self.store.device)
        self._prepare()
        self._record(False)  # warm-up outside the capture: nothing staged, so the flush appends nothing
        if self._pool is None:
            self._pool = torch.cuda.graph_pool_handle()
            self._side = torch.cuda.Stream(device=dev)
        cur = torch.cuda.current_stream(dev)
        self._side.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self._side):
            g.capture_begin(pool=self._pool)
            try:
                self._record(True)
            finally:
                g.capture_end()
        cur.wait_stream(self._side)
        self._graph = g
        self._key = self._state()
        self.captures += 1

    def step(self, k=None, v=None, q=None, active=None, out=None) -> torch.Tensor:
        """active (optional, [B] bool / 0-1): the sequences that append a token
        this step (the others only attend); their lengths then diverge on the
        device (a ragged batch, pkv_append_flush_masked).  out (optional, pinned
        host f32 [layers, B, Hq, D]): the attention kernels store every layer's
        output straight into it inside the graph (zero-copy; its address is part
        of the capture, so reuse one buffer); the return value is then `out`."""
        import numpy as np
        o = self.store
        if out is not None:
            if out.is_cuda or not out.is_pinned() or out.dtype != torch.float32 or not out.is_contiguous() \
                    or tuple(out.shape) != tuple(self.out.shape):
                raise E.ShapeMismatchError(f"out must be a pinned host f32 tensor of shape {tuple(self.out.shape)}")
        if ptr_of(out) != ptr_of(self._hout):
            self._hout = out  # a different output target: the capture key changes
        for dst, src in ((self.k, k), (self.v, v), (self.q, q)):
            if src is not None and src.data_ptr() != dst.data_ptr():
                dst.copy_(src.reshape(dst.shape), non_blocking=True)
        if active is None:
            act = np.ones(o.batch, bool)
            if not bool(self._active_all):
                self.active.fill_(1)
                self._active_all = True
        else:
            act = np.asarray(active.cpu() if isinstance(active, torch.Tensor) else active, dtype=bool).reshape(-1)
            if act.shape != (o.batch,):
                raise E.ShapeMismatchError(f"active must have {o.batch} entries")
            if not self.fused_append and not act.all():
                raise ValueError("an active mask needs fused_append (pkv_append_flush_masked)")
            self.active.copy_(torch.from_numpy(act.astype(np.uint8)), non_blocking=True)
            self._active_all = bool(act.all())
        # the graph covers blocks j < cap: re-capture once a flush could create block cap
        need = any(o[l].nblk_h >= self._cap[i] for i, l in enumerate(self.layers))
        if self._graph is None or need or self._state() != self._key:
            self._capture()
        self._graph.replay()
        for i, l in enumerate(self.layers):  # host mirrors follow the device, sequence by sequence
            ls = o[l]
            nres, nblk = self._seq_nres[i], self._seq_nblk[i]
            nres[act] += 1
            done = nres >= o.block
            nblk[done] += 1
            nres[done] -= o.block
            ls.tail_ub += int(done.sum()) * 2 * o.heads * ls.blk_max
            ls.nblk_h, ls.nres_h = int(nblk.max()), int(nres.max())
            ls.ragged = ls.ragged or not (np.all(nblk == nblk[0]) and np.all(nres == nres[0]))
        return self.out if self._hout is None else self._hout

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


def permutation_invariance_check(K, V, q, trials: int = 10, seed: int = 0, rel_scale_k: float = 0.1,
                                 rel_scale_v: float = 0.2) -> dict:
    """SPEC.md:537-545 (failures reported, not thrown).  K, V: [T, D] (one head),
    q: [D].  (1) f64 attention under `trials` random joint permutations of the
    rows against the unpermuted result (<= 1e-5 * |out|); (2) the compressed
    path (device store, fused attention) with repacking greedy / v_median
    against none (within 1e-4 relative)."""
    import numpy as np
    Kt = torch.as_tensor(np.asarray(K, dtype=np.float16) if not isinstance(K, torch.Tensor) else K)
    Vt = torch.as_tensor(np.asarray(V, dtype=np.float16) if not isinstance(V, torch.Tensor) else V)
    qt = torch.as_tensor(q).double()
    if Kt.dim() != 2 or Kt.shape != Vt.shape or qt.shape != (Kt.shape[1],) or trials < 1:
        raise E.ShapeMismatchError("K, V must be [T, D] and q [D]; trials >= 1")
    dev = torch.device("cuda", torch.cuda.current_device())
    Kd, Vd, qd = Kt.to(dev), Vt.to(dev), qt.to(dev)
    T, D = Kt.shape
    ref = attention_reference(Kd, Vd, qd)
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    worst = 0.0
    fails = 0
    for _ in range(trials):
        p = torch.randperm(T, generator=g).to(dev)
        err = float((attention_reference(Kd[p], Vd[p], qd) - ref).abs().max() / ref.abs().max().clamp_min(1e-300))
        worst = max(worst, err)
        fails += err > 1e-5
    outs = {}
    for strategy in ("none", "greedy", "v_median"):
        st = CompressedStore(1, 1, D, rel_scale_k=rel_scale_k, rel_scale_v=rel_scale_v, repack=strategy)
        st.compress_batch(0, Kd[:, None, :], Vd[:, None, :])
        outs[strategy] = attention_decode(st, 0, 0, qd.float()).double()
    base = outs["none"]
    rep = {s: float((o - base).abs().max() / base.abs().max().clamp_min(1e-300)) for s, o in outs.items() if s != "none"}
    return {"trials": trials, "f64_max_rel_err": worst, "f64_failures": int(fails),
            "repack_vs_none_max_rel": rep, "repack_pass": all(v <= 1e-4 for v in rep.values()),
            "pass": fails == 0 and all(v <= 1e-4 for v in rep.values())}
