"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the PackKV reference algorithm for the decode-time hot
path, following ``/root/reference/SPEC.md`` module by module (file:line cited
per function).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
as the checker / the CPU baseline — never as the product path.  The product
(``paper_2512_24449_b200``) never imports it and fails loudly when its CUDA
library is missing.

Parity pinning.  The reference ships no implementation (only
``pkg/src/packkv/errors.py``), so there is nothing to run or compile.  This
restatement is pinned against every known-answer example the SPEC gives for
the path (``tests/test_oracle_kat.py``); everything the SPEC leaves open is
pinned per SURVEY.md Appendix A and recorded in DESIGN.md ("Pinned format
decisions").  Beyond those examples parity is *anchored on the SPEC text*,
not on reference-produced vectors: "parity pinned to SPEC KATs only".

Arithmetic conventions:
  * quantization is f32: scale = f32(rel) * (mx - mn); t = (x - mn) / scale
    (IEEE divide); q = round-half-away-from-zero(t) computed exactly as
    r = floor(t); r += (t - r >= 0.5)   (never np.round / floor(t + 0.5));
  * dequantization is q * scale + zp in f32, mul then add (no FMA);
  * wire params are f16 (RNE), widened to f32 for dequantization.
"""
from __future__ import annotations

import itertools
import struct
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

try:  # error classes shared with the product so tests can assert on them
    from paper_2512_24449_b200 import errors as _E
except Exception:  # pragma: no cover - oracle usable stand-alone
    class _E:  # type: ignore
        class PackKVError(Exception):
            pass
        NonFiniteValueError = ShapeMismatchError = WidthOverflowError = PackKVError
        MalformedBlockError = InstanceTooLargeError = PackKVError

KIND_K, KIND_V = 0, 1
LAYOUT_K_INTERLEAVED, LAYOUT_V_CONTIGUOUS = 0, 1
META_BITS = 20           # 4-bit width + 16-bit minimum
FIXED_HEADER = 8         # kind, layout, pack_size, reserved, rows u16, cols u16
PACK_SIZES = (2, 4, 8, 16, 32)

# bit_length lookup for ranges < 2**16 (width = ceil(log2(range+1)))
_BITLEN = np.zeros(1 << 16, dtype=np.int64)
for _b in range(1, 17):
    _BITLEN[1 << (_b - 1): 1 << _b] = _b


def bit_length(a: np.ndarray) -> np.ndarray:
    a = np.asarray(a, dtype=np.int64)
    if a.size and a.max() >= (1 << 16):
        return np.array([int(v).bit_length() for v in a.ravel()], dtype=np.int64).reshape(a.shape)
    return _BITLEN[a]


# --------------------------------------------------------------------------
# quantizer
# --------------------------------------------------------------------------
@dataclass
class QuantBlock:
    """SPEC.md:102-108.  q: [rows, cols] int64 >= 0; scale/zp: f32 per row."""
    q: np.ndarray
    scale: np.ndarray
    zp: np.ndarray
    kind: int = KIND_K
    rel: float = 0.1

    @property
    def rows(self):
        return self.q.shape[0]

    @property
    def cols(self):
        return self.q.shape[1]


def round_half_away_nonneg(t: np.ndarray) -> np.ndarray:
    """Exact round-half-away-from-zero for t >= 0 in f32."""
    t = t.astype(np.float32)
    r = np.floor(t)
    r = r + ((t - r) >= np.float32(0.5)).astype(np.float32)
    return r


def quantize_token_wise(x: np.ndarray, rel: float, kind: int = KIND_K) -> QuantBlock:
    """per row mn, mx, scale = rel*(mx-mn), q = round((x-mn)/scale)."""
    x = np.asarray(x)
    if x.dtype != np.float16:
        x = x.astype(np.float16)
    if x.ndim != 2:
        raise _E.ShapeMismatchError("quantize_token_wise expects a 2-D [rows, cols] half tensor")
    if not (0.0 < rel <= 1.0):
        raise ValueError("rel_quant_scale must be in (0, 1]")
    xf = x.astype(np.float32)
    if not np.all(np.isfinite(xf)):
        raise _E.NonFiniteValueError("non-finite value in quantizer input")
    rows, cols = xf.shape
    if rows == 0 or cols == 0:
        return QuantBlock(np.zeros((rows, cols), np.int64), np.zeros(rows, np.float32),
                          np.zeros(rows, np.float32), kind, rel)
    mn = xf.min(axis=1)
    mx = xf.max(axis=1)
    scale = (np.float32(rel) * (mx - mn).astype(np.float32)).astype(np.float32)
    safe = np.where(scale > 0, scale, np.float32(1.0)).astype(np.float32)
    t = ((xf - mn[:, None]).astype(np.float32) / safe[:, None]).astype(np.float32)
    q = round_half_away_nonneg(t).astype(np.int64)
    q[scale == 0] = 0
    return QuantBlock(q, scale.astype(np.float32), mn.astype(np.float32), kind, rel)


def dequantize(q, scale, zp) -> np.ndarray:
    """q*scale + zp in f32, mul then add."""
    q = np.asarray(q)
    s = np.asarray(scale, dtype=np.float32)
    z = np.asarray(zp, dtype=np.float32)
    if q.ndim == 2:
        s = s[:, None]
        z = z[:, None]
    prod = (q.astype(np.float32) * s).astype(np.float32)
    return (prod + z).astype(np.float32)


def max_abs_error(x: np.ndarray, rel: float) -> float:
    """SPEC.md:129-137."""
    qb = quantize_token_wise(x, rel)
    d = dequantize(qb.q, qb.scale, qb.zp)
    if d.size == 0:
        return 0.0
    return float(np.max(np.abs(x.astype(np.float32) - d)))


# --------------------------------------------------------------------------
# repacker
# --------------------------------------------------------------------------
@dataclass
class RepackPlan:
    """SPEC.md:181-186."""
    permutation: np.ndarray
    strategy: str
    cost_bits: int


def pack_cost(group: np.ndarray) -> int:
    """sum_d (|g| * w_d + META_BITS), w_d = bit_length(range_d)."""
    g = np.asarray(group, dtype=np.int64)
    if g.ndim == 1:
        g = g[None, :]
    if g.shape[0] == 0:
        raise ValueError("pack_cost of an empty group")
    rng = g.max(axis=0) - g.min(axis=0)
    return int(np.sum(g.shape[0] * bit_length(rng) + META_BITS))


def plan_cost(vectors: np.ndarray, perm: Sequence[int], k: int) -> int:
    v = np.asarray(vectors, dtype=np.int64)[np.asarray(perm, dtype=np.int64)]
    return sum(pack_cost(v[i:i + k]) for i in range(0, v.shape[0], k))


def repack_none(vectors: np.ndarray, k: int) -> RepackPlan:
    n = np.asarray(vectors).shape[0]
    perm = np.arange(n, dtype=np.int64)
    return RepackPlan(perm, "none", plan_cost(vectors, perm, k) if n else 0)


def lower_median(v: np.ndarray) -> np.ndarray:
    """Lower median per row: sorted(row)[(n-1)//2] (Appendix A #18)."""
    v = np.asarray(v, dtype=np.int64)
    n = v.shape[1]
    return np.partition(v, (n - 1) // 2, axis=1)[:, (n - 1) // 2]


def repack_v_median(vectors: np.ndarray, v_parts: np.ndarray, k: int) -> RepackPlan:
    """stable ascending sort of tokens by lower median of v_part."""
    med = lower_median(v_parts)
    perm = np.argsort(med, kind="stable").astype(np.int64)
    return RepackPlan(perm, "v_median", plan_cost(vectors, perm, k))


def repack_greedy(vectors: np.ndarray, k: int) -> RepackPlan:
    """SPEC.md:198-207 / PAPER.md:333-350 (Algorithm 1).

    Centroid seed is integer-exact: argmin_i ||m*x_i - S||^2 with m = |R|,
    S = sum_{i in R} x_i (same order as exact real L2; Appendix A #7).  Ties
    (equal distance or equal marginal cost) go to the lowest original index
    (SPEC.md:236).  Marginal cost uses pack_cost over both parts.
    """
    X = np.asarray(vectors, dtype=np.int64)
    n = X.shape[0]
    remaining = list(range(n))
    perm: List[int] = []
    total = 0
    while remaining:
        R = np.array(remaining, dtype=np.int64)
        XR = X[R]
        m = len(remaining)
        S = XR.sum(axis=0)
        diff = m * XR - S[None, :]
        dist = np.einsum("ij,ij->i", diff, diff)
        s_pos = int(np.argmin(dist))          # first minimum = lowest index (R ascending)
        seed = remaining.pop(s_pos)
        group = [seed]
        gmax = X[seed].copy()
        gmin = X[seed].copy()
        cur_cost_w = 0                        # sum_d w_d(P)
        while len(group) < k and remaining:
            R = np.array(remaining, dtype=np.int64)
            XR = X[R]
            nmax = np.maximum(gmax[None, :], XR)
            nmin = np.minimum(gmin[None, :], XR)
            wsum = bit_length(nmax - nmin).sum(axis=1)
            p = len(group)
            marg = (p + 1) * wsum - p * cur_cost_w
            j_pos = int(np.argmin(marg))
            j = remaining.pop(j_pos)
            group.append(j)
            gmax = np.maximum(gmax, X[j])
            gmin = np.minimum(gmin, X[j])
            cur_cost_w = int(wsum[j_pos])
        total += pack_cost(X[group])
        perm.extend(group)
    return RepackPlan(np.array(perm, dtype=np.int64), "greedy", total)


def _partitions(items: List[int], k: int):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for comb in itertools.combinations(rest, k - 1):
        left = [x for x in rest if x not in comb]
        for tail in _partitions(left, k):
            yield [[first, *comb]] + tail


def count_partitions(n: int, k: int) -> int:
    return sum(1 for _ in _partitions(list(range(n)), k))


def oracle_optimal(vectors: np.ndarray, k: int):
    """exhaustive search, n <= 12 and n % k == 0."""
    X = np.asarray(vectors, dtype=np.int64)
    n = X.shape[0]
    if n > 12 or n % k != 0:
        raise _E.InstanceTooLargeError(f"oracle_optimal needs n <= 12 and n % k == 0 (n={n}, k={k})")
    best = None
    best_part = None
    for part in _partitions(list(range(n)), k):   # canonical, lexicographic order
        c = sum(pack_cost(X[g]) for g in part)
        if best is None or c < best:
            best, best_part = c, part
    return best_part, int(best)


# --------------------------------------------------------------------------
# bitpack codec (byte map SURVEY.md Appendix C)
# --------------------------------------------------------------------------
def k_pos(cols: int) -> np.ndarray:
    """Physical position of column c within a row-group for the K layout.

    pos(c) = sum_{r < c mod 4} ceil((cols - r)/4) + c div 4.
    """
    c = np.arange(cols)
    counts = [(cols - r + 3) // 4 for r in range(4)]
    base = np.cumsum([0] + counts[:3])
    return (base[c % 4] + c // 4).astype(np.int64)


def phys_pos(cols: int, layout: int) -> np.ndarray:
    if layout == LAYOUT_K_INTERLEAVED:
        return k_pos(cols)
    return np.arange(cols, dtype=np.int64)


def header_bytes(rows: int, cols: int, k: int) -> int:
    P = (rows // k) * cols
    return FIXED_HEADER + (P + 1) // 2 + 2 * P + 4 * rows


def payload_bytes(k: int, w: np.ndarray) -> np.ndarray:
    return (k * np.asarray(w, dtype=np.int64) + 7) // 8


def _f16_bits(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float16).view(np.uint16)


def params_to_f16(scale, zp):
    """Wire params.  Scale overflow in f16 -> WidthOverflowError (Appendix A #14)."""
    s16 = np.asarray(scale, dtype=np.float32).astype(np.float16)
    z16 = np.asarray(zp, dtype=np.float32).astype(np.float16)
    if not np.all(np.isfinite(s16)):
        raise _E.WidthOverflowError("per-token scale overflows the f16 wire field")
    return s16, z16


@dataclass
class PackInfo:
    widths: np.ndarray     # [P] physical order
    minima: np.ndarray     # [P]
    offsets: np.ndarray    # [P] byte offset of payload from block start
    hdr: int


def encode_block(qb: QuantBlock, k: int = 16, layout: Optional[int] = None,
                 kind: Optional[int] = None) -> bytes:
    """SPEC.md:275-283 and wire layout SPEC.md:330."""
    q = np.asarray(qb.q, dtype=np.int64)
    rows, cols = q.shape
    kind = qb.kind if kind is None else kind
    if layout is None:
        layout = LAYOUT_K_INTERLEAVED if kind == KIND_K else LAYOUT_V_CONTIGUOUS
    if k not in PACK_SIZES:
        raise ValueError(f"pack_size must be one of {PACK_SIZES}")
    if rows % k != 0:
        raise _E.ShapeMismatchError("rows must be divisible by pack_size")
    if q.size and (q.min() < 0 or q.max() >= (1 << 16)):
        raise _E.WidthOverflowError("quantized values must lie in [0, 2^16)")
    G = rows // k
    P = G * cols
    pos = phys_pos(cols, layout)
    inv = np.empty(cols, dtype=np.int64)
    inv[pos] = np.arange(cols)                       # physical position -> column
    # packs in physical order: [G, cols(phys), k]
    packs = q.reshape(G, k, cols).transpose(0, 2, 1)[:, inv, :].reshape(P, k)
    mins = packs.min(axis=1) if P else np.zeros(0, np.int64)
    rng = (packs.max(axis=1) - mins) if P else np.zeros(0, np.int64)
    w = bit_length(rng)
    if np.any(w > 15):
        raise _E.WidthOverflowError("pack width exceeds 15 bits")
    s16, z16 = params_to_f16(qb.scale, qb.zp)
    out = bytearray()
    out += bytes([kind, layout, k, 0])
    out += int(rows).to_bytes(2, "little") + int(cols).to_bytes(2, "little")
    nib = np.zeros((P + 1) // 2, dtype=np.uint8)
    wi = w.astype(np.uint8)
    nib[:] = 0
    if P:
        nib_full = np.zeros(((P + 1) // 2) * 2, dtype=np.uint8)
        nib_full[:P] = wi
        nib = (nib_full[0::2] | (nib_full[1::2] << 4)).astype(np.uint8)
    out += nib.tobytes()
    out += mins.astype("<u2").tobytes()
    par = np.empty(2 * rows, dtype=np.uint16)
    par[0::2] = s16.view(np.uint16)
    par[1::2] = z16.view(np.uint16)
    out += par.astype("<u2").tobytes()
    # payloads, little-endian bit numbering, value j at bits [j*w, (j+1)*w)
    pb = payload_bytes(k, w)
    total_pay = int(pb.sum())
    if total_pay:
        delta = packs - mins[:, None]
        maxw = int(w.max())
        bitpos0 = np.concatenate([[0], np.cumsum(pb)[:-1]]) * 8
        bits = np.zeros(total_pay * 8, dtype=np.uint8)
        for b in range(maxw):
            sel = w > b                                   # packs with at least b+1 bits
            if not np.any(sel):
                continue
            j = np.arange(k)[None, :]
            idx = bitpos0[sel][:, None] + j * w[sel][:, None] + b
            bits[idx.ravel()] = ((delta[sel] >> b) & 1).astype(np.uint8).ravel()
        out += np.packbits(bits, bitorder="little").tobytes()
    return bytes(out)


def parse_header(buf: bytes):
    if len(buf) < FIXED_HEADER:
        raise _E.MalformedBlockError("block shorter than its fixed header")
    kind, layout, k, _rsv = buf[0], buf[1], buf[2], buf[3]
    rows = int.from_bytes(buf[4:6], "little")
    cols = int.from_bytes(buf[6:8], "little")
    if kind not in (KIND_K, KIND_V) or layout not in (0, 1) or k not in PACK_SIZES:
        raise _E.MalformedBlockError("bad kind/layout/pack_size in block header")
    if rows % k != 0:
        raise _E.MalformedBlockError("rows not divisible by pack_size")
    return kind, layout, k, rows, cols


def pack_info(buf: bytes) -> Tuple[Tuple[int, int, int, int, int], PackInfo]:
    kind, layout, k, rows, cols = parse_header(buf)
    G = rows // k
    P = G * cols
    hdr = header_bytes(rows, cols, k)
    if len(buf) < hdr:
        raise _E.MalformedBlockError("block shorter than its header")
    a = np.frombuffer(buf, dtype=np.uint8)
    nb = a[FIXED_HEADER:FIXED_HEADER + (P + 1) // 2]
    w = np.empty(((P + 1) // 2) * 2, dtype=np.int64)
    w[0::2] = nb & 0xF
    w[1::2] = nb >> 4
    w = w[:P]
    m0 = FIXED_HEADER + (P + 1) // 2
    mins = np.frombuffer(buf[m0:m0 + 2 * P], dtype="<u2").astype(np.int64)
    pb = payload_bytes(k, w)
    offs = hdr + np.concatenate([[0], np.cumsum(pb)[:-1]]).astype(np.int64) if P else np.zeros(0, np.int64)
    if len(buf) != hdr + int(pb.sum()):
        raise _E.MalformedBlockError("payload length does not match the width table")
    return (kind, layout, k, rows, cols), PackInfo(w, mins, offs, hdr)


def decode_block(buf: bytes) -> QuantBlock:
    """exact inverse of encode_block (params widened from f16)."""
    (kind, layout, k, rows, cols), pi = pack_info(buf)
    G = rows // k
    P = G * cols
    a = np.frombuffer(buf, dtype=np.uint8)
    p0 = FIXED_HEADER + (P + 1) // 2 + 2 * P
    par = np.frombuffer(buf[p0:p0 + 4 * rows], dtype="<u2")
    scale = par[0::2].view(np.float16).astype(np.float32)
    zp = par[1::2].view(np.float16).astype(np.float32)
    vals = np.zeros((P, k), dtype=np.int64)
    if P and pi.widths.max() > 0:
        bits = np.unpackbits(a[pi.hdr:], bitorder="little").astype(np.int64)
        base = (pi.offsets - pi.hdr) * 8
        j = np.arange(k)[None, :]
        for b in range(int(pi.widths.max())):
            sel = pi.widths > b
            idx = base[sel][:, None] + j * pi.widths[sel][:, None] + b
            vals[sel] |= bits[idx] << b
    vals += pi.minima[:, None]
    pos = phys_pos(cols, layout)
    # packs [G, phys, k] -> q[g*k + j, c] = packs[g, pos[c], j]
    pk = vals.reshape(G, cols, k)[:, pos, :]          # [G, cols, k]
    q = pk.transpose(0, 2, 1).reshape(rows, cols)
    return QuantBlock(q, scale, zp, kind, 0.0)


def decode_pack_at(buf: bytes, i: int) -> np.ndarray:
    """k values of physical pack i, without decoding others."""
    (kind, layout, k, rows, cols), pi = pack_info(buf)
    P = (rows // k) * cols
    if i < 0 or i >= P:
        raise IndexError(f"pack index {i} out of range [0, {P})")
    w = int(pi.widths[i])
    out = np.full(k, pi.minima[i], dtype=np.int64)
    if w:
        off = int(pi.offsets[i])
        nbytes = (k * w + 7) // 8
        v = int.from_bytes(buf[off:off + nbytes], "little")
        mask = (1 << w) - 1
        out += np.array([(v >> (j * w)) & mask for j in range(k)], dtype=np.int64)
    return out


def compression_ratio(buf: bytes) -> float:
    """SPEC.md:302-310, pinned to the worked example 131072/22528 = 5.82 (excludes the 8 B fixed header)."""
    _, _, _, rows, cols = parse_header(buf)
    return rows * cols * 16 / (8 * (len(buf) - FIXED_HEADER))


def wire_compression_ratio(buf: bytes) -> float:
    _, _, _, rows, cols = parse_header(buf)
    return rows * cols * 2 / len(buf)


def kivi_baseline_cr(bit_width: int, group: int, meta_bits_per_group: int) -> float:
    """SPEC.md:606-614."""
    return 16 * group / (bit_width * group + meta_bits_per_group)


# --------------------------------------------------------------------------
# kv_store
# --------------------------------------------------------------------------
@dataclass
class DirEntry:
    """SPEC.md:351-356."""
    kind: int
    layer: int
    head: int
    token_start: int
    token_end: int
    byte_offset: int
    byte_len: int
    permutation: np.ndarray


@dataclass
class OracleStore:
    """SPEC.md:357-362.  One arena for all layers, appended in call order."""
    layers: int
    heads: int
    head_dim: int
    rel_k: float = 0.1
    rel_v: float = 0.2
    pack_size: int = 16
    repack: str = "none"
    block: int = 64
    buffer: int = 128
    arena: bytearray = field(default_factory=bytearray)
    directory: List[DirEntry] = field(default_factory=list)

    def __post_init__(self):
        self.stage_k = [np.zeros((0, self.heads, self.head_dim), np.float16) for _ in range(self.layers)]
        self.stage_v = [np.zeros((0, self.heads, self.head_dim), np.float16) for _ in range(self.layers)]
        self.flushed = [0] * self.layers   # tokens already compressed per layer

    def _check(self, layer, kv):
        if not (0 <= layer < self.layers):
            raise IndexError("layer out of range")
        kv = np.asarray(kv)
        if kv.shape[-2:] != (self.heads, self.head_dim):
            raise _E.ShapeMismatchError(
                f"expected [..., {self.heads}, {self.head_dim}], got {kv.shape}")
        kv = kv.astype(np.float16)
        if not np.all(np.isfinite(kv.astype(np.float32))):
            raise _E.NonFiniteValueError("non-finite KV value")
        return kv

    def append_token(self, layer: int, k_vec, v_vec):
        """SPEC.md:365-373."""
        k_vec = self._check(layer, np.asarray(k_vec).reshape(self.heads, self.head_dim))
        v_vec = self._check(layer, np.asarray(v_vec).reshape(self.heads, self.head_dim))
        self.stage_k[layer] = np.concatenate([self.stage_k[layer], k_vec[None]], 0)
        self.stage_v[layer] = np.concatenate([self.stage_v[layer], v_vec[None]], 0)
        if self.stage_k[layer].shape[0] >= self.block:
            self._flush(layer)

    def compress_batch(self, layer: int, k_tokens, v_tokens):
        """equivalent to appending each token in order."""
        k_tokens = self._check(layer, k_tokens)
        v_tokens = self._check(layer, v_tokens)
        if k_tokens.shape != v_tokens.shape:
            raise _E.ShapeMismatchError("K and V batches differ in shape")
        self.stage_k[layer] = np.concatenate([self.stage_k[layer], k_tokens], 0)
        self.stage_v[layer] = np.concatenate([self.stage_v[layer], v_tokens], 0)
        while self.stage_k[layer].shape[0] >= self.block:
            self._flush(layer)

    def plan(self, qk: List[QuantBlock], qv: List[QuantBlock]) -> RepackPlan:
        kp = np.concatenate([b.q for b in qk], axis=1)   # [64, H*D]
        vp = np.concatenate([b.q for b in qv], axis=1)
        vec = np.concatenate([kp, vp], axis=1)
        if self.repack == "none":
            return repack_none(vec, self.pack_size)
        if self.repack == "v_median":
            return repack_v_median(vec, vp, self.pack_size)
        if self.repack == "greedy":
            return repack_greedy(vec, self.pack_size)
        raise ValueError(f"unknown repack strategy {self.repack}")

    def _flush(self, layer: int):
        n = self.block
        kb, vb = self.stage_k[layer][:n], self.stage_v[layer][:n]
        qk = [quantize_token_wise(kb[:, h, :], self.rel_k, KIND_K) for h in range(self.heads)]
        qv = [quantize_token_wise(vb[:, h, :], self.rel_v, KIND_V) for h in range(self.heads)]
        plan = self.plan(qk, qv)
        perm = plan.permutation
        t0 = self.flushed[layer]
        for kind, qs in ((KIND_K, qk), (KIND_V, qv)):
            for h, qb in enumerate(qs):
                pq = QuantBlock(qb.q[perm], qb.scale[perm], qb.zp[perm], kind, qb.rel)
                layout = LAYOUT_K_INTERLEAVED if kind == KIND_K else LAYOUT_V_CONTIGUOUS
                blk = encode_block(pq, self.pack_size, layout, kind)
                self.directory.append(DirEntry(kind, layer, h, t0, t0 + n, len(self.arena),
                                               len(blk), perm.copy()))
                self.arena += blk
        self.flushed[layer] += n
        self.stage_k[layer] = self.stage_k[layer][n:]
        self.stage_v[layer] = self.stage_v[layer][n:]

    def iterate_blocks(self, layer: int, kind: int):
        """directory entries of (layer, kind) + residue count."""
        ents = [e for e in self.directory if e.layer == layer and e.kind == kind]
        return ents, self.stage_k[layer].shape[0]

    def block_bytes(self, e: DirEntry) -> bytes:
        return bytes(self.arena[e.byte_offset:e.byte_offset + e.byte_len])

    def layer_stream(self, layer: int) -> bytes:
        """Concatenation of the layer's blocks in directory order (per-layer sub-store)."""
        return b"".join(self.block_bytes(e) for e in self.directory if e.layer == layer)

    def total_tokens(self, layer: int) -> int:
        return self.flushed[layer] + self.stage_k[layer].shape[0]

    def snapshot_stats(self):
        """SPEC.md:383-391 (exact byte counts and CR per kind/layer)."""
        out = {}
        for e in self.directory:
            d = out.setdefault((e.layer, e.kind), {"bytes": 0, "logical": 0, "blocks": 0})
            d["bytes"] += e.byte_len
            d["logical"] += (e.token_end - e.token_start) * self.head_dim * 2
            d["blocks"] += 1
        for d in out.values():
            d["cr"] = d["logical"] / d["bytes"] if d["bytes"] else None
        return out


# --------------------------------------------------------------------------
# fused kernels
# --------------------------------------------------------------------------
def _head_entries(store: OracleStore, layer: int, head: int, kind: int):
    if not (0 <= head < store.heads):
        raise IndexError("head out of range")
    ents, _ = store.iterate_blocks(layer, kind)
    return [e for e in ents if e.head == head]


def _deq_block_from_bytes(buf: bytes) -> np.ndarray:
    qb = decode_block(buf)
    return dequantize(qb.q, qb.scale, qb.zp)


def fused_k_scores(store: OracleStore, layer: int, head: int, q) -> Tuple[np.ndarray, np.ndarray]:
    """scores in block/permuted order + residue; f32 accumulation.

    Processes one block at a time (block-sized scratch, independent of L).
    """
    q = np.asarray(q, dtype=np.float32)
    if q.shape != (store.head_dim,):
        raise _E.ShapeMismatchError("|q| must equal head_dim")
    scores, tmap = [], []
    for e in _head_entries(store, layer, head, KIND_K):
        deq = _deq_block_from_bytes(store.block_bytes(e))
        scores.append((deq @ q).astype(np.float32))
        tmap.append(e.token_start + e.permutation)
    res = store.stage_k[layer][:, head, :].astype(np.float32)
    scores.append((res @ q).astype(np.float32))
    tmap.append(store.flushed[layer] + np.arange(res.shape[0]))
    return np.concatenate(scores).astype(np.float32), np.concatenate(tmap).astype(np.int64)


def fused_v_output(store: OracleStore, layer: int, head: int, w) -> np.ndarray:
    """out[c] = sum_t w[t] * deq(v[t][c]), fixed-order f32 reduction."""
    w = np.asarray(w, dtype=np.float32)
    if w.shape != (store.total_tokens(layer),):
        raise _E.ShapeMismatchError("|w| must equal total tokens")
    out = np.zeros(store.head_dim, dtype=np.float32)
    t = 0
    for e in _head_entries(store, layer, head, KIND_V):
        deq = _deq_block_from_bytes(store.block_bytes(e))
        n = deq.shape[0]
        out = (out + (w[t:t + n] @ deq).astype(np.float32)).astype(np.float32)
        t += n
    res = store.stage_v[layer][:, head, :].astype(np.float32)
    out = (out + (w[t:] @ res).astype(np.float32)).astype(np.float32)
    return out


def naive_k_scores(store: OracleStore, layer: int, head: int, q) -> np.ndarray:
    """decode everything, dequantize, f64 matvec."""
    q = np.asarray(q, dtype=np.float64)
    mats = [_deq_block_from_bytes(store.block_bytes(e)).astype(np.float64)
            for e in _head_entries(store, layer, head, KIND_K)]
    mats.append(store.stage_k[layer][:, head, :].astype(np.float64))
    return np.concatenate(mats, 0) @ q


def naive_v_output(store: OracleStore, layer: int, head: int, w) -> np.ndarray:
    w = np.asarray(w, dtype=np.float64)
    mats = [_deq_block_from_bytes(store.block_bytes(e)).astype(np.float64)
            for e in _head_entries(store, layer, head, KIND_V)]
    mats.append(store.stage_v[layer][:, head, :].astype(np.float64))
    return w @ np.concatenate(mats, 0)


# --------------------------------------------------------------------------
# attention_sim
# --------------------------------------------------------------------------
def softmax64(s: np.ndarray) -> np.ndarray:
    s = np.asarray(s, dtype=np.float64)
    e = np.exp(s - s.max())
    return e / e.sum()


def attention_decode(store: OracleStore, layer: int, head: int, q) -> np.ndarray:
    """fused K -> 1/sqrt(d) -> stable softmax -> fused V."""
    s, _ = fused_k_scores(store, layer, head, q)
    a = softmax64(s.astype(np.float64) / math.sqrt(store.head_dim)).astype(np.float32)
    return fused_v_output(store, layer, head, a)


def attention_reference(K, V, q) -> np.ndarray:
    """direct f64 softmax(Kq/sqrt(d))^T V."""
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    if K.shape != V.shape or K.shape[1] != q.shape[0]:
        raise _E.ShapeMismatchError("K, V, q dimensions disagree")
    return softmax64(K @ q / math.sqrt(K.shape[1])) @ V


# --------------------------------------------------------------------------
# synthetic data (bench inputs per BASELINE.md §3)
# --------------------------------------------------------------------------
def gen_gauss_outlier(rng: np.random.Generator, tokens: int, head_dim: int, n_outlier: int,
                      amp: float = 8.0, sigma: float = 2.0) -> np.ndarray:
    """N(0,1) fp16 [tokens, head_dim] with n_outlier channels of +-amp + N(0, sigma)."""
    x = rng.standard_normal((tokens, head_dim), dtype=np.float32)
    if n_outlier:
        ch = rng.choice(head_dim, size=n_outlier, replace=False)
        sign = rng.choice([-1.0, 1.0], size=n_outlier).astype(np.float32)
        x[:, ch] = sign[None, :] * amp + sigma * rng.standard_normal((tokens, n_outlier), dtype=np.float32)
    return x.astype(np.float16)


def generate_synthetic(mode: str, seed: int, layers: int, heads: int, head_dim: int, tokens: int,
                       amplitude: float = 1.0):
    """SPEC.md:58-66.  Returns (K, V) of shape [layers, heads, tokens, head_dim] fp16."""
    rng = np.random.default_rng(seed)
    shape = (layers, heads, tokens, head_dim)
    if mode == "uniform":
        K = rng.uniform(-amplitude, amplitude, shape)
        V = rng.uniform(-amplitude, amplitude, shape)
    elif mode == "channel-banded":
        offk = rng.uniform(-4 * amplitude, 4 * amplitude, (layers, heads, 1, head_dim))
        offv = rng.uniform(-4 * amplitude, 4 * amplitude, (layers, heads, 1, head_dim))
        K = offk + 0.25 * amplitude * rng.standard_normal(shape)
        V = offv + 0.25 * amplitude * rng.standard_normal(shape)
    elif mode == "token-scaled":
        sk = rng.uniform(0.1, 2.0, (layers, heads, tokens, 1)) * amplitude
        sv = rng.uniform(0.1, 2.0, (layers, heads, tokens, 1)) * amplitude
        K = sk * rng.standard_normal(shape)
        V = sv * rng.standard_normal(shape)
    elif mode == "gauss-outlier":
        K = np.empty(shape, np.float16)
        V = np.empty(shape, np.float16)
        for l in range(layers):
            for h in range(heads):
                K[l, h] = gen_gauss_outlier(rng, tokens, head_dim, max(1, head_dim * 4 // 128))
                V[l, h] = gen_gauss_outlier(rng, tokens, head_dim, max(1, head_dim // 128))
    else:
        raise ValueError(f"unknown synthetic mode {mode}")
    return np.asarray(K, dtype=np.float16), np.asarray(V, dtype=np.float16)


def threads() -> int:
    return int(os.environ.get("PACKKV_THREADS", len(os.sched_getaffinity(0))))


# --------------------------------------------------------------------------
# file formats (test infrastructure restatements)
# --------------------------------------------------------------------------
# KV dump, SPEC.md:40-57 (ops) and :82 (layout): "PKKV" | version u16 = 1 |
# layers u16 | heads u16 | head_dim u16 | tokens u32 | per (layer, head): K then
# V, tokens x head_dim raw f16, row-major, little-endian, no padding.
_DUMP_HDR = struct.Struct("<4sHHHHI")


def write_dump(k, v, path):
    """k, v: [layers, heads, tokens, head_dim] float16 arrays."""
    k = np.asarray(k, np.float16)
    v = np.asarray(v, np.float16)
    L, H, T, D = k.shape
    with open(path, "wb") as f:
        f.write(_DUMP_HDR.pack(b"PKKV", 1, L, H, D, T))
        for l in range(L):
            for h in range(H):
                f.write(k[l, h].astype("<f2").tobytes())
                f.write(v[l, h].astype("<f2").tobytes())


def read_dump(path):
    """(k, v) [layers, heads, tokens, head_dim] f16; distinct
    errors for bad magic, truncation and non-finite values."""
    data = open(path, "rb").read()
    if len(data) < 4 or data[:4] != b"PKKV":
        raise _E.BadMagicError("not a PKKV dump")
    if len(data) < _DUMP_HDR.size:
        raise _E.TruncatedDumpError("header truncated")
    _, ver, L, H, D, T = _DUMP_HDR.unpack_from(data)
    if ver != 1:
        raise _E.DumpFormatError(f"unsupported dump version {ver}")
    n = L * H * T * D
    if len(data) < _DUMP_HDR.size + 4 * n:
        raise _E.TruncatedDumpError("payload truncated")
    if len(data) > _DUMP_HDR.size + 4 * n:
        raise _E.DumpFormatError("trailing bytes after the payload")
    a = np.frombuffer(data, "<f2", count=2 * n, offset=_DUMP_HDR.size).reshape(L, H, 2, T, D)
    if not np.all(np.isfinite(a.astype(np.float32))):
        raise _E.NonFiniteValueError("non-finite value in dump")
    return a[:, :, 0].astype(np.float16), a[:, :, 1].astype(np.float16)


# Compressed store file "PKKS" v1 (header + arena + directory;
# the field layout is the builder's, documented in DESIGN.md §3.1).  One
# sequence here (batch = 1); arena offsets 16-byte aligned, zero padding.
_PKKS_HDR = struct.Struct("<4sHHHHHHHHB3xff")
_PKKS_LAYER = struct.Struct("<IIQ")
_PKKS_REC = struct.Struct("<QI")
_REPACK_CODE = {"none": 0, "greedy": 1, "v_median": 2}


def save_pkks(store: "OracleStore", path):
    out = bytearray(_PKKS_HDR.pack(b"PKKS", 1, store.layers, 1, store.heads, store.head_dim, store.block,
                                   store.pack_size, store.buffer, _REPACK_CODE[store.repack],
                                   np.float32(store.rel_k), np.float32(store.rel_v)))
    for l in range(store.layers):
        ents = [e for e in store.directory if e.layer == l]   # order (block-set, kind, head)
        nblk = len(ents) // (2 * store.heads)
        nres = store.stage_k[l].shape[0]
        arena, recs, perms = bytearray(), [], []
        for i, e in enumerate(ents):
            recs.append((len(arena), e.byte_len))
            arena += store.block_bytes(e)
            arena += bytes(-len(arena) % 16)
            if i % (2 * store.heads) == 0:
                perms.append(np.asarray(e.permutation, np.uint8))
        out += _PKKS_LAYER.pack(nblk, nres, len(arena))
        out += arena
        for r in recs:
            out += _PKKS_REC.pack(*r)
        for p in perms:
            out += p.tobytes()
        for st in (store.stage_k[l], store.stage_v[l]):      # [nres, H, D] -> per head
            for h in range(store.heads):
                out += np.ascontiguousarray(st[:, h, :]).astype("<f2").tobytes()
    open(path, "wb").write(bytes(out))


def load_pkks(path) -> "OracleStore":
    try:
        return _load_pkks(open(path, "rb").read())
    except (ValueError, struct.error, KeyError) as e:
        raise _E.StoreFormatError(f"malformed PKKS file: {e}") from e


def _load_pkks(data: bytes) -> "OracleStore":
    if data[:4] != b"PKKS" or len(data) < _PKKS_HDR.size:
        raise _E.StoreFormatError("not a PKKS store file")
    (_, ver, layers, batch, heads, head_dim, block, k, buffer, rep, rel_k,
     rel_v) = _PKKS_HDR.unpack_from(data)
    if ver != 1 or batch != 1:
        raise _E.StoreFormatError("unsupported PKKS version or batch")
    repack = {v: s for s, v in _REPACK_CODE.items()}[rep]
    st = OracleStore(layers, heads, head_dim, float(rel_k), float(rel_v), k, repack, block, buffer)
    pos = _PKKS_HDR.size
    for l in range(layers):
        nblk, nres, alen = _PKKS_LAYER.unpack_from(data, pos)
        pos += _PKKS_LAYER.size
        arena = data[pos:pos + alen]
        pos += alen
        recs = [_PKKS_REC.unpack_from(data, pos + i * _PKKS_REC.size) for i in range(nblk * 2 * heads)]
        pos += len(recs) * _PKKS_REC.size
        perms = [np.frombuffer(data, np.uint8, block, pos + j * block).astype(np.int64) for j in range(nblk)]
        pos += nblk * block
        for i, (off, ln) in enumerate(recs):
            j, r = divmod(i, 2 * heads)
            kind, h = divmod(r, heads)
            st.directory.append(DirEntry(kind, l, h, j * block, (j + 1) * block, len(st.arena), ln, perms[j]))
            st.arena += arena[off:off + ln]
        st.flushed[l] = nblk * block
        sk = np.frombuffer(data, "<f2", heads * nres * head_dim, pos).reshape(heads, nres, head_dim)
        pos += sk.nbytes
        sv = np.frombuffer(data, "<f2", heads * nres * head_dim, pos).reshape(heads, nres, head_dim)
        pos += sv.nbytes
        st.stage_k[l] = sk.transpose(1, 0, 2).astype(np.float16)
        st.stage_v[l] = sv.transpose(1, 0, 2).astype(np.float16)
    if pos != len(data):
        raise _E.StoreFormatError("trailing or missing bytes")
    return st
