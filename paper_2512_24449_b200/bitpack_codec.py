"""Lossless bit-pack codec on the GPU.

``encode_block`` / ``decode_block`` / ``decode_pack_at`` / ``compression_ratio``
with the reference's exact wire layout (byte map in DESIGN.md).
Encoding is two device passes (``pkv_encode_sizes`` for the data-dependent
length, then ``pkv_encode``); a PackedBlock holds its bytes in a device uint8
tensor.  Batched variants encode/decode many independent blocks per launch.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import _native as N
from . import errors as E
from .quantizer import KIND_K, KIND_V, QuantBlock

LAYOUT_K_INTERLEAVED, LAYOUT_V_CONTIGUOUS = 0, 1
PACK_SIZES = (2, 4, 8, 16, 32)
META_BITS = 20
FIXED_HEADER = 8


def header_bytes(rows: int, cols: int, k: int) -> int:
    P = (rows // k) * cols
    return FIXED_HEADER + (P + 1) // 2 + 2 * P + 4 * rows


@dataclass
class PackDescriptor:
    """SPEC.md:260-265."""
    width: int
    minimum: int

    def payload_bytes(self, k: int) -> int:
        return (k * self.width + 7) // 8


@dataclass
class PackedBlock:
    """SPEC.md:266-272.  `data` is the exact encoded byte string on the device."""
    data: torch.Tensor
    kind: int
    layout: int
    pack_size: int
    rows: int
    cols: int

    def __len__(self):
        return int(self.data.numel())

    def to_bytes(self) -> bytes:
        return bytes(self.data.cpu().numpy().tobytes())

    @staticmethod
    def from_bytes(buf: bytes, device="cuda") -> "PackedBlock":
        if len(buf) < FIXED_HEADER:
            raise E.MalformedBlockError("block shorter than its fixed header")
        kind, layout, k = buf[0], buf[1], buf[2]
        rows = int.from_bytes(buf[4:6], "little")
        cols = int.from_bytes(buf[6:8], "little")
        data = torch.frombuffer(bytearray(buf), dtype=torch.uint8).to(device)
        return PackedBlock(data, kind, layout, k, rows, cols)


def _check_k(k):
    if k not in PACK_SIZES:
        raise ValueError(f"pack_size must be one of {PACK_SIZES}")


def encode_blocks(qb: QuantBlock, pack_size: int = 16, layout: Optional[int] = None) -> List[PackedBlock]:
    """Encode n independent blocks (qb.q: [n, rows, cols]) in two launches."""
    _check_k(pack_size)
    if layout is None:
        layout = LAYOUT_K_INTERLEAVED if qb.kind == KIND_K else LAYOUT_V_CONTIGUOUS
    q = qb.q
    if q.dim() == 2:
        q = q.unsqueeze(0)
    q = q.to(torch.uint16).contiguous()
    n, rows, cols = (int(s) for s in q.shape)
    if rows % pack_size:
        raise E.ShapeMismatchError("rows must be divisible by pack_size")
    dev = q.device
    params = torch.stack([qb.scale.reshape(n, rows).float(), qb.zp.reshape(n, rows).float()], -1).contiguous()
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    sizes = torch.empty(n, dtype=torch.int64, device=dev)
    lib = N.lib()
    N.check(lib.pkv_encode_sizes(N.ptr(q), n, rows, cols, pack_size, layout, N.ptr(sizes), N.ptr(err), N.stream()),
            "encode_block")
    offs = torch.zeros(n, dtype=torch.int64, device=dev)
    if n > 1:
        offs[1:] = torch.cumsum(sizes[:-1], 0)
    total = int((offs[-1] + sizes[-1]).item()) if n else 0
    N.raise_flags(int(err.item()), "encode_block")
    out = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    N.check(lib.pkv_encode(N.ptr(q), N.ptr(params), n, rows, cols, pack_size, layout, qb.kind, N.ptr(offs),
                           N.ptr(out), N.ptr(err), N.stream()), "encode_block")
    N.raise_flags(int(err.item()), "encode_block")
    o = offs.tolist()
    s = sizes.tolist()
    return [PackedBlock(out[o[i]:o[i] + s[i]], qb.kind, layout, pack_size, rows, cols) for i in range(n)]


def encode_block(qb: QuantBlock, pack_size: int = 16, layout: Optional[int] = None) -> PackedBlock:
    """SPEC.md:275-283."""
    if qb.q.dim() != 2:
        raise E.ShapeMismatchError("encode_block takes one [rows, cols] block; use encode_blocks")
    return encode_blocks(qb, pack_size, layout)[0]


def _parse(p: PackedBlock):
    if len(p) < FIXED_HEADER:
        raise E.MalformedBlockError("block shorter than its fixed header")
    return p.rows, p.cols


def decode_blocks(blocks: Sequence[PackedBlock]) -> QuantBlock:
    """Decode many blocks of identical geometry in one launch."""
    if not blocks:
        raise ValueError("no blocks")
    rows, cols = _parse(blocks[0])
    dev = blocks[0].data.device
    for b in blocks:
        if (b.rows, b.cols) != (rows, cols):
            raise E.ShapeMismatchError("decode_blocks needs blocks of one geometry")
        if len(b) < FIXED_HEADER:
            raise E.MalformedBlockError("block shorter than its fixed header")
    lens = torch.tensor([len(b) for b in blocks], dtype=torch.int64)
    offs = torch.zeros_like(lens)
    offs[1:] = torch.cumsum(lens[:-1], 0)
    buf = torch.cat([b.data for b in blocks]) if len(blocks) > 1 else blocks[0].data.contiguous()
    buf = torch.cat([buf, torch.zeros(16, dtype=torch.uint8, device=dev)])
    n = len(blocks)
    q = torch.empty((n, rows, cols), dtype=torch.uint16, device=dev)
    params = torch.zeros((n, rows, 2), dtype=torch.float32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    offs_d, lens_d = offs.to(dev), lens.to(dev)     # keep alive across the async launch
    N.check(N.lib().pkv_decode(N.ptr(buf), N.ptr(offs_d), N.ptr(lens_d), n, rows, cols, N.ptr(q),
                               N.ptr(params), N.ptr(err), N.stream()), "decode_block")
    N.raise_flags(int(err.item()), "decode_block")
    return QuantBlock(q, params[..., 0], params[..., 1], blocks[0].kind, 0.0)


def decode_block(p: PackedBlock) -> QuantBlock:
    """SPEC.md:284-292."""
    qb = decode_blocks([p])
    return QuantBlock(qb.q[0], qb.scale[0], qb.zp[0], p.kind, 0.0)


def decode_pack_at(p: PackedBlock, pack_index: int) -> torch.Tensor:
    """k values of physical pack `pack_index`."""
    rows, cols = _parse(p)
    P = (rows // p.pack_size) * cols
    if not (0 <= pack_index < P):
        raise IndexError(f"pack index {pack_index} out of range [0, {P})")
    dev = p.data.device
    buf = torch.cat([p.data, torch.zeros(16, dtype=torch.uint8, device=dev)])
    offs = torch.zeros(1, dtype=torch.int64, device=dev)
    out = torch.empty(p.pack_size, dtype=torch.uint16, device=dev)
    N.check(N.lib().pkv_decode_pack_at(N.ptr(buf), N.ptr(offs), 1, pack_index, N.ptr(out), N.stream()),
            "decode_pack_at")
    return out


def compression_ratio(p: PackedBlock) -> float:
    """SPEC.md:302-310, pinned to the worked example (excludes the 8-byte fixed header)."""
    return p.rows * p.cols * 16 / (8 * (len(p) - FIXED_HEADER))


def wire_compression_ratio(p: PackedBlock) -> float:
    """rows*cols*2 / total block bytes (every header byte included)."""
    return p.rows * p.cols * 2 / len(p)


def kivi_baseline_cr(bit_width: int, group: int, meta_bits_per_group: int) -> float:
    """SPEC.md:606-614 (format arithmetic only)."""
    return 16 * group / (bit_width * group + meta_bits_per_group)
