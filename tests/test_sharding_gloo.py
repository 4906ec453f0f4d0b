"""Multi-rank host logic of the (batch, kv-head) sharding on CPU: world_size 2
over gloo.  Each rank runs the per-unit attention on its own units (the CPU
oracle stands in for the CUDA kernels here — test infrastructure only), the
outputs are all-gathered and must equal the unsharded computation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_24449_b200 import sharding as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(B, H, G, D, T, seed=0):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((B, T, H, D)).astype(np.float16)
    V = rng.standard_normal((B, T, H, D)).astype(np.float16)
    q = rng.standard_normal((B, H * G, D)).astype(np.float32)
    return K, V, q


def _oracle_attention(K, V, q, b_ids, h_ids, G):
    """Per-unit CPU attention over compressed stores (oracle), [len(b), len(h)*G, D]."""
    from oracle import packkv_oracle as O
    B_loc, H_loc = len(b_ids), len(h_ids)
    D = K.shape[-1]
    out = np.zeros((B_loc, H_loc * G, D), np.float32)
    for bi, b in enumerate(b_ids):
        st = O.OracleStore(1, H_loc, D)
        st.compress_batch(0, K[b][:, h_ids], V[b][:, h_ids])
        for hi in range(H_loc):
            for g in range(G):
                out[bi, hi * G + g] = O.attention_decode(st, 0, hi, q[b, h_ids[hi] * G + g])
    return out


def _worker(rank, world, port, B, H, G, D, T, prefer, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, V, q = _data(B, H, G, D, T)
        p = S.plan_partition(B, H, world, rank, prefer=prefer)
        b_ids = list(range(p.b0, p.b1))
        h_ids = list(range(p.h0, p.h1))
        dec = S.ShardedDecoder(p, lambda ql: torch.from_numpy(
            _oracle_attention(K, V, q, b_ids, h_ids, G)), H * G, D)
        ql = dec.local_q(torch.from_numpy(q))
        assert tuple(ql.shape) == (p.local_batch, p.local_heads * G, D)
        assert torch.equal(ql, torch.from_numpy(q)[p.b0:p.b1, p.h0 * G:p.h1 * G])
        out = dec.step(ql)
        # a caller-provided host output buffer receives the same gathered result
        host = torch.full((B * H * G * D,), float("nan"))
        assert dec.step(ql, out=host) is host
        assert torch.equal(host.view(out.shape), out)
        ret[rank] = out.numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prefer", ["head", "batch"])
def test_sharded_decode_matches_unsharded(prefer):
    B, H, G, D, T = 2, 4, 2, 32, 70
    world = 2
    mgr = mp.get_context("spawn").Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, B, H, G, D, T, prefer, ret), nprocs=world,
                       start_method="spawn", join=True)
    K, V, q = _data(B, H, G, D, T)
    full = _oracle_attention(K, V, q, list(range(B)), list(range(H)), G)
    for r in range(world):
        np.testing.assert_allclose(ret[r], full, rtol=0, atol=1e-6)


def test_plan_partition_rules():
    p = S.plan_partition(8, 8, 8, 3)
    assert p.mode == "head" and (p.h0, p.h1) == (3, 4) and (p.b0, p.b1) == (0, 8)
    p = S.plan_partition(8, 52, 8, 5)          # LLaMA-30B shape: heads don't divide -> batch split
    assert p.mode == "batch" and (p.b0, p.b1) == (5, 6) and p.local_heads == 52
    units = set()
    for r in range(4):
        units |= set(S.plan_partition(8, 52, 4, r).units())
    assert units == {(b, h) for b in range(8) for h in range(52)}
    with pytest.raises(Exception):
        S.plan_partition(3, 5, 2, 0)
    g = torch.arange(2 * 3 * 4 * 5, dtype=torch.float32).reshape(2, 3, 4, 5)   # [world, B, Hq_loc, D]
    p0 = S.plan_partition(3, 4, 2, 0, prefer="head")
    a = S.assemble(p0, g)
    assert a.shape == (3, 8, 5) and torch.equal(a[:, 4:], g[1])


def _codes_worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nsets, B, H, blk, D = 2, 3, 4, 64, 16
        full = torch.arange(nsets * B * 2 * H * blk * D, dtype=torch.int32).reshape(nsets, B, 2, H, blk, D)
        full = (full * 7919 % 65536 - 32768).to(torch.int16)
        p = S.plan_partition(B, H, world, rank, prefer="head")
        mine = full[:, :, :, p.h0:p.h1].contiguous()
        allc = S.gather_codes(mine, p, lambda t: S._all_gather(t, world))
        ret[rank] = bool(torch.equal(allc, full))
    finally:
        dist.destroy_process_group()


def test_sharded_repack_codes_exchange():
    """The code exchange behind kv-head-split repacking (sharding.compress_sharded):
    every rank reassembles all heads' codes in global head order."""
    world = 2
    mgr = mp.get_context("spawn").Manager()
    ret = mgr.dict()
    mp.start_processes(_codes_worker, args=(world, _free_port(), ret), nprocs=world, start_method="spawn",
                       join=True)
    assert all(ret[r] for r in range(world))
