"""Parity of the single-pass decode attention (attn_fused_kernel, §8 f1).

attention_decode as ONE launch: K decode, online softmax
and V decode block by block, per-warp partials merged in a fixed order.
Checked against the f64 oracle -- softmax(naive_k_scores / sqrt(d)) fed to
naive_v_output over the oracle's own compressed store (oracle/
packkv_oracle.py) -- with tolerance ||gpu - f64||_inf <= 1e-3 * ||f64||_inf
(SURVEY Appendix A #12), for G in {1..8}, residues straddling the 32-row
residue chunks, wide packs (scalar paths, blocks read in place), the
BASELINE config shapes on sampled sequences, and against the three-launch
path.  Every call asserts pkv_last_path() == PATH_SINGLE."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import packkv_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _mods():
    from paper_2512_24449_b200 import _native as N
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    from paper_2512_24449_b200.kv_store import CompressedStore
    return N, attention_decode_batched, CompressedStore


def _close(a, ref):
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(a - ref).max()
    assert err <= TOL * scale, f"max abs err {err:.3e} > {TOL} * {scale:.3e}"
    return err / scale


def _oracle_attention(ref, h, q):
    s = O.naive_k_scores(ref, 0, h, q).astype(np.float64) / math.sqrt(ref.head_dim)
    return O.naive_v_output(ref, 0, h, O.softmax64(s))


def _single(N, A, st, q, **kw):
    out = A(st, 0, q, single_pass=True, **kw)
    assert N.last_path() == N.PATH_SINGLE, "attention left the single-pass kernel"
    return out


@pytest.mark.parametrize("rels", [(0.1, 0.2), (0.02, 0.03)], ids=["paper_rel", "wide_packs"])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 5, 8])
def test_single_pass_vs_oracle(G, rels):
    N, A, CS = _mods()
    rng = np.random.default_rng(500 + G)
    B, H, D = 2, 2, 128
    for T in (64 * 9 + 45, 64 * 3, 31, 64 * 4 + 1):
        k = O.gen_gauss_outlier(rng, B * H * T, D, 4).reshape(B, H, T, D).transpose(0, 2, 1, 3).copy()
        v = O.gen_gauss_outlier(rng, B * H * T, D, 1).reshape(B, H, T, D).transpose(0, 2, 1, 3).copy()
        st = CS(1, H, D, batch=B, rel_scale_k=rels[0], rel_scale_v=rels[1])
        st.compress_batch(0, k, v)
        q = (rng.standard_normal((B, H * G, D)) * 3).astype(np.float32)
        out = _single(N, A, st, torch.from_numpy(q)).cpu().numpy()
        for b in range(B):
            ref = O.OracleStore(1, H, D, rel_k=rels[0], rel_v=rels[1])
            ref.compress_batch(0, k[b], v[b])
            for hq in range(H * G):
                _close(out[b, hq], _oracle_attention(ref, hq // G, q[b, hq]))


# (name, batch, kv heads, G, tokens, sampled sequences)
CONFIG_SHAPES = [
    ("B", 8, 8, 4, 8192, (0, 7)),
    ("E", 2, 8, 8, 16384, (1,)),
    ("D", 1, 52, 1, 2048, (0,)),
    ("C", 1, 40, 1, 2048, (0,)),
]


@pytest.mark.parametrize("r", [0, 33])
@pytest.mark.parametrize("cfg", CONFIG_SHAPES, ids=[c[0] for c in CONFIG_SHAPES])
def test_single_pass_config_shapes_vs_oracle(cfg, r):
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    name, B, H, G, T0, samples = cfg
    N, A, CS = _mods()
    T = T0 + r
    k = gauss_outlier((B, T, H, 128), seed=3 + r)
    v = gauss_outlier((B, T, H, 128), n_outlier=1, seed=10 + r)
    st = CS(1, H, 128, batch=B, max_tokens=T)
    st.compress_batch(0, k, v)
    g = torch.Generator(device="cuda")
    g.manual_seed(r)
    q = torch.randn((B, H * G, 128), device="cuda", generator=g) * 2
    out = _single(N, A, st, q).cpu().numpy()
    qh = q.cpu().numpy()
    for b in samples:
        ref = O.OracleStore(1, H, 128)
        ref.compress_batch(0, k[b].cpu().numpy(), v[b].cpu().numpy())
        heads = range(H) if H <= 8 else (0, 17, H - 1)
        for h in heads:
            for hq in (h * G, h * G + G - 1):
                _close(out[b, hq], _oracle_attention(ref, h, qh[b, hq]))


def test_single_pass_matches_three_launch_and_is_deterministic():
    """The single pass agrees with the three-launch path (scores written)
    within f32 accumulation (1e-5 relative) and is bit-identical run to run
    and across block-count headroom (nblocks larger than the store)."""
    N, A, CS = _mods()
    rng = np.random.default_rng(9)
    B, H, G, D, T = 3, 4, 4, 128, 64 * 50 + 17
    k = rng.standard_normal((B, T, H, D)).astype(np.float16)
    v = rng.standard_normal((B, T, H, D)).astype(np.float16)
    st = CS(1, H, D, batch=B)
    st.compress_batch(0, k, v)
    q = torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32) * 2).cuda()
    one = _single(N, A, st, q).clone()
    two = _single(N, A, st, q).clone()
    assert torch.equal(one, two)
    three = A(st, 0, q, single_pass=False)
    assert N.last_path() == N.PATH_FAST
    assert float((one - three).abs().max() / three.abs().max()) <= 1e-5
    st[0]._ensure(8)
    hr = _single(N, A, st, q, nblocks=st[0].nblk_h + 8)
    assert float((hr - three).abs().max() / three.abs().max()) <= 1e-5


def test_single_pass_softmax_edges():
    """One-token cache -> the V row (softmax of a singleton);
    identical K rows (uniform weights over the compressed rows); very large
    score spreads (one row dominates)."""
    N, A, CS = _mods()
    D = 128
    rng = np.random.default_rng(4)
    st = CS(1, 1, D)
    kv = rng.standard_normal((1, 1, D)).astype(np.float16)
    vv = rng.standard_normal((1, 1, D)).astype(np.float16)
    st.compress_batch(0, kv, vv)
    out = _single(N, A, st, torch.from_numpy(rng.standard_normal((1, 1, D)).astype(np.float32))).cpu().numpy()
    np.testing.assert_allclose(out[0, 0], vv[0, 0].astype(np.float32), rtol=1e-6, atol=1e-6)
    T = 64 * 6 + 5
    st = CS(1, 1, D)
    krow = rng.standard_normal(D).astype(np.float16)
    vv = rng.standard_normal((T, 1, D)).astype(np.float16)
    st.compress_batch(0, np.broadcast_to(krow, (T, 1, D)).copy(), vv)
    q = rng.standard_normal(D).astype(np.float32)
    out = _single(N, A, st, torch.from_numpy(q[None, None])).cpu().numpy()
    ref = O.OracleStore(1, 1, D)
    ref.compress_batch(0, np.broadcast_to(krow, (T, 1, D)).copy(), vv)
    # the compressed rows dequantize identically (the staged residue rows stay fp16)
    _close(out[0, 0], _oracle_attention(ref, 0, q))
    nb = 64 * (T // 64)
    s = O.naive_k_scores(ref, 0, 0, q)
    assert np.all(s[:nb] == s[0])
    # a score spread of ~1e3: exp underflows for almost every row
    T = 64 * 20 + 7
    kk = rng.standard_normal((T, 1, D)).astype(np.float16)
    vv = rng.standard_normal((T, 1, D)).astype(np.float16)
    st = CS(1, 1, D)
    st.compress_batch(0, kk, vv)
    ref = O.OracleStore(1, 1, D)
    ref.compress_batch(0, kk, vv)
    q = (rng.standard_normal(D) * 60).astype(np.float32)
    out = _single(N, A, st, torch.from_numpy(q[None, None])).cpu().numpy()
    _close(out[0, 0], _oracle_attention(ref, 0, q))


@pytest.mark.parametrize("seed", range(12))
def test_randomized_decode_loop(seed):
    """GraphedDecodeLoop (append-flush + attention per layer, one graph replay per
    step; either attention path) against eager append_token + attention on a
    twin store, over random batch / heads / groups / prefill / headroom and enough
    steps to cross block completions and a re-capture; streams byte-identical."""
    N, A, CS = _mods()
    from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop
    rng = np.random.default_rng(7000 + seed)
    B, H, G, Ly = int(rng.integers(1, 4)), int(rng.integers(1, 5)), int(rng.choice([1, 2, 4, 8])), int(rng.integers(1, 3))
    T0, steps, headroom = int(rng.integers(1, 200)), int(rng.integers(60, 140)), int(rng.integers(1, 3))
    D = 128
    k = (rng.standard_normal((Ly, B, T0 + steps, H, D)) * 2).astype(np.float16)
    v = rng.standard_normal((Ly, B, T0 + steps, H, D)).astype(np.float16)
    q = rng.standard_normal((steps, Ly, B, H * G, D)).astype(np.float32)
    a, r = CS(Ly, H, D, batch=B, check=False), CS(Ly, H, D, batch=B, check=False)
    for l in range(Ly):
        a.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
        r.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
    loop = GraphedDecodeLoop(a, H * G, headroom=headroom)
    loop.single_pass = bool(seed % 2)
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    worst = 0.0
    for t in range(steps):
        out = loop.step(kd[:, :, T0 + t:T0 + t + 1], vd[:, :, T0 + t:T0 + t + 1], qd[t]).clone()
        for l in range(Ly):
            r.append_token(l, kd[l, :, T0 + t], vd[l, :, T0 + t])
            ref = A(r, l, qd[t, l], single_pass=loop.single_pass)  # the same path (f32 order, digit scaling)
            worst = max(worst, float((out[l] - ref).abs().max() / ref.abs().max()))
    assert worst <= 1e-5, worst
    torch.cuda.synchronize()
    a.check_errors()
    for l in range(Ly):
        assert a[l].nblk_h == r[l].nblk_h and a[l].nres_h == r[l].nres_h
        for b in range(B):
            assert a[l].stream_bytes(b) == r[l].stream_bytes(b)


@pytest.mark.parametrize("single", [True, False])
def test_ragged_decode_loop(single):
    """A ragged decode batch: each step a random subset of the sequences appends
    its next token (GraphedDecodeLoop.step(active=...), pkv_append_flush_masked)
    and every sequence attends over its own history.  Each sequence must match
    a batch-1 store fed only its own tokens (eager append_token + attention),
    and its packed stream must be byte-identical to that store's."""
    N, A, CS = _mods()
    from paper_2512_24449_b200 import errors as E
    from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop
    rng = np.random.default_rng(31 + int(single))
    B, H, G, Ly, D = 3, 2, 4, 2, 128
    T0, steps = 50, 180
    k = rng.standard_normal((Ly, B, T0 + steps, H, D)).astype(np.float16)
    v = rng.standard_normal((Ly, B, T0 + steps, H, D)).astype(np.float16)
    q = rng.standard_normal((steps, Ly, B, H * G, D)).astype(np.float32)
    a = CS(Ly, H, D, batch=B, check=False)
    refs = [CS(Ly, H, D, batch=1, check=False) for _ in range(B)]
    for l in range(Ly):
        a.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
        for b in range(B):
            refs[b].compress_batch(l, k[l, b:b + 1, :T0], v[l, b:b + 1, :T0])
    loop = GraphedDecodeLoop(a, H * G, headroom=2)
    loop.single_pass = single
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    pos = np.full(B, T0)
    worst = 0.0
    for t in range(steps):
        act = rng.random(B) < 0.7
        act[t % B] = True if t < 3 else act[t % B]
        kin = torch.stack([kd[:, b, pos[b]] for b in range(B)], 1)[:, :, None]   # [Ly, B, 1, H, D]
        vin = torch.stack([vd[:, b, pos[b]] for b in range(B)], 1)[:, :, None]
        out = loop.step(kin, vin, qd[t], active=act).clone()
        for b in range(B):
            for l in range(Ly):
                if act[b]:
                    refs[b].append_token(l, kd[l, b, pos[b]][None], vd[l, b, pos[b]][None])
                ref = A(refs[b], l, qd[t, l, b][None], single_pass=single)[0]
                worst = max(worst, float((out[l, b] - ref).abs().max() / ref.abs().max()))
        pos += act
    assert worst <= 1e-5, worst
    torch.cuda.synchronize()
    a.check_errors()
    assert any(a[l].ragged for l in range(Ly)) and len(set(pos.tolist())) > 1
    for l in range(Ly):
        assert a[l].nblk.tolist() == [refs[b][l].nblk_h for b in range(B)]
        assert a[l].nres.tolist() == [refs[b][l].nres_h for b in range(B)]
        for b in range(B):
            assert a[l].stream_bytes(b) == refs[b][l].stream_bytes(0), f"layer {l} seq {b}"
    with pytest.raises(ValueError):  # eager appends need a lockstep batch
        a.append_token(0, kd[0, :, 0], vd[0, :, 0])
    with pytest.raises(E.StoreFormatError):
        from paper_2512_24449_b200.kv_store import save_store
        save_store(a, "/tmp/ragged.pkks")


def test_ragged_prefill_then_decode():
    """compress_batch(lengths=...) builds a ragged store (common prefix in
    lockstep, the rest as masked append steps); every sequence's stream, block
    table and attention equal a batch-1 store of its own tokens, then the
    decode loop keeps going from the ragged state."""
    N, A, CS = _mods()
    from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop
    rng = np.random.default_rng(12)
    B, H, G, D = 3, 2, 4, 128
    lens = np.array([100, 37, 200])
    T = 260
    k = rng.standard_normal((B, T, H, D)).astype(np.float16)
    v = rng.standard_normal((B, T, H, D)).astype(np.float16)
    st = CS(1, H, D, batch=B, check=False)
    st.compress_batch(0, k, v, lengths=lens)
    refs = [CS(1, H, D, batch=1, check=False) for _ in range(B)]
    for b in range(B):
        refs[b].compress_batch(0, k[b:b + 1, :lens[b]], v[b:b + 1, :lens[b]])
    assert st[0].ragged
    assert st[0].nblk.tolist() == [r[0].nblk_h for r in refs] and st[0].nres.tolist() == [r[0].nres_h for r in refs]
    q = rng.standard_normal((B, H * G, D)).astype(np.float32)
    out = A(st, 0, torch.from_numpy(q), single_pass=True).cpu().numpy()
    for b in range(B):
        assert st[0].stream_bytes(b) == refs[b][0].stream_bytes(0)
        ref = A(refs[b], 0, torch.from_numpy(q[b:b + 1]), single_pass=True).cpu().numpy()[0]
        _close(out[b], ref)
        assert len(st.iterate_blocks(0, 0, b)) == H * (lens[b] // 64) + 1  # every head's K blocks + the residue
    loop = GraphedDecodeLoop(st, H * G, headroom=2)
    pos = lens.copy()
    for t in range(40):
        kin = torch.from_numpy(np.stack([k[b, pos[b]] for b in range(B)])[None, :, None]).cuda()
        vin = torch.from_numpy(np.stack([v[b, pos[b]] for b in range(B)])[None, :, None]).cuda()
        qt = torch.from_numpy(rng.standard_normal((1, B, H * G, D)).astype(np.float32)).cuda()
        o = loop.step(kin, vin, qt).clone()
        for b in range(B):
            refs[b].append_token(0, torch.from_numpy(k[b, pos[b]][None]).cuda(), torch.from_numpy(v[b, pos[b]][None]).cuda())
            r = A(refs[b], 0, qt[0, b:b + 1], single_pass=loop.single_pass)[0]
            assert float((o[0, b] - r).abs().max() / r.abs().max()) <= 1e-5
        pos += 1
    for b in range(B):
        assert st[0].stream_bytes(b) == refs[b][0].stream_bytes(0)


@pytest.mark.parametrize("single", [True, False])
def test_decode_loop_host_output(single):
    """GraphedDecodeLoop.step(..., out=pinned host buffer): the attention kernels store
    every layer's output straight to host memory inside the graph.  Equal (bit for bit)
    to a twin loop writing its device buffer, across block completions and re-captures;
    switching back to device output re-captures."""
    N, A, CS = _mods()
    from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop
    rng = np.random.default_rng(77)
    B, H, G, Ly, D, T0, steps = 2, 2, 4, 2, 128, 100, 90
    k = rng.standard_normal((Ly, B, T0 + steps, H, D)).astype(np.float16)
    v = rng.standard_normal((Ly, B, T0 + steps, H, D)).astype(np.float16)
    q = rng.standard_normal((steps, Ly, B, H * G, D)).astype(np.float32)
    a, r = CS(Ly, H, D, batch=B, check=False), CS(Ly, H, D, batch=B, check=False)
    for l in range(Ly):
        a.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
        r.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
    la, lr = GraphedDecodeLoop(a, H * G, headroom=1), GraphedDecodeLoop(r, H * G, headroom=1)
    la.single_pass = lr.single_pass = single
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    host = torch.empty((Ly, B, H * G, D)).pin_memory()
    for t in range(steps):
        sl = slice(T0 + t, T0 + t + 1)
        got = la.step(kd[:, :, sl], vd[:, :, sl], qd[t], out=host)
        ref = lr.step(kd[:, :, sl], vd[:, :, sl], qd[t])
        torch.cuda.synchronize()
        assert got.data_ptr() == host.data_ptr()
        assert torch.equal(host, ref.cpu()), t
    caps = la.captures
    dev = la.step(kd[:, :, T0 + steps - 1:T0 + steps], vd[:, :, T0 + steps - 1:T0 + steps], qd[0])
    assert dev.is_cuda and la.captures == caps + 1
