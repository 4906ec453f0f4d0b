"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact: quantized codes, params, packed bytes, store streams, CR.
Tolerance: fused GEMV outputs, ||gpu - f64 oracle||_inf <= 1e-3 * ||f64||_inf
(SURVEY Appendix A #12)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import packkv_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _pk():
    import paper_2512_24449_b200 as pk
    from paper_2512_24449_b200 import bitpack_codec as C, fused_kernels as F, quantizer as Q
    from paper_2512_24449_b200.kv_store import CompressedStore
    return pk, C, F, Q, CompressedStore


def _close(a, ref):
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(a - ref).max() if ref.size else 0.0
    assert err <= TOL * scale, f"max abs err {err:.3e} > {TOL} * {scale:.3e}"
    return err / scale


# ------------------------------------------------------------------ quantizer
@pytest.mark.parametrize("rel", [0.05, 0.1, 0.2, 0.5, 1.0, 0.0123])
def test_quantize_bit_exact(rel):
    _, _, _, Q, _ = _pk()
    rng = np.random.default_rng(int(rel * 1000))
    x = (rng.standard_normal((40, 64, 128)) * rng.uniform(0.001, 50, (40, 64, 1))).astype(np.float16)
    x[0, 0, :] = 3.0                                     # constant row
    x[1, 0, :3] = [0, 0.25, 1]                           # tie trap
    qb = Q.quantize_token_wise(torch.from_numpy(x).cuda(), rel)
    q = qb.q.cpu().numpy().astype(np.int64)
    for i in range(40):
        r = O.quantize_token_wise(x[i], rel)
        assert np.array_equal(q[i], r.q), f"codes differ in block {i}"
        assert np.array_equal(qb.scale[i].cpu().numpy(), r.scale)
        assert np.array_equal(qb.zp[i].cpu().numpy(), r.zp)
    d = Q.dequantize(qb).cpu().numpy()
    for i in range(3):
        r = O.quantize_token_wise(x[i], rel)
        assert np.array_equal(d[i], O.dequantize(r.q, r.scale, r.zp))


def test_quantize_examples_and_errors():
    pk, _, _, Q, _ = _pk()
    qb = Q.quantize_token_wise(torch.tensor([[0.0, 0.34, 1.0]], dtype=torch.float16).cuda(), 0.1)
    assert qb.q.cpu().tolist() == [[0, 3, 10]]
    with pytest.raises(pk.errors.NonFiniteValueError):
        Q.quantize_token_wise(torch.tensor([[0.0, float("inf")]], dtype=torch.float16).cuda(), 0.1)
    assert Q.max_abs_error(torch.full((4, 8), 2.0, dtype=torch.float16).cuda(), 0.1) == 0.0


# ------------------------------------------------------------------ codec
def _rand_codes(rng, rows, cols, maxw):
    return rng.integers(0, 1 << maxw, (rows, cols)) if maxw else np.zeros((rows, cols), np.int64)


@pytest.mark.parametrize("k", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("layout", [0, 1])
def test_encode_bit_exact(k, layout):
    _, C, _, Q, _ = _pk()
    rng = np.random.default_rng(k * 10 + layout)
    for rows, cols in [(64, 128), (k, 5), (2 * k, 37), (128, 64)]:
        n = 6
        q = np.stack([_rand_codes(rng, rows, cols, int(rng.integers(0, 16))) for _ in range(n)])
        q[0] = 0
        q[1, 0, 0] = 32767                                # width 15
        scale = rng.uniform(0.01, 2, (n, rows)).astype(np.float32)
        zp = rng.uniform(-3, 3, (n, rows)).astype(np.float16).astype(np.float32)
        qb = Q.QuantBlock(torch.from_numpy(q.astype(np.int32)).to(torch.uint16).cuda(),
                          torch.from_numpy(scale).cuda(), torch.from_numpy(zp).cuda(), 0 if layout == 0 else 1)
        blocks = C.encode_blocks(qb, k, layout)
        for i in range(n):
            ref = O.encode_block(O.QuantBlock(q[i], scale[i], zp[i], qb.kind), k, layout, qb.kind)
            got = blocks[i].to_bytes()
            assert got == ref, f"block {i} ({rows}x{cols}) differs"
            assert C.compression_ratio(blocks[i]) == O.compression_ratio(ref)
        dec = C.decode_blocks([C.PackedBlock.from_bytes(
            O.encode_block(O.QuantBlock(q[i], scale[i], zp[i], 0), k, layout, 0)) for i in range(n)])
        assert np.array_equal(dec.q.cpu().numpy().astype(np.int64), q)
        pb = C.PackedBlock.from_bytes(O.encode_block(O.QuantBlock(q[2], scale[2], zp[2], 0), k, layout, 0))
        P = (rows // k) * cols
        for p in (0, P // 3, P - 1):
            assert np.array_equal(C.decode_pack_at(pb, p).cpu().numpy().astype(np.int64),
                                  O.decode_pack_at(pb.to_bytes(), p))


def test_decode_malformed():
    pk, C, _, _, _ = _pk()
    q = np.arange(64 * 8).reshape(64, 8) % 7
    good = O.encode_block(O.QuantBlock(q, np.ones(64, np.float32), np.zeros(64, np.float32)), 16)
    for bad in (good[:-1], good + b"\0", bytes([0, 0, 7]) + good[3:]):
        with pytest.raises(pk.errors.MalformedBlockError):
            C.decode_block(C.PackedBlock.from_bytes(bad))
    with pytest.raises(IndexError):
        C.decode_pack_at(C.PackedBlock.from_bytes(good), 10 ** 6)


def test_encode_width_overflow():
    pk, C, _, Q, _ = _pk()
    q = np.zeros((16, 4), np.int64)
    q[0, 0] = 65535
    qb = Q.QuantBlock(torch.from_numpy(q.astype(np.int32)).to(torch.uint16).cuda(),
                      torch.ones(16).cuda(), torch.zeros(16).cuda())
    with pytest.raises(pk.errors.WidthOverflowError):
        C.encode_block(qb, 16)


# ------------------------------------------------------------------ store
def _kv(rng, T, H, D, batch=None):
    shape = (T, H, D) if batch is None else (batch, T, H, D)
    return rng.standard_normal(shape).astype(np.float16), rng.standard_normal(shape).astype(np.float16)


@pytest.mark.parametrize("repack", ["none", "v_median", "greedy"])
@pytest.mark.parametrize("k", [8, 16])
def test_store_stream_bit_exact(repack, k):
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(1)
    H, D = 4, 64
    kk, vv = _kv(rng, 200, H, D)
    ref = O.OracleStore(1, H, D, pack_size=k, repack=repack)
    ref.compress_batch(0, kk, vv)
    st = CS(1, H, D, pack_size=k, repack=repack)
    st.compress_batch(0, kk[:70], vv[:70])
    st.compress_batch(0, kk[70:], vv[70:])
    assert st[0].stream_bytes(0) == ref.layer_stream(0)
    got = [(e.kind, e.head, e.token_start, e.byte_len, e.permutation.tolist()) for e in st[0].directory()]
    exp = [(e.kind, e.head, e.token_start, e.byte_len, e.permutation.tolist()) for e in ref.directory]
    assert got == exp
    assert st[0].nres_h == 200 - 3 * 64
    assert np.array_equal(st[0].stage[0, :, :st[0].nres_h].permute(1, 0, 2).cpu().numpy(), ref.stage_k[0])


def test_store_incremental_equals_batch_and_thresholds():
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(2)
    H, D = 2, 128
    kk, vv = _kv(rng, 300, H, D)
    a = CS(1, H, D)
    for t in range(63):
        a.append_token(0, kk[t], vv[t])
    assert a[0].nblk_h == 0 and a[0].nres_h == 63
    a.append_token(0, kk[63], vv[63])
    assert a[0].nblk_h == 1 and a[0].nres_h == 0
    for t in range(64, 300):
        a.append_token(0, kk[t], vv[t])
    b = CS(1, H, D)
    b.compress_batch(0, kk[:100], vv[:100])
    assert b[0].nblk_h == 1 and b[0].nres_h == 36
    b.compress_batch(0, kk[100:], vv[100:])
    assert a[0].stream_bytes(0) == b[0].stream_bytes(0)
    c = CS(1, H, D)
    c.compress_batch(0, kk[:0], vv[:0])
    assert c[0].tokens == 0


@pytest.mark.parametrize("repack", ["none", "v_median", "greedy"])
def test_store_default_format_fast_path(repack):
    """64 x 128, k = 16 runs the warp-per-block compressor (store_fast_*):
    batch > 1, staged residues across calls, repack permutations applied
    while re-quantizing from the f16 source, bit-exact against the oracle."""
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(11)
    B, H, D, T = 2, 3, 128, 64 * 5 + 17
    kk, vv = _kv(rng, T, H, D, batch=B)
    kk = (kk * rng.uniform(0.01, 30, (B, T, 1, 1))).astype(np.float16)
    st = CS(1, H, D, batch=B, repack=repack, rel_scale_k=0.03, rel_scale_v=0.07)
    for a, b in ((0, 30), (30, 31), (31, 200), (200, T)):
        st.compress_batch(0, kk[:, a:b], vv[:, a:b])
    for b in range(B):
        ref = O.OracleStore(1, H, D, repack=repack, rel_k=0.03, rel_v=0.07)
        ref.compress_batch(0, kk[b], vv[b])
        assert st[0].stream_bytes(b) == ref.layer_stream(0)
        got = [(e.kind, e.head, e.byte_len, e.permutation.tolist()) for e in st[0].directory() if e.seq == b]
        exp = [(e.kind, e.head, e.byte_len, e.permutation.tolist()) for e in ref.directory]
        assert got == exp


@pytest.mark.parametrize("rel", [(1.0, 0.5), (0.34, 0.2), (1 / 15.5, 1 / 16.5), (0.1, 0.2), (0.01, 0.003), (2e-4, 1e-3)])
def test_store_fast_buffer_bound(rel):
    """The compressor's per-warp assembly buffer is sized from rel (codes <= round(1/rel),
    store.cu fastc::buf_bytes); uniform data puts the full code range in nearly every pack,
    so blocks reach the bound's width, at the power-of-two edges (1/15.5, 1/16.5) too.
    Bytes equal the oracle's and no flag is raised."""
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(23)
    B, H, D, T = 2, 2, 128, 64 * 3 + 5
    kk = rng.uniform(-4, 4, (B, T, H, D)).astype(np.float16)
    vv = rng.uniform(-1, 3, (B, T, H, D)).astype(np.float16)
    st = CS(1, H, D, batch=B, rel_scale_k=rel[0], rel_scale_v=rel[1])
    st.compress_batch(0, kk, vv)
    for b in range(B):
        ref = O.OracleStore(1, H, D, rel_k=rel[0], rel_v=rel[1])
        ref.compress_batch(0, kk[b], vv[b])
        assert st[0].stream_bytes(b) == ref.layer_stream(0)


def test_store_default_format_errors():
    pk, _, _, _, CS = _pk()
    bad = np.zeros((70, 2, 128), np.float16)
    bad[65, 1, 7] = np.inf
    st = CS(1, 2, 128)
    with pytest.raises(pk.errors.NonFiniteValueError):
        st.compress_batch(0, bad, np.zeros_like(bad))
    # scale = rel * (max - min) above the f16 range -> WidthOverflowError
    big = np.zeros((64, 2, 128), np.float16)
    big[:, :, 0] = -60000
    big[:, :, 1] = 60000
    st = CS(1, 2, 128, rel_scale_k=1.0)
    with pytest.raises(pk.errors.WidthOverflowError):
        st.compress_batch(0, big, np.zeros_like(big))


def test_store_errors():
    pk, _, _, _, CS = _pk()
    st = CS(1, 2, 64)
    with pytest.raises(pk.errors.ShapeMismatchError):
        st.append_token(0, np.zeros(127, np.float16), np.zeros(128, np.float16))
    bad = np.zeros((2, 64), np.float16)
    bad[1, 3] = np.nan
    with pytest.raises(pk.errors.NonFiniteValueError):
        st.append_token(0, bad, np.zeros((2, 64), np.float16))
    with pytest.raises(IndexError):
        st.append_token(3, np.zeros((2, 64), np.float16), np.zeros((2, 64), np.float16))


def test_store_growth():
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(3)
    H, D = 2, 64
    kk, vv = _kv(rng, 1000, H, D)
    st = CS(1, H, D, max_tokens=64)
    for i in range(0, 1000, 130):
        st.compress_batch(0, kk[i:i + 130], vv[i:i + 130])
    ref = O.OracleStore(1, H, D)
    ref.compress_batch(0, kk, vv)
    assert st[0].stream_bytes(0) == ref.layer_stream(0)


# ------------------------------------------------------------------ fused
def _oracle_per_seq(kk, vv, H, D, k, repack="none"):
    ref = O.OracleStore(1, H, D, pack_size=k, repack=repack)
    ref.compress_batch(0, kk, vv)
    return ref


@pytest.mark.parametrize("k", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("D", [64, 128])
def test_fused_vs_oracle(k, D):
    _, _, F, _, CS = _pk()
    rng = np.random.default_rng(k + D)
    H, T = 2, 64 * 5 + 17
    kk, vv = _kv(rng, T, H, D)
    ref = _oracle_per_seq(kk, vv, H, D, k)
    st = CS(1, H, D, pack_size=k)
    st.compress_batch(0, kk, vv)
    for G in (1, 4, 8):
        q = rng.standard_normal((1, H * G, D)).astype(np.float32)
        w = rng.random((1, H * G, T)).astype(np.float32)
        s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
        o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
        for hq in range(H * G):
            _close(s[0, hq], O.naive_k_scores(ref, 0, hq // G, q[0, hq]))
            _close(o[0, hq], O.naive_v_output(ref, 0, hq // G, w[0, hq]))


def test_fused_spec_api_and_token_map():
    _, _, F, _, CS = _pk()
    rng = np.random.default_rng(5)
    H, D, T = 2, 128, 150
    kk, vv = _kv(rng, T, H, D)
    ref = _oracle_per_seq(kk, vv, H, D, 16, "v_median")
    st = CS(1, H, D, repack="v_median")
    st.compress_batch(0, kk, vv)
    q = rng.standard_normal(D).astype(np.float32)
    sv = F.fused_k_scores(st, 0, 1, q)
    rs, rmap = O.fused_k_scores(ref, 0, 1, q)
    _close(sv.scores.cpu().numpy(), rs)
    assert np.array_equal(sv.token_map.cpu().numpy(), rmap)
    e = np.zeros(D, np.float32)
    e[7] = 1
    col = F.fused_k_scores(st, 0, 0, e).scores.cpu().numpy()
    _close(col, O.fused_k_scores(ref, 0, 0, e)[0])
    w = np.zeros(T, np.float32)
    w[70] = 1
    _close(F.fused_v_output(st, 0, 0, w).cpu().numpy(), O.fused_v_output(ref, 0, 0, w))
    assert np.all(F.fused_v_output(st, 0, 1, np.zeros(T, np.float32)).cpu().numpy() == 0)
    assert np.all(F.fused_k_scores(st, 0, 1, np.zeros(D, np.float32)).scores.cpu().numpy() == 0)


def test_fused_batched_gqa_ragged_residue():
    _, _, F, _, CS = _pk()
    rng = np.random.default_rng(6)
    B, H, D, G = 3, 2, 128, 4
    T = 64 * 3 + 5
    kk, vv = _kv(rng, T, H, D, batch=B)
    st = CS(1, H, D, batch=B)
    st.compress_batch(0, kk[:, :40], vv[:, :40])
    st.compress_batch(0, kk[:, 40:], vv[:, 40:])
    q = rng.standard_normal((B, H * G, D)).astype(np.float32)
    w = rng.random((B, H * G, T)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
    for b in range(B):
        ref = _oracle_per_seq(kk[b], vv[b], H, D, 16)
        assert st[0].stream_bytes(b) == ref.layer_stream(0)
        for hq in range(H * G):
            _close(s[b, hq], O.naive_k_scores(ref, 0, hq // G, q[b, hq]))
            _close(o[b, hq], O.naive_v_output(ref, 0, hq // G, w[b, hq]))


def test_fused_v_deterministic_and_linear():
    _, _, F, _, CS = _pk()
    rng = np.random.default_rng(7)
    H, D, T = 2, 128, 64 * 40 + 3
    kk, vv = _kv(rng, T, H, D)
    st = CS(1, H, D)
    st.compress_batch(0, kk, vv)
    w = torch.rand((1, H * 4, T)).cuda()
    a = F.fused_v_output_batched(st, 0, w).clone()
    b = F.fused_v_output_batched(st, 0, w)
    assert torch.equal(a, b)
    q1, q2 = torch.randn((2, 1, H * 4, D)).cuda()
    s12 = F.fused_k_scores_batched(st, 0, q1 + q2)
    s1 = F.fused_k_scores_batched(st, 0, q1).clone() + F.fused_k_scores_batched(st, 0, q2)
    assert (s12 - s1).abs().max() <= TOL * s12.abs().max()


def test_fused_large_property():
    """Large context through the size-independent property: fused == GPU
    decode-then-f64-GEMV (naive) on the same store (config-B-like unit)."""
    _, _, F, _, CS = _pk()
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    H, D, G, T = 2, 128, 4, 32768 + 21
    kk = gauss_outlier((1, T, H, D), seed=1)
    vv = gauss_outlier((1, T, H, D), n_outlier=1, seed=2)
    st = CS(1, H, D, max_tokens=T)
    st.compress_batch(0, kk, vv)
    q = torch.randn((1, H * G, D), device="cuda")
    w = torch.softmax(torch.randn((1, H * G, T), device="cuda"), -1)
    s = F.fused_k_scores_batched(st, 0, q)
    o = F.fused_v_output_batched(st, 0, w)
    Kd = F.decode_layer(st, 0, 0).double()          # [H, L, D]
    Vd = F.decode_layer(st, 0, 1).double()
    for hq in range(H * G):
        rk = Kd[hq // G] @ q[0, hq].double()
        rv = w[0, hq].double() @ Vd[hq // G]
        assert (s[0, hq].double() - rk).abs().max() <= TOL * rk.abs().max()
        assert (o[0, hq].double() - rv).abs().max() <= TOL * rv.abs().max()
    # quantization error of the dequantized cache stays within the SPEC bound
    k32 = kk[0].permute(1, 0, 2).float()
    tm = F.token_map(st, 0)[0]
    err = (Kd.float() - k32[:, tm]).abs()
    rng_row = k32.amax(-1) - k32.amin(-1)
    # f32-scale codes dequantized with the f16 wire scale: + range * 2^-10 slack
    assert bool((err <= (0.1 / 2 + 2 ** -10) * rng_row[:, tm, None] + 2 ** -10).all())


def test_attention_decode_singleton():
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import attention_decode
    rng = np.random.default_rng(9)
    st = CS(1, 2, 64)
    k, v = _kv(rng, 1, 2, 64)
    st.compress_batch(0, k, v)
    out = attention_decode(st, 0, 1, rng.standard_normal(64)).cpu().numpy()
    assert np.allclose(out, v[0, 1].astype(np.float32))


@pytest.mark.parametrize("rels", [(0.1, 0.2), (0.02, 0.05), (0.0004, 0.01)])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 6, 8])
def test_fused_default_format_paths(rels, G):
    """k=16, D=128 runs the tensor-core kernels; wide packs (w > 5) and codes
    above 2047 exercise their in-launch scalar path."""
    _, _, F, _, CS = _pk()
    rng = np.random.default_rng(int(G * 100 + rels[0] * 1e4))
    H, D, T = 3, 128, 64 * 7 + 9
    kk = (rng.standard_normal((T, H, D)) * rng.uniform(0.1, 4, (T, 1, 1))).astype(np.float16)
    vv = rng.standard_normal((T, H, D)).astype(np.float16)
    ref = O.OracleStore(1, H, D, rel_k=rels[0], rel_v=rels[1])
    ref.compress_batch(0, kk, vv)
    st = CS(1, H, D, rel_scale_k=rels[0], rel_scale_v=rels[1])
    st.compress_batch(0, kk[:100], vv[:100])
    st.compress_batch(0, kk[100:], vv[100:])
    assert st[0].stream_bytes(0) == ref.layer_stream(0)
    q = rng.standard_normal((1, H * G, D)).astype(np.float32)
    w = rng.standard_normal((1, H * G, T)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
    for hq in range(H * G):
        _close(s[0, hq], O.naive_k_scores(ref, 0, hq // G, q[0, hq]))
        _close(o[0, hq], O.naive_v_output(ref, 0, hq // G, w[0, hq]))


def test_graphed_attention_matches_eager_and_recaptures():
    """attention_sim.GraphedAttention (one CUDA-graph launch per decode step)
    is bit-identical to the eager composition and re-captures after appends
    change the block / residue counts."""
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import GraphedAttention, attention_decode_batched
    rng = np.random.default_rng(21)
    B, H, D, G = 2, 2, 128, 4
    st = CS(1, H, D, batch=B)
    k = (rng.standard_normal((B, 200, H, D))).astype(np.float16)
    v = (rng.standard_normal((B, 200, H, D))).astype(np.float16)
    st.compress_batch(0, k, v)
    ga = GraphedAttention(st, 0)
    for step in range(3):
        q = torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32)).cuda()
        a = ga(q).clone()
        e = attention_decode_batched(st, 0, q)
        assert torch.equal(a, e)
        kn = rng.standard_normal((B, 40, H, D)).astype(np.float16)
        vn = rng.standard_normal((B, 40, H, D)).astype(np.float16)
        st.compress_batch(0, kn, vn)  # 200 -> 240 -> 280: residue and block counts change
    # a host (pinned) query is copied straight into the graph's buffer
    qh = torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32)).pin_memory()
    ga(qh.cuda())
    assert torch.equal(ga(qh).clone(), attention_decode_batched(st, 0, qh.cuda()))
    # single-token appends that only stage (280 -> 283, 4 blocks + 24..27
    # staged): the same graph replays, the kernels read the residue length
    # from the device
    q = torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32)).cuda()
    ga(q)
    g0 = ga._graph
    for t in range(3):
        st.append_token(0, rng.standard_normal((B, H, D)).astype(np.float16),
                        rng.standard_normal((B, H, D)).astype(np.float16))
        a = ga(q).clone()
        assert ga._graph is g0
        assert torch.equal(a, attention_decode_batched(st, 0, q))
    torch.cuda.synchronize()


@pytest.mark.parametrize("rels", [(0.1, 0.2), (0.0004, 0.01)])
@pytest.mark.parametrize("G", [1, 3, 4, 5, 8])
def test_fused_attention_decode_vs_oracle(rels, G):
    """pkv_attention_decode (softmax folded into the fused K / V launches) against
    the f64 oracle softmax(K q / sqrt(d)) V over the dequantized store, with a
    residue and, at the small rel, wide packs (scalar path, blocks read in place)."""
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    rng = np.random.default_rng(33 + G)
    B, H, D, T = 2, 2, 128, 64 * 6 + 23
    k = O.gen_gauss_outlier(rng, B * H * T, D, 4).reshape(B, H, T, D).transpose(0, 2, 1, 3).copy()
    v = O.gen_gauss_outlier(rng, B * H * T, D, 1).reshape(B, H, T, D).transpose(0, 2, 1, 3).copy()
    st = CS(1, H, D, batch=B, rel_scale_k=rels[0], rel_scale_v=rels[1])
    st.compress_batch(0, k, v)
    q = rng.standard_normal((B, H * G, D)).astype(np.float32) * 3
    out = attention_decode_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    assert st[0].a_scratch.numel() > 0, "fused attention path not taken"
    F = __import__("paper_2512_24449_b200.fused_kernels", fromlist=["decode_layer"])
    Kd = F.decode_layer(st, 0, 0).double().cpu().numpy()  # [B*H, L, D] score order
    Vd = F.decode_layer(st, 0, 1).double().cpu().numpy()
    for b in range(B):
        for hq in range(H * G):
            u = b * H + hq // G
            s = Kd[u] @ q[b, hq].astype(np.float64) / np.sqrt(D)
            p = np.exp(s - s.max())
            ref = (p / p.sum()) @ Vd[u]
            _close(out[b, hq], ref)


def test_graphed_decode_step_matches_eager():
    """attention_sim.GraphedDecodeStep (stage token + attention in one graph,
    eager compressor on block completion) against append_token +
    attention_decode_batched on a twin store: identical outputs every step and
    identical streams, across two block completions."""
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import GraphedDecodeStep, attention_decode_batched
    rng = np.random.default_rng(23)
    B, H, D, G = 2, 2, 128, 4
    k0, v0 = _kv(rng, 100, H, D, batch=B)
    a, b = CS(1, H, D, batch=B), CS(1, H, D, batch=B)
    a.compress_batch(0, k0, v0)
    b.compress_batch(0, k0, v0)
    step = GraphedDecodeStep(a, 0)
    for t in range(100):
        kt = torch.from_numpy(rng.standard_normal((B, H, D)).astype(np.float16)).cuda()
        vt = torch.from_numpy(rng.standard_normal((B, H, D)).astype(np.float16)).cuda()
        q = torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32)).cuda()
        got = step(kt, vt, q).clone()
        b.append_token(0, kt, vt)
        assert torch.equal(got, attention_decode_batched(b, 0, q)), f"step {t}"
    # in-place inputs: write the token / query into the graph's own buffers
    kb, vb, qb = step.inputs(H * G)
    for t in range(3):
        kt = torch.from_numpy(rng.standard_normal((B, H, D)).astype(np.float16)).cuda()
        vt = torch.from_numpy(rng.standard_normal((B, H, D)).astype(np.float16)).cuda()
        q = torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32)).cuda()
        kb.copy_(kt.view_as(kb))
        vb.copy_(vt.view_as(vb))
        qb.copy_(q)
        got = step(kb, vb, qb).clone()
        b.append_token(0, kt, vt)
        assert torch.equal(got, attention_decode_batched(b, 0, q)), f"in-place step {t}"
    assert a[0].nblk_h == b[0].nblk_h == 3 and a[0].nres_h == b[0].nres_h == 11
    assert int(a[0].nres[0].item()) == 11
    for s in range(B):
        assert a[0].stream_bytes(s) == b[0].stream_bytes(s)
    assert torch.equal(a[0].stage[:, :, :11], b[0].stage[:, :, :11])


@pytest.mark.parametrize("repack", ["v_median", "greedy"])
def test_sharded_repack_plan_matches_single_device(repack):
    """kv-head split with repacking: two simulated ranks holding
    heads {0,1} and {2,3} exchange codes, compute the shared plan and produce
    exactly the blocks (bytes and permutations) of one store holding all 4."""
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200 import sharding as S
    rng = np.random.default_rng(31)
    B, H, D, T, W = 2, 4, 128, 64 * 3 + 20, 2
    kk, vv = _kv(rng, T, H, D, batch=B)
    full = CS(1, H, D, batch=B, repack=repack)
    parts = [S.plan_partition(B, H, W, r) for r in range(W)]
    local = [CS(1, p.local_heads, D, batch=B, repack=repack) for p in parts]
    for a, b in ((0, 70), (70, 150), (150, T)):
        full.compress_batch(0, kk[:, a:b], vv[:, a:b])
        ks = [np.ascontiguousarray(kk[:, a:b, p.h0:p.h1]) for p in parts]
        vs = [np.ascontiguousarray(vv[:, a:b, p.h0:p.h1]) for p in parts]
        codes = []
        for st, k1, v1 in zip(local, ks, vs):
            c = st[0].pending_codes(st._norm(k1, True), st._norm(v1, True))
            codes.append(None if c is None else c.view(torch.uint8))
        for st, p, k1, v1 in zip(local, parts, ks, vs):
            S.compress_sharded(st, p, 0, k1, v1, all_gather=lambda t: torch.stack(codes))
    fe = {(e.seq, e.kind, e.head, e.token_start): e for e in full[0].directory()}
    n = 0
    for st, p in zip(local, parts):
        for e in st[0].directory():
            g = fe[(e.seq, e.kind, e.head + p.h0, e.token_start)]
            assert st[0].block_bytes(e) == full[0].block_bytes(g)
            assert np.array_equal(e.permutation, g.permutation)
            n += 1
    assert n == len(fe) == 3 * B * 2 * H


@pytest.mark.parametrize("repack", ["none", "v_median"])
def test_pkks_store_file_matches_oracle_and_round_trips(repack, tmp_path):
    """The "PKKS" store file: the GPU store's file is byte-identical
    to the oracle's for the same tokens; load -> save is bit-exact; a loaded
    store attends bit-identically; the oracle reads the GPU's file."""
    pk, _, _, _, CS = _pk()
    from paper_2512_24449_b200.kv_store import load_store, save_store
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    rng = np.random.default_rng(41)
    H, D, T = 2, 128, 64 * 3 + 10
    kk, vv = _kv(rng, T, H, D)
    ref = O.OracleStore(2, H, D, repack=repack)
    st = CS(2, H, D, repack=repack)
    for layer in range(2):
        ref.compress_batch(layer, kk[:T - 40 * layer], vv[:T - 40 * layer])
        st.compress_batch(layer, kk[:T - 40 * layer], vv[:T - 40 * layer])
    save_store(st, tmp_path / "g.pkks")
    O.save_pkks(ref, tmp_path / "o.pkks")
    assert (tmp_path / "g.pkks").read_bytes() == (tmp_path / "o.pkks").read_bytes()
    ld = load_store(tmp_path / "o.pkks")
    save_store(ld, tmp_path / "g2.pkks")
    assert (tmp_path / "g2.pkks").read_bytes() == (tmp_path / "g.pkks").read_bytes()
    q = torch.from_numpy(rng.standard_normal((1, 4 * H, D)).astype(np.float32)).cuda()
    for layer in range(2):
        assert torch.equal(attention_decode_batched(ld, layer, q), attention_decode_batched(st, layer, q))
    back = O.load_pkks(tmp_path / "g.pkks")
    for layer in range(2):
        assert back.layer_stream(layer) == ref.layer_stream(layer)
    # appends continue identically after a load
    kn, vn = _kv(rng, 70, H, D)
    ld.compress_batch(0, kn, vn)
    st.compress_batch(0, kn, vn)
    assert ld[0].stream_bytes(0) == st[0].stream_bytes(0)
    data = (tmp_path / "g.pkks").read_bytes()
    for bad in (b"XKKS" + data[4:], data[:-3], data + b"\0"):
        (tmp_path / "bad.pkks").write_bytes(bad)
        with pytest.raises(pk.errors.StoreFormatError):
            load_store(tmp_path / "bad.pkks")


def test_pkks_batched_round_trip(tmp_path):
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200.kv_store import load_store, save_store
    rng = np.random.default_rng(43)
    B, H, D = 3, 2, 128
    kk, vv = _kv(rng, 150, H, D, batch=B)
    st = CS(1, H, D, batch=B, repack="greedy")
    st.compress_batch(0, kk, vv)
    save_store(st, tmp_path / "a.pkks")
    ld = load_store(tmp_path / "a.pkks")
    save_store(ld, tmp_path / "b.pkks")
    assert (tmp_path / "a.pkks").read_bytes() == (tmp_path / "b.pkks").read_bytes()
    for b in range(B):
        assert ld[0].stream_bytes(b) == st[0].stream_bytes(b)


def test_store_multi_chunk_prefill_equals_incremental():
    """A prefill larger than one compressor chunk (the scan keeps <= 12224 block
    sizes in shared memory: 38 block-sets at B=4, H=40) equals the same tokens
    appended in single-chunk calls (SPEC.md:374-382 batch/incremental identity)."""
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(51)
    B, H, D, T = 4, 40, 128, 64 * 45 + 7
    kk, vv = _kv(rng, T, H, D, batch=B)
    a, b = CS(1, H, D, batch=B), CS(1, H, D, batch=B)
    a.compress_batch(0, kk, vv)
    for s0 in range(0, T, 64 * 10 + 3):
        b.compress_batch(0, kk[:, s0:s0 + 64 * 10 + 3], vv[:, s0:s0 + 64 * 10 + 3])
    assert a[0].nblk_h == b[0].nblk_h == 45
    for s in range(B):
        assert a[0].stream_bytes(s) == b[0].stream_bytes(s)


@pytest.mark.parametrize("T", [1, 5, 63, 64, 65, 128])
def test_fused_default_format_block_boundaries(T):
    """Residue-only stores, exact block multiples and one token past them on the
    default-format kernels (fused K / V and the folded-softmax attention)."""
    _, _, F, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    rng = np.random.default_rng(60 + T)
    B, H, D, G = 2, 2, 128, 4
    st = CS(1, H, D, batch=B)
    kk, vv = _kv(rng, T, H, D, batch=B)
    st.compress_batch(0, kk, vv)
    q = rng.standard_normal((B, H * G, D)).astype(np.float32)
    w = rng.random((B, H * G, T)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
    a = attention_decode_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    for b in range(B):
        ref = _oracle_per_seq(kk[b], vv[b], H, D, 16)
        for hq in range(H * G):
            rs = O.naive_k_scores(ref, 0, hq // G, q[b, hq])
            _close(s[b, hq], rs)
            _close(o[b, hq], O.naive_v_output(ref, 0, hq // G, w[b, hq]))
            p = np.exp(rs / np.sqrt(D) - (rs / np.sqrt(D)).max())
            _close(a[b, hq], O.naive_v_output(ref, 0, hq // G, (p / p.sum()).astype(np.float64)))


def test_fused_many_heads_config_d_shape():
    """52 kv-heads (the LLaMA-30B shape of config D), MHA, ragged residue."""
    _, _, F, _, CS = _pk()
    rng = np.random.default_rng(71)
    H, D, T = 52, 128, 64 * 2 + 9
    kk, vv = _kv(rng, T, H, D)
    ref = O.OracleStore(1, H, D)
    ref.compress_batch(0, kk, vv)
    st = CS(1, H, D)
    st.compress_batch(0, kk, vv)
    assert st[0].stream_bytes(0) == ref.layer_stream(0)
    q = rng.standard_normal((1, H, D)).astype(np.float32)
    w = rng.random((1, H, T)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
    for h in range(0, H, 7):
        _close(s[0, h], O.naive_k_scores(ref, 0, h, q[0, h]))
        _close(o[0, h], O.naive_v_output(ref, 0, h, w[0, h]))


def test_store_shrink_to_fit_keeps_bytes_and_appends():
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(81)
    H, D = 2, 128
    kk, vv = _kv(rng, 400, H, D)
    a, b = CS(1, H, D, max_tokens=64), CS(1, H, D)
    a.compress_batch(0, kk[:300], vv[:300])
    b.compress_batch(0, kk[:300], vv[:300])
    cap0 = a[0].capacity
    a.shrink_to_fit()
    assert a[0].capacity <= cap0 and a[0].capacity >= int(a[0].tail.item())
    assert a[0].stream_bytes(0) == b[0].stream_bytes(0)
    a.compress_batch(0, kk[300:], vv[300:])
    b.compress_batch(0, kk[300:], vv[300:])
    assert a[0].stream_bytes(0) == b[0].stream_bytes(0)


# ------------------------------------------------------------------ repacker
def test_repacker_spec_examples():
    """SPEC.md:196,205,214-216 through the GPU plan kernel."""
    from paper_2512_24449_b200 import repacker as R
    assert R.pack_cost(np.array([[0, 5], [3, 1]])) == 50
    p = R.repack_greedy(np.array([[0], [9], [0], [9]]), 2)
    assert p.cost_bits == 40 and sorted(p.permutation.tolist()) == [0, 1, 2, 3]
    v = np.array([[5], [1], [3]])
    assert R.repack_v_median(v, v, 2).permutation.tolist() == [1, 2, 0]
    v = np.array([[2], [2], [1]])
    assert R.repack_v_median(v, v, 2).permutation.tolist() == [2, 0, 1]
    assert R.repack_none(v, 2).permutation.tolist() == [0, 1, 2]


@pytest.mark.parametrize("n,d,k", [(8, 6, 4), (37, 50, 8), (64, 256, 16), (64, 2048, 16), (20, 9, 16), (5, 3, 2)])
def test_repacker_matches_oracle(n, d, k):
    """Greedy and v_median plans (permutation and cost) equal the oracle's, partial
    last groups and K+V vectors longer than one kernel head included."""
    from paper_2512_24449_b200 import repacker as R
    rng = np.random.default_rng(n * 1000 + d + k)
    X = rng.integers(0, 12, (n, d)) + (rng.integers(0, 3, (n, 1)) * 7)
    g = R.repack_greedy(X, k)
    og = O.repack_greedy(X, k)
    assert g.permutation.tolist() == og.permutation.tolist()
    assert g.cost_bits == og.cost_bits
    vp = X[:, d // 2:]
    m = R.repack_v_median(X, vp, k)
    om = O.repack_v_median(X, vp, k)
    assert m.permutation.tolist() == om.permutation.tolist() and m.cost_bits == om.cost_bits
    assert R.plan_cost(X, g.permutation, k) <= R.plan_cost(X, np.arange(n), k) or n <= k


def test_generate_synthetic_profiles():
    """determinism per seed; channel-banded packs have smaller
    per-pack code ranges than uniform at equal amplitude."""
    from paper_2512_24449_b200 import tensor_model as TM
    from paper_2512_24449_b200.quantizer import quantize_token_wise
    for mode in TM.SYNTH_MODES:
        k1, v1 = TM.generate_synthetic(mode, 7, 2, 3, 128, 64)
        k2, v2 = TM.generate_synthetic(mode, 7, 2, 3, 128, 64)
        assert k1.shape == (2, 3, 64, 128) and torch.equal(k1, k2) and torch.equal(v1, v2)
        assert torch.isfinite(k1.float()).all()
    ranges = {}
    for mode in ("uniform", "channel-banded"):
        k, _ = TM.generate_synthetic(mode, 3, 1, 4, 128, 128)
        q = quantize_token_wise(k.reshape(-1, 64, 128), 0.1).q.long().reshape(-1, 16, 128)
        ranges[mode] = float((q.max(1).values - q.min(1).values).float().mean())
    assert ranges["channel-banded"] < ranges["uniform"]


def test_permutation_invariance_check():
    """SPEC.md:537-545 (+ repacking neutrality)."""
    from paper_2512_24449_b200.attention_sim import permutation_invariance_check
    rng = np.random.default_rng(91)
    K = rng.standard_normal((64 * 3 + 5, 128)).astype(np.float16)
    V = rng.standard_normal((64 * 3 + 5, 128)).astype(np.float16)
    rep = permutation_invariance_check(K, V, rng.standard_normal(128), trials=20)
    assert rep["pass"], rep
    assert rep["f64_failures"] == 0


def test_snapshot_stats_width_histogram():
    """exact bytes, CR and the pack-width histogram per (layer, kind)."""
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(93)
    H, D = 2, 128
    kk, vv = _kv(rng, 64 * 3 + 10, H, D)
    st = CS(1, H, D)
    st.compress_batch(0, kk, vv)
    ref = O.OracleStore(1, H, D)
    ref.compress_batch(0, kk, vv)
    stats = st.snapshot_stats()
    for kind in (0, 1):
        ents = [e for e in ref.directory if e.kind == kind]
        hist = np.zeros(16, np.int64)
        for e in ents:
            b = ref.block_bytes(e)
            P = 4 * 128
            nib = np.frombuffer(b[8:8 + P // 2], np.uint8)
            hist += np.bincount(np.stack([nib & 15, nib >> 4], 1).ravel(), minlength=16)
        s = stats[(0, kind)]
        assert s["width_hist"] == hist.tolist()
        assert s["bytes_physical"] == sum(e.byte_len for e in ents) and s["blocks"] == len(ents)
    empty = CS(1, H, D).snapshot_stats()
    assert empty[(0, 0)]["cr"] is None and empty[(0, 0)]["width_hist"] == [0] * 16


@pytest.mark.parametrize("seed", range(48))
def test_randomized_end_to_end_parity(seed):
    """Seeded random shapes / codec settings through the whole path: compressor
    (split appends, repack strategy), streams bit-exact per sequence, fused K, V
    and attention within the 1e-3 bar."""
    _, _, F, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 4))
    H = int(rng.integers(1, 5))
    G = int(rng.choice([1, 2, 4, 8]))
    T = int(rng.integers(1, 64 * 5))
    rel_k = float(rng.choice([0.05, 0.1, 0.2]))
    rel_v = float(rng.choice([0.1, 0.2, 0.3]))
    repack = str(rng.choice(["none", "v_median", "greedy"]))
    D = 128
    kk = (rng.standard_normal((B, T, H, D)) * rng.uniform(0.2, 5, (B, T, 1, 1))).astype(np.float16)
    vv = rng.standard_normal((B, T, H, D)).astype(np.float16)
    st = CS(1, H, D, batch=B, rel_scale_k=rel_k, rel_scale_v=rel_v, repack=repack)
    cut = int(rng.integers(0, T + 1))
    st.compress_batch(0, kk[:, :cut], vv[:, :cut])
    for t in range(cut, min(T, cut + 3)):
        st.append_token(0, kk[:, t], vv[:, t])
    if cut + 3 < T:
        st.compress_batch(0, kk[:, cut + 3:], vv[:, cut + 3:])
    q = rng.standard_normal((B, H * G, D)).astype(np.float32)
    w = rng.random((B, H * G, T)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
    a = attention_decode_batched(st, 0, torch.from_numpy(q), single_pass=True).cpu().numpy()
    a3 = attention_decode_batched(st, 0, torch.from_numpy(q), single_pass=False).cpu().numpy()
    for b in range(B):
        ref = O.OracleStore(1, H, D, rel_k=rel_k, rel_v=rel_v, repack=repack)
        ref.compress_batch(0, kk[b], vv[b])
        assert st[0].stream_bytes(b) == ref.layer_stream(0)
        for hq in range(H * G):
            rs = O.naive_k_scores(ref, 0, hq // G, q[b, hq])
            _close(s[b, hq], rs)
            _close(o[b, hq], O.naive_v_output(ref, 0, hq // G, w[b, hq]))
            x = rs / np.sqrt(D)
            p = np.exp(x - x.max())
            ra = O.naive_v_output(ref, 0, hq // G, p / p.sum())
            _close(a[b, hq], ra)   # single pass
            _close(a3[b, hq], ra)  # three launches


@pytest.mark.parametrize("seed", range(24))
def test_randomized_generic_formats_parity(seed):
    """Seeded random pack sizes / head dims (the generic kernels) and the default
    format, with a decode loop through GraphedDecodeStep: streams bit-exact,
    fused K, V and attention within the 1e-3 bar."""
    _, _, F, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import GraphedDecodeStep, attention_decode_batched
    rng = np.random.default_rng(5000 + seed)
    k = int(rng.choice([2, 4, 8, 16, 32]))
    D = int(rng.choice([64, 128, 256]))
    B = int(rng.integers(1, 3))
    H = int(rng.integers(1, 4))
    G = int(rng.choice([1, 2, 4]))
    T = int(rng.integers(1, 64 * 3))
    repack = str(rng.choice(["none", "v_median"]))
    kk = (rng.standard_normal((B, T, H, D)) * rng.uniform(0.2, 3, (B, T, 1, 1))).astype(np.float16)
    vv = rng.standard_normal((B, T, H, D)).astype(np.float16)
    st = CS(1, H, D, batch=B, pack_size=k, repack=repack)
    t0 = int(rng.integers(0, T + 1))
    st.compress_batch(0, kk[:, :t0], vv[:, :t0])
    step = GraphedDecodeStep(st, 0)
    q = rng.standard_normal((B, H * G, D)).astype(np.float32)
    for t in range(t0, T):  # decode steps: append token t, attend
        out = step(torch.from_numpy(kk[:, t]).cuda(), torch.from_numpy(vv[:, t]).cuda(), torch.from_numpy(q).cuda())
    if t0 == T:
        out = attention_decode_batched(st, 0, torch.from_numpy(q))
    out = out.cpu().numpy()
    w = rng.random((B, H * G, T)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
    for b in range(B):
        ref = O.OracleStore(1, H, D, pack_size=k, repack=repack)
        ref.compress_batch(0, kk[b], vv[b])
        assert st[0].stream_bytes(b) == ref.layer_stream(0)
        for hq in range(H * G):
            rs = O.naive_k_scores(ref, 0, hq // G, q[b, hq])
            _close(s[b, hq], rs)
            _close(o[b, hq], O.naive_v_output(ref, 0, hq // G, w[b, hq]))
            x = rs / np.sqrt(D)
            p = np.exp(x - x.max())
            _close(out[b, hq], O.naive_v_output(ref, 0, hq // G, p / p.sum()))


@pytest.mark.parametrize("seed", range(12))
def test_randomized_store_files_layers_and_shards(seed, tmp_path):
    """Random multi-layer stores (formats, repack, batch): PKKS save -> load ->
    save bit-exact and attention-identical; kv-head-split repacking through
    simulated ranks equals the single store."""
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200 import sharding as S
    from paper_2512_24449_b200.kv_store import load_store, save_store
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    rng = np.random.default_rng(9000 + seed)
    k = int(rng.choice([8, 16]))
    D = int(rng.choice([64, 128]))
    B = int(rng.integers(1, 3))
    H = int(rng.choice([2, 4]))
    layers = int(rng.integers(1, 3))
    repack = str(rng.choice(["none", "v_median", "greedy"]))
    st = CS(layers, H, D, batch=B, pack_size=k, repack=repack)
    data = []
    for layer in range(layers):
        T = int(rng.integers(1, 64 * 3))
        kk, vv = _kv(rng, T, H, D, batch=B)
        data.append((kk, vv))
        c = int(rng.integers(0, T + 1))
        st.compress_batch(layer, kk[:, :c], vv[:, :c])
        st.compress_batch(layer, kk[:, c:], vv[:, c:])
    save_store(st, tmp_path / "a.pkks")
    ld = load_store(tmp_path / "a.pkks")
    save_store(ld, tmp_path / "b.pkks")
    assert (tmp_path / "a.pkks").read_bytes() == (tmp_path / "b.pkks").read_bytes()
    q = torch.from_numpy(rng.standard_normal((B, H * 2, D)).astype(np.float32)).cuda()
    for layer in range(layers):
        assert torch.equal(attention_decode_batched(ld, layer, q), attention_decode_batched(st, layer, q))
    # shards of layer 0 (kv-head split over 2 simulated ranks)
    kk, vv = data[0]
    parts = [S.plan_partition(B, H, 2, r, prefer="head") for r in range(2)]
    local = [CS(1, p.local_heads, D, batch=B, pack_size=k, repack=repack) for p in parts]
    ks = [np.ascontiguousarray(kk[:, :, p.h0:p.h1]) for p in parts]
    vs = [np.ascontiguousarray(vv[:, :, p.h0:p.h1]) for p in parts]
    codes = []
    for lst, k1, v1 in zip(local, ks, vs):
        c = lst[0].pending_codes(lst._norm(k1, True), lst._norm(v1, True))
        codes.append(None if c is None else c.view(torch.uint8))
    for lst, p, k1, v1 in zip(local, parts, ks, vs):
        S.compress_sharded(lst, p, 0, k1, v1, all_gather=lambda t: torch.stack(codes))
    full = {(e.seq, e.kind, e.head, e.token_start): e for e in st[0].directory()}
    for lst, p in zip(local, parts):
        for e in lst[0].directory():
            g = full[(e.seq, e.kind, e.head + p.h0, e.token_start)]
            assert lst[0].block_bytes(e) == st[0].block_bytes(g)


@pytest.mark.parametrize("G", [4, 8])
def test_fused_normal_regime_parity(G):
    """More blocks per kind than the grid has warps (ranges of 1-2 blocks that
    straddle unit boundaries, the regime the benchmarks run in): fused K, V and
    attention against the oracle on two sequences of a B = 8, H = 8 store."""
    _, _, F, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    rng = np.random.default_rng(77 + G)
    B, H, D, T = 8, 8, 128, 64 * 32 + 17
    kk = (rng.standard_normal((B, T, H, D)) * rng.uniform(0.3, 3, (B, T, 1, 1))).astype(np.float16)
    vv = rng.standard_normal((B, T, H, D)).astype(np.float16)
    st = CS(1, H, D, batch=B)
    st.compress_batch(0, kk, vv)
    assert 2 * B * H * st[0].nblk_h > 2 * 1776
    q = rng.standard_normal((B, H * G, D)).astype(np.float32)
    w = rng.random((B, H * G, T)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
    a = attention_decode_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    for b in (0, 5):
        ref = O.OracleStore(1, H, D)
        ref.compress_batch(0, kk[b], vv[b])
        assert st[0].stream_bytes(b) == ref.layer_stream(0)
        for hq in range(0, H * G, 3):
            rs = O.naive_k_scores(ref, 0, hq // G, q[b, hq])
            _close(s[b, hq], rs)
            _close(o[b, hq], O.naive_v_output(ref, 0, hq // G, w[b, hq]))
            x = rs / np.sqrt(D)
            p = np.exp(x - x.max())
            _close(a[b, hq], O.naive_v_output(ref, 0, hq // G, p / p.sum()))


@pytest.mark.parametrize("seed", range(16))
def test_randomized_codec_and_quantizer(seed):
    """Random shapes / widths / scales through quantize, encode, decode and
    decode_pack_at against the oracle (bit-exact)."""
    _, C, _, Q, _ = _pk()
    rng = np.random.default_rng(3000 + seed)
    k = int(rng.choice([2, 4, 8, 16, 32]))
    rows = k * int(rng.integers(1, 9))
    cols = int(rng.integers(1, 300))
    layout = int(rng.integers(0, 2))
    mag = float(10 ** rng.uniform(-3, 4))
    x = (rng.standard_normal((3, rows, cols)) * mag).astype(np.float16)
    x[0, 0] = x[0, 0, 0]  # a constant row
    rel = float(rng.choice([0.01, 0.05, 0.1, 0.3, 1.0]))
    qb = Q.quantize_token_wise(torch.from_numpy(x).cuda(), rel, layout)
    for i in range(3):
        r = O.quantize_token_wise(x[i], rel)
        assert np.array_equal(qb.q[i].cpu().numpy().astype(np.int64), r.q)
        assert np.array_equal(qb.scale[i].cpu().numpy(), r.scale) and np.array_equal(qb.zp[i].cpu().numpy(), r.zp)
    try:
        blocks = C.encode_blocks(qb, k, layout)
    except Exception as e:  # wide ranges at tiny rel: the oracle must refuse too
        with pytest.raises(type(e)):
            O.encode_block(O.quantize_token_wise(x[1], rel), k, layout, layout)
        return
    for i in range(3):
        r = O.quantize_token_wise(x[i], rel)
        ref = O.encode_block(O.QuantBlock(r.q, r.scale, r.zp, layout), k, layout, layout)
        assert blocks[i].to_bytes() == ref
        assert C.compression_ratio(blocks[i]) == O.compression_ratio(ref)
        d = C.decode_block(C.PackedBlock.from_bytes(ref))
        assert np.array_equal(d.q.cpu().numpy().astype(np.int64), r.q)
        P = (rows // k) * cols
        for p in rng.integers(0, P, 3):
            assert np.array_equal(C.decode_pack_at(blocks[i], int(p)).cpu().numpy().astype(np.int64),
                                  O.decode_pack_at(ref, int(p)))


@pytest.mark.parametrize("seed", range(8))
def test_randomized_graphed_decode_loop(seed):
    """GraphedDecodeStep (default format) over random batch / heads / groups and
    start lengths, across block completions: every step bit-identical to the eager
    append + attention on a twin store."""
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import GraphedDecodeStep, attention_decode_batched
    rng = np.random.default_rng(7000 + seed)
    B, H, G = int(rng.integers(1, 4)), int(rng.integers(1, 5)), int(rng.choice([1, 2, 4, 8]))
    T0, steps, D = int(rng.integers(0, 200)), int(rng.integers(1, 140)), 128
    a, b = CS(1, H, D, batch=B), CS(1, H, D, batch=B)
    if T0:
        k0, v0 = _kv(rng, T0, H, D, batch=B)
        a.compress_batch(0, k0, v0)
        b.compress_batch(0, k0, v0)
    step = GraphedDecodeStep(a, 0)
    for t in range(steps):
        kt = torch.from_numpy(rng.standard_normal((B, H, D)).astype(np.float16)).cuda()
        vt = torch.from_numpy(rng.standard_normal((B, H, D)).astype(np.float16)).cuda()
        q = torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32)).cuda()
        got = step(kt, vt, q).clone()
        b.append_token(0, kt, vt)
        assert torch.equal(got, attention_decode_batched(b, 0, q)), f"step {t}"
    assert a[0].nblk_h == b[0].nblk_h and a[0].nres_h == b[0].nres_h
    for s in range(B):
        assert a[0].stream_bytes(s) == b[0].stream_bytes(s)


@pytest.mark.parametrize("repack", ["none", "v_median"])
def test_iterate_blocks_matches_oracle(repack):
    """iterate_blocks on the device store: per (layer, kind) the
    directory entries in order -- head, token range, length, permutation and the
    block bytes -- then the residue handle, equal to the oracle's after a prefill
    and token appends that cross block boundaries (two layers)."""
    _, _, _, _, CS = _pk()
    rng = np.random.default_rng(31)
    H, D, T0, A = 3, 128, 64 * 2 + 40, 90
    st = CS(2, H, D, repack=repack)
    ref = O.OracleStore(2, H, D, repack=repack)
    for layer in range(2):
        kk, vv = _kv(rng, T0 + A, H, D)
        st.compress_batch(layer, kk[:T0], vv[:T0])
        ref.compress_batch(layer, kk[:T0], vv[:T0])
        for t in range(T0, T0 + A):
            st.append_token(layer, kk[t], vv[t])
            ref.append_token(layer, kk[t], vv[t])
    for layer in range(2):
        for kind in (0, 1):
            got = st.iterate_blocks(layer, kind)
            ents, nres = ref.iterate_blocks(layer, kind)
            blocks, res = got[:-1], got[-1]
            assert [(e.head, e.token_start, e.token_end, e.byte_len, e.permutation.tolist()) for e in blocks] == \
                   [(e.head, e.token_start, e.token_end, e.byte_len, e.permutation.tolist()) for e in ents]
            assert [st[layer].block_bytes(e) for e in blocks] == [ref.block_bytes(e) for e in ents]
            assert (res.layer, res.tokens, res.token_start) == (layer, nres, (T0 + A) // 64 * 64)


@pytest.mark.parametrize("single_pass", [None, True, False])
def test_graphed_attention_zero_copy_host_io(single_pass):
    """GraphedAttention with pinned host q / out: the graph reads q from host memory
    (pkv_copy_scaled, prescale folded in) and writes the output to host memory; equal to
    the device-q replay (<= 1e-6 relative), replays follow new host contents, a residue
    append replays the same capture, a new host buffer re-captures, and
    ShardedDecoder.step(q_host, out=...) takes the same path."""
    _, _, _, _, CS = _pk()
    from paper_2512_24449_b200.attention_sim import GraphedAttention
    from paper_2512_24449_b200 import sharding as S
    rng = np.random.default_rng(41)
    B, H, G, D, T = 2, 2, 4, 128, 64 * 6 + 11
    st = CS(1, H, D, batch=B)
    kk, vv = _kv(rng, T + 3, H, D, batch=B)
    st.compress_batch(0, kk[:, :T], vv[:, :T])
    ga_d, ga_h = GraphedAttention(st, 0), GraphedAttention(st, 0)
    ga_d.single_pass = ga_h.single_pass = single_pass  # None: the heuristic; True / False: either attention path
    qh = torch.empty((B, H * G, D)).pin_memory()
    oh = torch.empty((B, H * G, D)).pin_memory()
    for step in range(3):
        qh.copy_(torch.from_numpy(rng.standard_normal((B, H * G, D)).astype(np.float32)))
        ref = ga_d(qh.cuda()).cpu()
        got = ga_h(qh, out=oh)
        torch.cuda.synchronize()
        assert got.data_ptr() == oh.data_ptr()
        assert torch.allclose(oh, ref, rtol=1e-6, atol=1e-6 * float(ref.abs().max()))
        if step == 1:  # a residue token: same capture
            st.append_token(0, kk[:, T], vv[:, T])
    assert ga_h.captures == 1
    qh2 = qh.clone().pin_memory()
    o2 = ga_h(qh2).cpu()  # new host buffer, device output: re-capture
    assert ga_h.captures == 2
    assert torch.allclose(o2, ga_d(qh2.cuda()).cpu(), rtol=1e-6, atol=1e-6 * float(o2.abs().max()))
    part = S.plan_partition(B, H, 1, 0)
    dec = S.ShardedDecoder(part, ga_h, H * G, D)
    oh2 = torch.empty(B * H * G * D).pin_memory()
    dec.step(qh, out=oh2)
    torch.cuda.synchronize()
    assert torch.allclose(oh2.view(B, H * G, D), ga_d(qh.cuda()).cpu(), rtol=1e-6, atol=1e-6 * float(oh2.abs().max()))
