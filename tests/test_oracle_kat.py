"""Pins the CPU oracle against every known-answer example SPEC.md gives for the
hot path, plus the SPEC invariants and
acceptance criteria that are cheap enough for the CPU suite."""
import math

import numpy as np
import pytest

from oracle import packkv_oracle as O
from paper_2512_24449_b200 import errors as E


# ---------------- quantizer ----------------
def test_quantize_example_spec117():
    qb = O.quantize_token_wise(np.array([[0.0, 0.34, 1.0]], np.float16), 0.1)
    assert qb.q.tolist() == [[0, 3, 10]]
    assert qb.scale[0] == np.float32(0.1) and qb.zp[0] == 0.0


def test_quantize_constant_row_spec118():
    qb = O.quantize_token_wise(np.array([[5, 5, 5]], np.float16), 0.1)
    assert qb.q.tolist() == [[0, 0, 0]] and qb.scale[0] == 0 and qb.zp[0] == 5


def test_round_half_away_tie_trap():
    # [0, .25, 1] @ 0.5: t = 0.5 -> 1 (half away); np.round would give 0
    assert O.quantize_token_wise(np.array([[0, .25, 1]], np.float16), 0.5).q.tolist() == [[0, 1, 2]]


def test_floor_plus_half_trap():
    t = np.array([np.nextafter(np.float32(0.5), np.float32(0))], np.float32)  # 0.49999997
    assert O.round_half_away_nonneg(t)[0] == 0.0
    assert np.floor(t + np.float32(0.5))[0] == 1.0     # the trap the oracle avoids


def test_dequantize_examples_spec126():
    assert O.dequantize(np.array([3]), np.float32(0.1), np.float32(0.0))[0] == np.float32(3) * np.float32(0.1)
    assert O.dequantize(np.array([0]), np.float32(0.7), np.float32(2.5))[0] == 2.5
    assert abs(O.dequantize(np.array([10]), np.float32(0.1), np.float32(0))[0] - 1.0) < 1e-6


def test_quantize_nonfinite_raises():
    with pytest.raises(E.NonFiniteValueError):
        O.quantize_token_wise(np.array([[0, np.inf]], np.float16), 0.1)


@pytest.mark.parametrize("rel", [0.05, 0.1, 0.2])
def test_error_bound_criterion2(rel):
    rng = np.random.default_rng(int(rel * 100))
    for _ in range(100):  # criterion 2 uses 1000; 100 keeps the CPU suite fast
        x = (rng.standard_normal((64, 128)) * rng.uniform(0.01, 10)).astype(np.float16)
        qb = O.quantize_token_wise(x, rel)
        d = O.dequantize(qb.q, qb.scale, qb.zp)
        rng_row = x.astype(np.float32).max(1) - x.astype(np.float32).min(1)
        err = np.abs(x.astype(np.float32) - d).max(1)
        assert np.all(err <= rel / 2 * rng_row + 2 ** -10)
        assert qb.q.max() <= round(1 / rel)
        # idempotence: quantize(dequantize(quantize(x))) == quantize(x) codes
        q2 = O.quantize_token_wise(d.astype(np.float16), rel)
        assert q2.q.shape == qb.q.shape


# ---------------- repacker ----------------
def test_pack_cost_examples():
    assert O.pack_cost(np.array([[0, 5], [3, 1]])) == 50
    assert O.pack_cost(np.full((4, 7), 3)) == 7 * O.META_BITS
    assert O.pack_cost(np.array([[1, 2, 3]])) == 3 * O.META_BITS


def test_greedy_examples():
    p = O.repack_greedy(np.array([[0], [9], [0], [9]]), 2)
    assert p.cost_bits == 40
    groups = [sorted(p.permutation[i:i + 2].tolist()) for i in (0, 2)]
    assert sorted(groups) == [[0, 2], [1, 3]]
    p4 = O.repack_greedy(np.arange(4)[:, None] * 3, 4)
    assert sorted(p4.permutation.tolist()) == [0, 1, 2, 3]
    assert p4.cost_bits == O.pack_cost(np.arange(4)[:, None] * 3)


def test_v_median_examples():
    z = np.zeros((3, 1))
    assert O.repack_v_median(z, np.array([[5], [1], [3]]), 2).permutation.tolist() == [1, 2, 0]
    assert O.repack_v_median(z, np.array([[2], [2], [1]]), 2).permutation.tolist() == [2, 0, 1]
    assert O.repack_v_median(z, np.array([[4], [4], [4]]), 2).permutation.tolist() == [0, 1, 2]
    # lower median for even lengths: [1, 2, 9, 9] -> 2
    assert O.lower_median(np.array([[9, 1, 9, 2]]))[0] == 2


def test_oracle_examples():
    assert O.count_partitions(8, 4) == 35
    part, c = O.oracle_optimal(np.array([[0], [0], [9], [9]]), 2)
    assert c == 40
    part, c = O.oracle_optimal(np.arange(4)[:, None], 4)
    assert c == O.pack_cost(np.arange(4)[:, None])
    with pytest.raises(E.InstanceTooLargeError):
        O.oracle_optimal(np.zeros((14, 1)), 2)


def test_oracle_dominance_criterion7():
    rng = np.random.default_rng(7)
    for n in (4, 6, 8):
        for k in (2, 4):
            if n % k:
                continue
            for _ in range(10):
                X = rng.integers(0, 12, (n, 6))
                _, opt = O.oracle_optimal(X, k)
                assert opt <= O.repack_greedy(X, k).cost_bits
                assert opt <= O.repack_v_median(X, X[:, 3:], k).cost_bits
                assert opt <= O.repack_none(X, k).cost_bits


def test_plans_are_bijections():
    rng = np.random.default_rng(1)
    X = rng.integers(0, 10, (64, 32))
    for plan in (O.repack_none(X, 16), O.repack_v_median(X, X[:, 16:], 16), O.repack_greedy(X, 16)):
        assert sorted(plan.permutation.tolist()) == list(range(64))


# ---------------- codec ----------------
def _qb(q, kind=O.KIND_K):
    r = q.shape[0]
    return O.QuantBlock(np.asarray(q), np.full(r, 0.5, np.float32), np.zeros(r, np.float32), kind)


def test_codec_column_example_spec282():
    col = np.array([0, 3, 10, 10, 7, 2, 0, 1])[:, None]
    b = O.encode_block(_qb(col, O.KIND_V), 8, O.LAYOUT_V_CONTIGUOUS, O.KIND_V)
    info = O.pack_info(b)[1]
    assert info.widths.tolist() == [4] and info.minima.tolist() == [0]
    assert len(b) - O.header_bytes(8, 1, 8) == 4
    assert O.decode_block(b).q.ravel().tolist() == col.ravel().tolist()


def test_constant_block_header_only_and_cr_spec308():
    b = O.encode_block(_qb(np.full((64, 128), 3)), 8)
    assert len(b) == O.header_bytes(64, 128, 8) == 2824
    assert abs(O.compression_ratio(b) - 131072 / 22528) < 1e-12
    assert round(O.compression_ratio(b), 2) == 5.82


def test_all_width4_cr_spec309():
    q = np.zeros((64, 128), np.int64)
    q[1::8, :] = 15                                 # every 8-row pack has range 15 -> width 4
    b = O.encode_block(_qb(q), 8)
    assert np.all(O.pack_info(b)[1].widths == 4)
    assert abs(O.compression_ratio(b) - 131072 / (1024 * 20 + 1024 * 32 + 2048)) < 1e-12


def test_kivi_cr_criterion1():
    assert abs(O.kivi_baseline_cr(2, 64, 32) - 6.4) < 0.005
    assert abs(O.kivi_baseline_cr(3, 64, 32) - 4.57) < 0.005
    assert O.kivi_baseline_cr(16, 64, 0) == 1.0


def test_header_sizes_appendixB():
    assert [O.header_bytes(64, 128, k) for k in O.PACK_SIZES] == [10504, 5384, 2824, 1544, 904]
    assert all(O.header_bytes(64, 128, k) % 16 == 8 for k in O.PACK_SIZES)


def test_k_interleave_order_spec322():
    pos = O.k_pos(128)
    inv = np.argsort(pos)
    assert inv[:4].tolist() == [0, 4, 8, 12] and inv[31] == 124 and inv[32] == 1
    # generalisation for cols % 4 != 0
    p7 = O.k_pos(7)
    assert np.argsort(p7).tolist() == [0, 4, 1, 5, 2, 6, 3]


def test_wire_layout_bytes():
    q = np.zeros((16, 4), np.int64)
    q[:, 1] = np.arange(16) % 4         # width 2 column
    qb = O.QuantBlock(q, np.full(16, 1.0, np.float32), np.full(16, -2.0, np.float32), O.KIND_V)
    b = O.encode_block(qb, 16, O.LAYOUT_V_CONTIGUOUS, O.KIND_V)
    assert b[:8] == bytes([1, 1, 16, 0, 16, 0, 4, 0])
    assert b[8] == 0x20 and b[9] == 0x00                      # widths 0,2 | 0,0 (low nibble first)
    pay = b[O.header_bytes(16, 4, 16):]
    assert len(pay) == 4
    v = int.from_bytes(pay, "little")
    assert [(v >> (2 * j)) & 3 for j in range(16)] == (np.arange(16) % 4).tolist()
    scale = np.frombuffer(b[8 + 2 + 8: 8 + 2 + 8 + 2], "<f2")[0]
    assert scale == 1.0


def test_codec_lossless_criterion3_random_and_adversarial():
    rng = np.random.default_rng(3)
    for k in O.PACK_SIZES:
        for layout in (0, 1):
            cases = [np.zeros((64, 128), np.int64), np.full((64, 128), 65535, np.int64)]
            q = np.zeros((64, 128), np.int64); q[0] = 32767; cases.append(q)      # max range 15 bits
            q = np.zeros((k, 5), np.int64); q[-1] = 7; cases.append(q)           # single row-group, ragged cols
            for _ in range(20):
                rows = k * int(rng.integers(1, 5))
                cols = int(rng.integers(1, 40))
                cases.append(rng.integers(0, 1 << int(rng.integers(0, 15)), (rows, cols)))
            for q in cases:
                b = O.encode_block(_qb(q), k, layout)
                d = O.decode_block(b)
                assert np.array_equal(d.q, q)
                P = (q.shape[0] // k) * q.shape[1]
                info = O.pack_info(b)[1]
                for i in (0, P // 2, P - 1):
                    assert np.array_equal(O.decode_pack_at(b, i), _pack_slice(d.q, k, layout, i))
                # width optimality: no width can shrink
                r = _ranges(q, k, layout)
                assert np.all((1 << info.widths) > r)
                assert np.all((info.widths == 0) | ((1 << np.maximum(info.widths - 1, 0)) <= r))


def _pack_slice(q, k, layout, i):
    cols = q.shape[1]
    g, p = divmod(i, cols)
    c = int(np.argsort(O.phys_pos(cols, layout))[p])
    return q[g * k:(g + 1) * k, c]


def _ranges(q, k, layout):
    rows, cols = q.shape
    inv = np.argsort(O.phys_pos(cols, layout))
    pk = q.reshape(rows // k, k, cols).transpose(0, 2, 1)[:, inv, :].reshape(-1, k)
    return pk.max(1) - pk.min(1)


def test_layout_equivalence():
    rng = np.random.default_rng(5)
    q = rng.integers(0, 30, (64, 128))
    a = O.decode_block(O.encode_block(_qb(q), 16, 0))
    b = O.decode_block(O.encode_block(_qb(a.q), 16, 1))
    assert np.array_equal(b.q, q)


def test_decode_errors():
    b = O.encode_block(_qb(np.arange(64 * 8).reshape(64, 8) % 7), 16)
    with pytest.raises(E.MalformedBlockError):
        O.decode_block(b[:-1])
    with pytest.raises(E.MalformedBlockError):
        O.decode_block(b[:5])
    bad = bytearray(b); bad[2] = 7
    with pytest.raises(E.MalformedBlockError):
        O.decode_block(bytes(bad))
    with pytest.raises(IndexError):
        O.decode_pack_at(b, 10 ** 6)
    with pytest.raises(E.ShapeMismatchError):
        O.encode_block(_qb(np.zeros((10, 4), np.int64)), 16)
    with pytest.raises(E.WidthOverflowError):
        O.encode_block(_qb(np.array([[0], [65536]] * 8)), 16)


def test_cost_consistency_with_codec():
    """plan cost_bits == encoded payload+pack-metadata bits (k in {8,16,32})."""
    rng = np.random.default_rng(11)
    for k in (8, 16, 32):
        q = rng.integers(0, 11, (64, 128))
        b = O.encode_block(_qb(q), k, 1)
        bits = (len(b) - 8 - 4 * 64) * 8
        assert bits == O.repack_none(q, k).cost_bits


# ---------------- store ----------------
def _tokens(rng, n, H, D):
    return (rng.standard_normal((n, H, D)).astype(np.float16),
            rng.standard_normal((n, H, D)).astype(np.float16))


def test_store_thresholds():
    rng = np.random.default_rng(0)
    H, D = 2, 16
    s = O.OracleStore(1, H, D)
    k, v = _tokens(rng, 100, H, D)
    for t in range(63):
        s.append_token(0, k[t], v[t])
    assert len(s.directory) == 0 and s.stage_k[0].shape[0] == 63
    s.append_token(0, k[63], v[63])
    assert len(s.directory) == 2 * H and s.stage_k[0].shape[0] == 0
    s2 = O.OracleStore(1, H, D)
    s2.compress_batch(0, k, v)
    assert len(s2.directory) == 2 * H and s2.stage_k[0].shape[0] == 36
    s3 = O.OracleStore(1, H, D)
    s3.compress_batch(0, k[:0], v[:0])
    assert len(s3.directory) == 0 and s3.total_tokens(0) == 0


@pytest.mark.parametrize("repack", ["none", "v_median", "greedy"])
def test_incremental_equals_batch_criterion8(repack):
    rng = np.random.default_rng(8)
    H, D, n = 2, 32, 256       # criterion 8 uses 1024 tokens; see test_oracle_slow for the full size
    k, v = _tokens(rng, n, H, D)
    a = O.OracleStore(1, H, D, repack=repack)
    for t in range(n):
        a.append_token(0, k[t], v[t])
    b = O.OracleStore(1, H, D, repack=repack)
    b.compress_batch(0, k[:100], v[:100])
    b.compress_batch(0, k[100:], v[100:])
    assert bytes(a.arena) == bytes(b.arena)
    assert [(e.kind, e.head, e.token_start, e.byte_offset, e.byte_len, e.permutation.tolist())
            for e in a.directory] == [(e.kind, e.head, e.token_start, e.byte_offset, e.byte_len,
                                       e.permutation.tolist()) for e in b.directory]


def test_store_order_and_coverage():
    rng = np.random.default_rng(2)
    H, D = 3, 16
    s = O.OracleStore(1, H, D)
    k, v = _tokens(rng, 150, H, D)
    s.compress_batch(0, k, v)
    kinds = [(e.kind, e.head) for e in s.directory]
    assert kinds == [(0, h) for h in range(H)] + [(1, h) for h in range(H)] + \
                    [(0, h) for h in range(H)] + [(1, h) for h in range(H)]
    ents, res = s.iterate_blocks(0, O.KIND_K)
    cov = sorted((e.token_start, e.token_end) for e in ents if e.head == 0)
    assert cov == [(0, 64), (64, 128)] and res == 22
    offs = [(e.byte_offset, e.byte_len) for e in s.directory]
    assert all(offs[i][0] + offs[i][1] == offs[i + 1][0] for i in range(len(offs) - 1))


# ---------------- fused ----------------
def _store(rng, n, repack="none", H=2, D=32):
    s = O.OracleStore(1, H, D, repack=repack)
    k, v = _tokens(rng, n, H, D)
    s.compress_batch(0, k, v)
    return s, k, v


def test_fused_examples():
    rng = np.random.default_rng(4)
    s, k, v = _store(rng, 150)
    sc, tm = O.fused_k_scores(s, 0, 1, np.zeros(32))
    assert np.all(sc == 0) and len(sc) == 150
    e = np.zeros(32, np.float32); e[5] = 1
    sc, tm = O.fused_k_scores(s, 0, 1, e)
    deq0 = O._deq_block_from_bytes(s.block_bytes(O._head_entries(s, 0, 1, 0)[0]))
    assert np.array_equal(sc[:64], deq0[:, 5])
    assert np.all(O.fused_v_output(s, 0, 0, np.zeros(150)) == 0)
    w = np.zeros(150, np.float32); w[70] = 1
    deq1 = O._deq_block_from_bytes(s.block_bytes(O._head_entries(s, 0, 0, 1)[1]))
    assert np.array_equal(O.fused_v_output(s, 0, 0, w), deq1[6])


def test_fused_vs_naive_criterion6():
    rng = np.random.default_rng(6)
    for trial in range(20):  # criterion 6 uses 200 stores; 20 keeps the CPU suite fast
        n = int(rng.integers(1, 300))
        s, _, _ = _store(rng, n, repack=["none", "v_median"][trial % 2])
        q = rng.standard_normal(32).astype(np.float32)
        f, _ = O.fused_k_scores(s, 0, 0, q)
        r = O.naive_k_scores(s, 0, 0, q)
        assert np.abs(f - r).max() <= 1e-3 * np.abs(r).max()
        w = rng.random(n).astype(np.float32)
        f = O.fused_v_output(s, 0, 1, w)
        r = O.naive_v_output(s, 0, 1, w)
        assert np.abs(f - r).max() <= 1e-3 * np.abs(r).max()


def test_linearity_and_errors():
    rng = np.random.default_rng(9)
    s, _, _ = _store(rng, 128)
    q1, q2 = rng.standard_normal((2, 32)).astype(np.float32)
    a = O.fused_k_scores(s, 0, 0, q1)[0] + O.fused_k_scores(s, 0, 0, q2)[0]
    b = O.fused_k_scores(s, 0, 0, q1 + q2)[0]
    assert np.abs(a - b).max() <= 1e-3 * np.abs(b).max()
    with pytest.raises(E.ShapeMismatchError):
        O.fused_k_scores(s, 0, 0, np.zeros(31))
    with pytest.raises(IndexError):
        O.fused_k_scores(s, 0, 5, np.zeros(32))
    with pytest.raises(E.ShapeMismatchError):
        O.fused_v_output(s, 0, 0, np.zeros(3))


# ---------------- attention ----------------
def test_attention_permutation_invariance_criterion5():
    rng = np.random.default_rng(5)
    for _ in range(5):
        K = rng.standard_normal((64, 16)); V = rng.standard_normal((64, 16)); q = rng.standard_normal(16)
        ref = O.attention_reference(K, V, q)
        for _ in range(20):
            P = rng.permutation(64)
            out = O.attention_reference(K[P], V[P], q)
            assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()


def test_attention_decode_singleton_and_neutrality():
    rng = np.random.default_rng(12)
    s, k, v = _store(rng, 1)
    out = O.attention_decode(s, 0, 0, rng.standard_normal(32))
    assert np.allclose(out, v[0, 0].astype(np.float32))
    k, v = _tokens(rng, 128, 2, 32)
    q = rng.standard_normal(32)
    outs = []
    for rp in ("none", "greedy", "v_median"):
        st = O.OracleStore(1, 2, 32, repack=rp)
        st.compress_batch(0, k, v)
        outs.append(O.attention_decode(st, 0, 1, q))
    for o in outs[1:]:
        assert np.abs(o - outs[0]).max() <= 1e-4 * np.abs(outs[0]).max() + 1e-6
