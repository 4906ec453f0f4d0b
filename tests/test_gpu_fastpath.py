"""Parity of exactly the kernels the benchmark times.

Every default-format call (pack 16, head_dim 128, block 64, G <= 8) must run
the tensor-core kernels (fused_k_fast_kernel / fused_v_fast_kernel) whatever
the context length or row stride; pkv_last_path() says which family a call
launched and every test here asserts it.  Parity is against the CPU oracle
(oracle/packkv_oracle.py, f64 naive GEMVs over its own compressed store) at
the BASELINE config shapes on sampled sequences, for all four residues of
L mod 4, and with extreme V weights (tolerance
||gpu - f64||_inf <= 1e-3 * ||f64||_inf)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import packkv_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _mods():
    from paper_2512_24449_b200 import _native as N
    from paper_2512_24449_b200 import errors as E
    from paper_2512_24449_b200 import fused_kernels as F
    from paper_2512_24449_b200.kv_store import CompressedStore
    return N, E, F, CompressedStore


def _close(a, ref):
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(a - ref).max() if ref.size else 0.0
    assert err <= TOL * scale, f"max abs err {err:.3e} > {TOL} * {scale:.3e}"
    return err / scale


def _bench_kv(B, T, H, seed):
    """Config-distribution K/V on the device (tensor_model.gauss_outlier: 4 / 1
    outlier channels per kv head), [B, T, H, 128] fp16."""
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    k = gauss_outlier((B, T, H, 128), seed=seed)
    v = gauss_outlier((B, T, H, 128), n_outlier=1, seed=seed + 7)
    return k, v


def _k(F, N, st, q):
    s = F.fused_k_scores_batched(st, 0, q)
    assert N.last_path() == N.PATH_FAST, "fused K left the tensor-core kernel"
    return s


def _v(F, N, st, w):
    o = F.fused_v_output_batched(st, 0, w)
    assert N.last_path() == N.PATH_FAST, "fused V left the tensor-core kernel"
    return o


@pytest.mark.parametrize("r", [0, 1, 2, 3])
@pytest.mark.parametrize("G", [1, 4, 8])
def test_fast_kernels_every_length_mod_4(r, G):
    """Lengths L = 64*n + residue with L mod 4 = r: scores are written with
    stride L and the weights read with stride L (no padding by the caller)."""
    N, _, F, CS = _mods()
    rng = np.random.default_rng(100 * r + G)
    H = 2
    for T in (64 * 37 + 20 + r, 64 * 5 + r, 64 * 2 + 40 + r):
        kk = rng.standard_normal((T, H, 128)).astype(np.float16)
        vv = rng.standard_normal((T, H, 128)).astype(np.float16)
        ref = O.OracleStore(1, H, 128)
        ref.compress_batch(0, kk, vv)
        st = CS(1, H, 128)
        st.compress_batch(0, kk, vv)
        q = torch.from_numpy(rng.standard_normal((1, H * G, 128)).astype(np.float32)).cuda()
        w = torch.from_numpy(rng.random((1, H * G, T)).astype(np.float32)).cuda()
        assert w.stride(1) == T
        s = _k(F, N, st, q).cpu().numpy()
        o = _v(F, N, st, w).cpu().numpy()
        for hq in range(H * G):
            _close(s[0, hq], O.naive_k_scores(ref, 0, hq // G, q[0, hq].cpu().numpy()))
            _close(o[0, hq], O.naive_v_output(ref, 0, hq // G, w[0, hq].cpu().numpy()))


# (name, batch, kv heads, G, tokens, sampled sequences)
CONFIG_SHAPES = [
    ("B", 8, 8, 4, 8192, (0, 5)),      # Llama-3-8B GQA, BASELINE configs[1]
    ("E", 2, 8, 8, 16384, (1,)),       # Llama-3-70B GQA G=8 (NU=2 / NT=2 templates)
    ("D", 1, 52, 1, 2048, (0,)),       # LLaMA-30B MHA, 52 heads
]


@pytest.mark.parametrize("r", [0, 1, 2, 3])
@pytest.mark.parametrize("cfg", CONFIG_SHAPES, ids=[c[0] for c in CONFIG_SHAPES])
def test_fast_kernels_config_shapes_vs_oracle(cfg, r):
    name, B, H, G, T0, samples = cfg
    N, _, F, CS = _mods()
    T = T0 + 21 + r  # block count plus a residue of 21 + r rows
    k, v = _bench_kv(B, T, H, seed=7 + r)
    st = CS(1, H, 128, batch=B, max_tokens=T)
    st.compress_batch(0, k, v)
    g = torch.Generator(device="cuda")
    g.manual_seed(r)
    q = torch.randn((B, H * G, 128), device="cuda", generator=g)
    w = torch.softmax(torch.randn((B, H * G, T), device="cuda", generator=g) * 3, -1)
    s = _k(F, N, st, q).cpu().numpy()
    o = _v(F, N, st, w).cpu().numpy()
    qh, wh = q.cpu().numpy(), w.cpu().numpy()
    for b in samples:
        ref = O.OracleStore(1, H, 128)
        ref.compress_batch(0, k[b].cpu().numpy(), v[b].cpu().numpy())
        assert st[0].stream_bytes(b) == ref.layer_stream(0), f"config {name}: packed stream differs"
        heads = range(H) if H <= 8 else (0, 17, H - 1)
        for h in heads:
            for hq in (h * G, h * G + G - 1):
                _close(s[b, hq], O.naive_k_scores(ref, 0, h, qh[b, hq]))
                _close(o[b, hq], O.naive_v_output(ref, 0, h, wh[b, hq]))


@pytest.mark.parametrize("kind", ["one_hot", "log_span", "sparse", "negative"])
@pytest.mark.parametrize("r", [0, 3])
def test_fast_v_extreme_weights(kind, r):
    """V weights the 2-digit fixed point must survive: one-hot rows, weights
    spanning 1e-7..1 inside one block, a few spikes over a flat floor, and
    signed weights."""
    N, _, F, CS = _mods()
    rng = np.random.default_rng(11 + r)
    H, G = 2, 4
    T = 64 * 40 + 9 + r
    kk = rng.standard_normal((T, H, 128)).astype(np.float16)
    vv = (rng.standard_normal((T, H, 128)) * rng.uniform(0.01, 30, (T, 1, 1))).astype(np.float16)
    ref = O.OracleStore(1, H, 128)
    ref.compress_batch(0, kk, vv)
    st = CS(1, H, 128)
    st.compress_batch(0, kk, vv)
    w = np.zeros((1, H * G, T), np.float32)
    for hq in range(H * G):
        if kind == "one_hot":
            w[0, hq, rng.integers(0, T)] = 1.0
        elif kind == "log_span":
            w[0, hq] = 10.0 ** rng.uniform(-7, 0, T)
        elif kind == "sparse":
            w[0, hq] = 1e-6
            w[0, hq, rng.integers(0, T, 5)] = rng.uniform(0.1, 1, 5)
        else:
            w[0, hq] = rng.standard_normal(T) * 10.0 ** rng.uniform(-7, 0, T)
    o = _v(F, N, st, torch.from_numpy(w).cuda()).cpu().numpy()
    for hq in range(H * G):
        _close(o[0, hq], O.naive_v_output(ref, 0, hq // G, w[0, hq]))


def test_row_stride_validation():
    """The C ABI rejects a stride shorter than the compressed blocks
    (ShapeMismatchError) and, for a stride that would cut into the residue
    rows, writes none past it and raises PKV_FLAG_SHAPE."""
    N, E, F, CS = _mods()
    from paper_2512_24449_b200.kv_store import ctypes_ref
    rng = np.random.default_rng(3)
    H, G, T = 2, 4, 64 * 3 + 30
    kk = rng.standard_normal((T, H, 128)).astype(np.float16)
    st = CS(1, H, 128)
    st.compress_batch(0, kk, kk)
    ls = st[0]
    lib = N.lib()
    q = torch.randn((1, H * G, 128), device="cuda")
    stride = 64 * 3 + 10                                          # cuts the 30 residue rows
    buf = torch.full((H * G * stride + 64,), 7.0, device="cuda")  # 64 canaries past the last row
    with pytest.raises(E.ShapeMismatchError):
        N.check(lib.pkv_fused_k_scores(ctypes_ref(ls.struct()), ls.nblk_h, N.ptr(q), H * G, N.ptr(buf), 100,
                                       N.stream()), "k")
    ls.err.zero_()
    N.check(lib.pkv_fused_k_scores(ctypes_ref(ls.struct()), ls.nblk_h, N.ptr(q), H * G, N.ptr(buf), stride,
                                   N.stream()), "k")
    torch.cuda.synchronize()
    assert bool((buf[H * G * stride:] == 7.0).all()), "scores written past the last row"
    with pytest.raises(E.ShapeMismatchError):
        N.raise_flags(int(ls.err.item()), "k")
    ls.err.zero_()
    w = torch.rand((1, H * G, 100), device="cuda")
    need = int(lib.pkv_fused_v_scratch_bytes(ctypes_ref(ls.struct()), ls.nblk_h, H * G))
    scr = torch.empty(need, dtype=torch.uint8, device="cuda")
    out = torch.empty((1, H * G, 128), device="cuda")
    with pytest.raises(E.ShapeMismatchError):
        N.check(lib.pkv_fused_v_output(ctypes_ref(ls.struct()), ls.nblk_h, N.ptr(w), H * G, 100, N.ptr(out),
                                       N.ptr(scr), need, N.stream()), "v")


def test_smoke_entry_runs_fast_kernels():
    import __graft_entry__ as ge
    N, _, _, _ = _mods()
    ge.smoke()
    assert N.last_path() == N.PATH_SINGLE  # smoke() asserts PATH_FAST after its K and V calls


def test_graphed_decode_loop_device_flush():
    """GraphedDecodeLoop: stage + device-side block flush + attention for two
    layers in one CUDA graph per step.  Block completions happen inside the
    replayed graph (no re-capture per 64 tokens); the arena streams stay
    bit-identical to eager appends and to the oracle, and every step's
    attention matches the eager composition on a store built by
    append_token."""
    N, _, F, CS = _mods()
    from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop, attention_decode_batched
    rng = np.random.default_rng(77)
    B, H, G, D, Ly = 2, 2, 4, 128, 2
    T0, steps = 100, 200
    k = (rng.standard_normal((Ly, B, T0 + steps, H, D))).astype(np.float16)
    v = (rng.standard_normal((Ly, B, T0 + steps, H, D))).astype(np.float16)
    q = rng.standard_normal((steps, Ly, B, H * G, D)).astype(np.float32)
    a = CS(Ly, H, D, batch=B, check=False)
    r = CS(Ly, H, D, batch=B, check=False)
    for l in range(Ly):
        a.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
        r.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
    loop = GraphedDecodeLoop(a, H * G, headroom=2)   # headroom 2: re-captures every 128 tokens
    kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    worst = 0.0
    for t in range(steps):
        out = loop.step(kd[:, :, T0 + t:T0 + t + 1], vd[:, :, T0 + t:T0 + t + 1], qd[t]).clone()
        for l in range(Ly):
            r.append_token(l, kd[l, :, T0 + t], vd[l, :, T0 + t])
            ref = attention_decode_batched(r, l, qd[t, l])
            e = float((out[l] - ref).abs().max() / ref.abs().max())
            worst = max(worst, e)
    assert worst <= 1e-5, worst
    torch.cuda.synchronize()
    a.check_errors()
    assert loop.captures <= steps // 128 + 2, loop.captures
    for l in range(Ly):
        assert a[l].nblk_h == r[l].nblk_h and a[l].nres_h == r[l].nres_h
        assert int(a[l].nblk[0].item()) == r[l].nblk_h and int(a[l].nres[0].item()) == r[l].nres_h
        for b in range(B):
            assert a[l].stream_bytes(b) == r[l].stream_bytes(b), f"layer {l} seq {b}: stream differs"
    ref = O.OracleStore(1, H, D)
    ref.compress_batch(0, k[1, 1], v[1, 1])
    assert a[1].stream_bytes(1) == ref.layer_stream(0)
