"""Reproduce one seed of test_randomized_end_to_end_parity and report which output misses."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from oracle import packkv_oracle as O
from paper_2512_24449_b200 import fused_kernels as F, _native as N
from paper_2512_24449_b200.kv_store import CompressedStore as CS
from paper_2512_24449_b200.attention_sim import attention_decode_batched
for seed in map(int, sys.argv[1:]):
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 4)); H = int(rng.integers(1, 5)); G = int(rng.choice([1, 2, 4, 8]))
    T = int(rng.integers(1, 64 * 5))
    rel_k = float(rng.choice([0.05, 0.1, 0.2])); rel_v = float(rng.choice([0.1, 0.2, 0.3]))
    repack = str(rng.choice(["none", "v_median", "greedy"])); D = 128
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
    a = attention_decode_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
    print(f"seed {seed}: B={B} H={H} G={G} T={T} rel={rel_k},{rel_v} repack={repack} nblk={st[0].nblk_h} nres={st[0].nres_h}")
    for b in range(B):
        ref = O.OracleStore(1, H, D, rel_k=rel_k, rel_v=rel_v, repack=repack)
        ref.compress_batch(0, kk[b], vv[b])
        for hq in range(H * G):
            rs = O.naive_k_scores(ref, 0, hq // G, q[b, hq])
            ro = O.naive_v_output(ref, 0, hq // G, w[b, hq])
            x = rs / np.sqrt(D); p = np.exp(x - x.max())
            ra = O.naive_v_output(ref, 0, hq // G, p / p.sum())
            es = np.abs(s[b, hq] - rs).max() / np.abs(rs).max()
            eo = np.abs(o[b, hq] - ro).max() / np.abs(ro).max()
            ea = np.abs(a[b, hq] - ra).max() / np.abs(ra).max()
            if max(es, eo, ea) > 1e-4:
                i = int(np.argmax(np.abs(s[b, hq] - rs)))
                print(f"  b={b} hq={hq} K {es:.2e} (worst t={i}) V {eo:.2e} A {ea:.2e}")
