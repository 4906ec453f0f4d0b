"""Reproduce a randomized parity case and report which stage differs (debug script)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import packkv_oracle as O
from paper_2512_24449_b200 import fused_kernels as F
from paper_2512_24449_b200.kv_store import CompressedStore as CS
from paper_2512_24449_b200.attention_sim import attention_decode_batched
seed = int(sys.argv[1])
rng = np.random.default_rng(1000 + seed)
B = int(rng.integers(1, 4)); H = int(rng.integers(1, 5)); G = int(rng.choice([1, 2, 4, 8])); T = int(rng.integers(1, 64 * 5))
rel_k = float(rng.choice([0.05, 0.1, 0.2])); rel_v = float(rng.choice([0.1, 0.2, 0.3])); repack = str(rng.choice(["none", "v_median", "greedy"]))
D = 128
kk = (rng.standard_normal((B, T, H, D)) * rng.uniform(0.2, 5, (B, T, 1, 1))).astype(np.float16)
vv = rng.standard_normal((B, T, H, D)).astype(np.float16)
st = CS(1, H, D, batch=B, rel_scale_k=rel_k, rel_scale_v=rel_v, repack=repack)
cut = int(rng.integers(0, T + 1))
print("cfg", B, H, G, T, rel_k, rel_v, repack, "cut", cut)
st.compress_batch(0, kk[:, :cut], vv[:, :cut])
print("after batch: nblk", st[0].nblk_h, "nres", st[0].nres_h, st[0].nres.cpu().tolist())
for t in range(cut, min(T, cut + 3)):
    st.append_token(0, kk[:, t], vv[:, t])
    print("after append", t, "nblk", st[0].nblk_h, "nres", st[0].nres_h, st[0].nres.cpu().tolist(), st[0].nblk.cpu().tolist())
if cut + 3 < T:
    st.compress_batch(0, kk[:, cut + 3:], vv[:, cut + 3:])
print("final nblk", st[0].nblk_h, "nres", st[0].nres_h, st[0].nres.cpu().tolist(), st[0].nblk.cpu().tolist())
for b in range(B):
    ref = O.OracleStore(1, H, D, rel_k=rel_k, rel_v=rel_v, repack=repack)
    ref.compress_batch(0, kk[b], vv[b])
    a, r = st[0].stream_bytes(b), ref.layer_stream(0)
    print("seq", b, "stream equal", a == r, len(a), len(r))
    stg = st[0].stage[0, b * H:(b + 1) * H, :st[0].nres_h].permute(1, 0, 2).cpu().numpy()
    print("   stage equal", np.array_equal(stg.view(np.uint16), ref.stage_k[0].view(np.uint16)), stg.shape, ref.stage_k[0].shape)
q = rng.standard_normal((B, H * G, D)).astype(np.float32)
w = rng.random((B, H * G, T)).astype(np.float32)
s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
o = F.fused_v_output_batched(st, 0, torch.from_numpy(w)).cpu().numpy()
a = attention_decode_batched(st, 0, torch.from_numpy(q)).cpu().numpy()
for b in range(B):
    ref = O.OracleStore(1, H, D, rel_k=rel_k, rel_v=rel_v, repack=repack)
    ref.compress_batch(0, kk[b], vv[b])
    for hq in range(H * G):
        rs = O.naive_k_scores(ref, 0, hq // G, q[b, hq])
        es = np.abs(s[b, hq] - rs)
        ro = O.naive_v_output(ref, 0, hq // G, w[b, hq])
        eo = np.abs(o[b, hq] - ro).max() / np.abs(ro).max()
        x = rs / np.sqrt(D); p = np.exp(x - x.max()); ra = O.naive_v_output(ref, 0, hq // G, p / p.sum())
        ea = np.abs(a[b, hq] - ra).max() / np.abs(ra).max()
        bad = np.nonzero(es > 1e-3 * np.abs(rs).max())[0]
        print(f"b{b} hq{hq}: K rel {es.max() / np.abs(rs).max():.2e} bad rows {bad[:8].tolist()}{'...' if len(bad) > 8 else ''} ({len(bad)}) | V rel {eo:.2e} | att rel {ea:.2e}")
