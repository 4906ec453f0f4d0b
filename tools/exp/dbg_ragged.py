import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2512_24449_b200.kv_store import CompressedStore as CS
rng = np.random.default_rng(12)
B, H, G, D = 3, 2, 4, 128
lens = np.array([100, 37, 200]); T = 260
k = rng.standard_normal((B, T, H, D)).astype(np.float16)
v = rng.standard_normal((B, T, H, D)).astype(np.float16)
st = CS(1, H, D, batch=B, check=False)
st.compress_batch(0, k, v, lengths=lens)
refs = [CS(1, H, D, batch=1, check=False) for _ in range(B)]
for b in range(B):
    refs[b].compress_batch(0, k[b:b + 1, :lens[b]], v[b:b + 1, :lens[b]])
torch.cuda.synchronize()
for b in range(B):
    a, r = st[0].stream_bytes(b), refs[b][0].stream_bytes(0)
    print(b, len(a), len(r), a == r)
    ents = [e for e in st[0].directory() if e.seq == b]
    rents = refs[b][0].directory()
    for e, f in zip(ents, rents):
        x, y = st[0].block_bytes(e), refs[b][0].block_bytes(f)
        if x != y:
            i = next(i for i in range(min(len(x), len(y))) if x[i] != y[i])
            print("  block", e.kind, e.head, e.t0 if hasattr(e, 't0') else '', "len", len(x), len(y), "first diff", i)
# staged rows compare
for b in range(B):
    nr = int(st[0].nres[b]); print("seq", b, "nres", nr, refs[b][0].nres_h, "stage eq K",
      bool(torch.equal(st[0].stage[0, b*H:(b+1)*H, :nr], refs[b][0].stage[0, :, :nr])))
