import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2512_24449_b200.kv_store import CompressedStore as CS
from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop, attention_decode_batched
rng = np.random.default_rng(77)
B, H, G, D, Ly = 2, 2, 4, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 1
T0, steps = 100, 60
k = (rng.standard_normal((Ly, B, T0 + steps, H, D))).astype(np.float16)
v = (rng.standard_normal((Ly, B, T0 + steps, H, D))).astype(np.float16)
q = rng.standard_normal((steps, Ly, B, H * G, D)).astype(np.float32)
a = CS(Ly, H, D, batch=B, check=False); r = CS(Ly, H, D, batch=B, check=False)
for l in range(Ly):
    a.compress_batch(l, k[l, :, :T0], v[l, :, :T0]); r.compress_batch(l, k[l, :, :T0], v[l, :, :T0])
loop = GraphedDecodeLoop(a, H * G, headroom=2)
kd, vd, qd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
for t in range(steps):
    out = loop.step(kd[:, :, T0 + t:T0 + t + 1], vd[:, :, T0 + t:T0 + t + 1], qd[t]).clone()
    for l in range(Ly):
        r.append_token(l, kd[l, :, T0 + t], vd[l, :, T0 + t])
        ref = attention_decode_batched(r, l, qd[t, l])
        e = float((out[l] - ref).abs().max() / ref.abs().max())
        na, nr = a[l].nres.tolist(), r[l].nres.tolist()
        if e > 1e-5 or t < 3:
            print(t, l, f"{e:.3e}", "nres dev", na, "ref", nr, "nblk", a[l].nblk.tolist(), r[l].nblk.tolist(),
                  "stage eq", bool(torch.equal(a[l].stage[:, :, :max(na)], r[l].stage[:, :, :max(na)])),
                  "per-head err", [round(float((out[l][b, hq] - ref[b, hq]).abs().max()), 4) for b in range(B) for hq in range(0, H * G, G)])
        if e > 1e-5 and t > 5: sys.exit(0)
print("ok")
