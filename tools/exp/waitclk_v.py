"""Per-warp feed-wait share of the fused V kernel (diagnostics build -DPKV_DIAG_WAITCLK=1)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
from paper_2512_24449_b200 import fused_kernels as F
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "B"]
B, Hkv, Hq, D, L, _ = cfg
st = bench.build_store(cfg, 0)
w = torch.softmax(torch.randn((B, Hq, L), device="cuda"), -1)
for _ in range(3):
    F.fused_v_output_batched(st, 0, w)
torch.cuda.synchronize()
d = st[0].v_scratch.view(torch.int64)[:3 * 2368].cpu().numpy().reshape(-1, 3)
wid_all = np.arange(len(d))
sm = d[:, 2] >> 32
d[:, 2] &= 0xffffffff
keep = d[:, 2] > 0
d, sm, wids = d[keep], sm[keep], wid_all[keep]
wt, t, n = d[:, 0].astype(float), d[:, 1].astype(float), d[:, 2]
per_sm = np.array([t[sm == s].mean() for s in range(sm.max() + 1) if (sm == s).any()])
print("per-SM mean loop cycles: min %.0f max %.0f std %.0f; within-SM std (mean over SMs) %.0f" % (
    per_sm.min(), per_sm.max(), per_sm.std(), np.mean([t[sm == s].std() for s in range(sm.max() + 1) if (sm == s).sum() > 1])))
print("mean loop cycles by warp-in-CTA:", [round(float(t[wids % 4 == w].mean())) for w in range(4)])
cta = wids // 4
print("by CTA wave (cta // 148):", [round(float(t[(cta // 148) == c].mean())) for c in range(int(cta.max() // 148) + 1)])
order = np.argsort(per_sm)
print("slowest SMs", order[-8:], "fastest", order[:8])
print(f"warps {len(d)}  blocks/warp {n.mean():.1f}  loop cycles mean {t.mean():.0f} max {t.max():.0f}")
print(f"wait share mean {np.mean(wt / t):.3f}  median {np.median(wt / t):.3f}  p90 {np.percentile(wt / t, 90):.3f}")
print(f"wait cycles per block {np.mean(wt / n):.0f}  loop cycles per block {np.mean(t / n):.0f}")
print("first-block-dominated?", np.mean(wt) , "cycles per warp total wait")
