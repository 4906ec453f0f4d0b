"""Per-warp feed-wait share of the fused K kernel (diagnostics build libwaitclk.so,
copied over the package library by the caller)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
from paper_2512_24449_b200 import fused_kernels as F
cfg = bench.CONFIGS["B"]
B, Hkv, Hq, D, L, _ = cfg
st = bench.build_store(cfg, 0)
q = torch.randn((B, Hq, D), device="cuda")
scores = torch.zeros((B, Hq, L), device="cuda")
for _ in range(3):
    F.fused_k_scores_batched(st, 0, q, out=scores)
torch.cuda.synchronize()
d = scores.view(torch.int64).view(-1)[:3 * 1776].cpu().numpy().reshape(-1, 3)
d = d[d[:, 2] > 0]
w, t, n = d[:, 0].astype(float), d[:, 1].astype(float), d[:, 2]
print(f"warps {len(d)}  blocks/warp {n.mean():.1f}  loop cycles mean {t.mean():.0f} max {t.max():.0f}")
print(f"wait share mean {np.mean(w / t):.3f}  median {np.median(w / t):.3f}  p90 {np.percentile(w / t, 90):.3f}")
print(f"wait cycles per block {np.mean(w / n):.0f}  loop cycles per block {np.mean(t / n):.0f}")
