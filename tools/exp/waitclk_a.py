"""Per-warp cycle breakdown of the single-pass attention kernel (diagnostics
build -DPKV_ADIAG=1 copied over the package library by the caller)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
from paper_2512_24449_b200.attention_sim import attention_decode_batched
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "B"]
B, Hkv, Hq, D, L, _ = cfg
st = bench.build_store(cfg, 0)
q = torch.randn((B, Hq, D), device="cuda")
out = torch.zeros((max(B * Hq * D, 6 * 2368 * 2),), device="cuda")[:B * Hq * D].view(B, Hq, D)
for _ in range(3):
    attention_decode_batched(st, 0, q, out=out, single_pass=True)
torch.cuda.synchronize()
n = min(B * Hq * D // 2 // 8, 2368)
d = out.view(-1).view(torch.int64)[:8 * n].cpu().numpy().reshape(-1, 8).astype(float)
d = d[d[:, 5] > 0]
wk, wv, pk, pv, tot, it, rf, uc = d.T
print(f"warps {len(d)} items/warp {it.mean():.1f} total cycles mean {tot.mean():.0f} max {tot.max():.0f}")
print(f"share: wait K {np.mean(wk / tot):.3f}  wait V {np.mean(wv / tot):.3f}  K phase {np.mean(pk / tot):.3f}  "
      f"V phase {np.mean(pv / tot):.3f}  rest {np.mean(1 - (wk + wv + pk + pv) / tot):.3f}")
print(f"end refill {np.mean(rf / tot):.3f}  unit change {np.mean(uc / tot):.3f}  per item refill {np.mean(rf / it):.0f}")
print(f"cycles per item: wait K {np.mean(wk / it):.0f} wait V {np.mean(wv / it):.0f} K {np.mean(pk / it):.0f} V {np.mean(pv / it):.0f}")
