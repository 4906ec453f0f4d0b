"""Fused K/V time vs the quantization scale (fast path w <= 4 vs in-launch scalar path)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2512_24449_b200 import fused_kernels as F
from paper_2512_24449_b200.kv_store import CompressedStore
from paper_2512_24449_b200.tensor_model import gauss_outlier
B, H, Hq, D, L = 8, 8, 32, 128, 8192
k = gauss_outlier((B, L, H, D), n_outlier=4, seed=1)
v = gauss_outlier((B, L, H, D), n_outlier=1, seed=2)
q = torch.randn((B, Hq, D), device="cuda")
w = torch.softmax(torch.randn((B, Hq, L), device="cuda"), -1)
def t(fn, n=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
for rk, rv in ((0.2, 0.3), (0.1, 0.2), (0.07, 0.15), (0.05, 0.1), (0.03, 0.05), (0.01, 0.02)):
    st = CompressedStore(1, H, D, batch=B, rel_scale_k=rk, rel_scale_v=rv, max_tokens=L, check=False)
    st.compress_batch(0, k, v)
    wh = st.snapshot_stats()
    wide_k = sum(wh[(0, 0)]["width_hist"][5:]) / max(1, sum(wh[(0, 0)]["width_hist"]))
    wide_v = sum(wh[(0, 1)]["width_hist"][5:]) / max(1, sum(wh[(0, 1)]["width_hist"]))
    tk = t(lambda: F.fused_k_scores_batched(st, 0, q))
    tv = t(lambda: F.fused_v_output_batched(st, 0, w))
    print(f"rel_k {rk} rel_v {rv}: K {tk:.1f} us (packs w>4: {wide_k:.3f})  V {tv:.1f} us ({wide_v:.3f})  CR K {wh[(0,0)]['cr']:.2f} V {wh[(0,1)]['cr']:.2f}")
    del st
