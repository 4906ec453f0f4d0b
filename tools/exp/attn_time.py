"""Device time of the attention graph (K ST + V SM + finalize) vs plain fused K + V (experiment)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2512_24449_b200 import fused_kernels as F
from paper_2512_24449_b200.attention_sim import GraphedAttention
cfg = bench.CONFIGS["B"]
B, Hkv, Hq, D, L, _ = cfg
st = bench.build_store(cfg, 0)
q = torch.randn((B, Hq, D), device="cuda")
ga = GraphedAttention(st, 0)
ga(q)
scores = torch.empty((B, Hq, L), device="cuda")
w = torch.softmax(torch.randn((B, Hq, L), device="cuda"), -1)
out = torch.empty((B, Hq, D), device="cuda")
gk, gv = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
F.fused_k_scores_batched(st, 0, q, out=scores); F.fused_v_output_batched(st, 0, w, out=out)
with torch.cuda.graph(gk):
    F.fused_k_scores_batched(st, 0, q, out=scores)
with torch.cuda.graph(gv):
    F.fused_v_output_batched(st, 0, w, out=out)
def t(fn, n=30):
    for _ in range(5): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
print(f"attention graph {t(lambda: ga._graph.replay()):.1f} us; plain K {t(gk.replay):.1f} + V {t(gv.replay):.1f} us")
