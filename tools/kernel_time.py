"""Time the fused K / V kernels alone on config B (for A/B experiments)."""
import sys, os, math, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_24449_b200 import fused_kernels as F
cfg = bench.CONFIGS["B"]
B, Hkv, Hq, D, L, _ = cfg
st = bench.build_store(cfg, 0)
q = torch.randn((B, Hq, D), device="cuda")
scores = torch.empty((B, Hq, L), device="cuda")
w = torch.softmax(torch.randn((B, Hq, L), device="cuda"), -1)
out = torch.empty((B, Hq, D), device="cuda")
which = sys.argv[1:] or ["k", "v"]
for name in which:
    fn = (lambda: F.fused_k_scores_batched(st, 0, q, out=scores)) if name == "k" else (lambda: F.fused_v_output_batched(st, 0, w, out=out))
    for _ in range(5):
        fn()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, "median us", round(statistics.median(ts), 2))
