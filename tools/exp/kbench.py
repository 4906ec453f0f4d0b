"""Fast A/B timing of the fused kernels on config-B shapes (graph-replayed, CUDA events).
usage: python tools/exp/kbench.py [k|v|a ...] [--cfg B|E|D|A] [--reps N]"""
import sys, os, statistics, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
from paper_2512_24449_b200 import fused_kernels as F
from paper_2512_24449_b200.attention_sim import attention_decode_batched

ap = argparse.ArgumentParser()
ap.add_argument("which", nargs="*", default=["k", "v"])
ap.add_argument("--cfg", default="B")
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
if a.cfg.startswith("BL"):  # config B shape at another context length, e.g. BL4352
    cfg = (8, 8, 32, 128, int(a.cfg[2:]), f"config B shape at {a.cfg[2:]} tokens")
else:
    cfg = bench.CONFIGS[a.cfg]
B, Hkv, Hq, D, L = cfg[:5]
st = bench.build_store(cfg, 0)
ls = st[0]
_, ln, _ = ls.tables()
phys = {0: float(ln[0].astype("int64").sum()), 1: float(ln[1].astype("int64").sum())}
q = torch.randn((B, Hq, D), device="cuda")
scores = torch.empty((B, Hq, L), device="cuda")
w = torch.softmax(torch.randn((B, Hq, L), device="cuda"), -1)
out = torch.empty((B, Hq, D), device="cuda")
fns = {"k": lambda: F.fused_k_scores_batched(st, 0, q, out=scores),
       "v": lambda: F.fused_v_output_batched(st, 0, w, out=out),
       "a": lambda: attention_decode_batched(st, 0, q, scores=scores, out=out, single_pass=False),
       "s": lambda: attention_decode_batched(st, 0, q, out=out, single_pass=True)}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in a.which:
    fn = fns[name]
    for _ in range(3):
        fn()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin(); fn(); g.capture_end()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):  # 16 back-to-back replays per event pair (timer granularity ~2 us)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(16):
            g.replay()
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 16)
    t = statistics.median(ts)
    extra = {"k": B * Hq * L * 4 + B * Hq * D * 4, "v": B * Hq * L * 4 + B * Hq * D * 4, "a": 0, "s": 0}[name]
    pb = (phys[0] if name == "k" else phys[1] if name == "v" else phys[0] + phys[1]) + extra
    print(f"{a.cfg} {name}: {t:.2f} us  phys {pb / t / 1e3:.0f} GB/s  frac {pb / t / 1e3 / 6532.9:.3f}  equiv {B*Hkv*L*D*2*(2 if name in 'as' else 1)/t/1e3:.0f} GB/s")
