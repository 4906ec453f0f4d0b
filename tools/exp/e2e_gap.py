"""Where the config-B e2e time goes (experiment script): graph replay alone, + H2D of q,
+ D2H of the output, both, and the prescale kernel's share."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2512_24449_b200.attention_sim import GraphedAttention

cfg = bench.CONFIGS["B"]
B, Hkv, Hq, D, L = cfg[:5]
st = bench.build_store(cfg, 0)
ga = GraphedAttention(st, 0)
qd = torch.randn((B, Hq, D), device="cuda")
qh = torch.randn((B, Hq, D)).pin_memory()
oh = torch.empty((B, Hq, D)).pin_memory()
ga(qd)
torch.cuda.synchronize()


def timed(fn, K=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3


def replay():
    ga._graph.replay()


def h2d():
    ga._q.copy_(qh, non_blocking=True)
    ga._graph.replay()


def d2h():
    ga._graph.replay()
    oh.copy_(ga._out, non_blocking=True)


def both():
    ga._q.copy_(qh, non_blocking=True)
    ga._graph.replay()
    oh.copy_(ga._out, non_blocking=True)


def copies_only():
    ga._q.copy_(qh, non_blocking=True)
    oh.copy_(ga._out, non_blocking=True)


def prescale():
    ga._q.mul_(1.0)


for name, fn in [("replay", replay), ("h2d+replay", h2d), ("replay+d2h", d2h), ("h2d+replay+d2h", both),
                 ("h2d+d2h only", copies_only), ("one elementwise kernel", prescale)]:
    print(f"{name:24s} {timed(fn):8.2f} us")
