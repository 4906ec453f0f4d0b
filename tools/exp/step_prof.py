"""Per-step timing of GraphedDecodeStep (experiment script)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2512_24449_b200.kv_store import CompressedStore
from paper_2512_24449_b200.attention_sim import GraphedDecodeStep
B, H, D, T, Hq = 8, 8, 128, 4096, 32
st = CompressedStore(1, H, D, batch=B, max_tokens=T + 256, check=False)
st[0]._ensure((T + 256) // 64)
k = torch.randn(B, T, H, D, device="cuda").half(); v = torch.randn(B, T, H, D, device="cuda").half()
st.compress_batch(0, k, v)
step = GraphedDecodeStep(st, 0)
q = torch.randn(B, Hq, D, device="cuda")
toks = [(torch.randn(B, H, D, device="cuda").half(), torch.randn(B, H, D, device="cuda").half()) for _ in range(140)]
torch.cuda.synchronize()
ts = []
for t in range(140):
    t0 = time.perf_counter()
    step(toks[t][0], toks[t][1], q)
    torch.cuda.synchronize()
    ts.append(1e6 * (time.perf_counter() - t0))
big = [(i, round(x)) for i, x in enumerate(ts) if x > 200]
print("slow steps:", big)
norm = sorted(x for x in ts if x <= 200)
print(f"median {norm[len(norm)//2]:.1f} us, captures {step.captures}")
# host-only cost of a replay step
t0 = time.perf_counter()
for t in range(20):
    step(toks[t][0], toks[t][1], q)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"20 steps: host {1e6*(t1-t0)/20:.1f} us/step, total {1e6*(t2-t0)/20:.1f} us/step")
