"""Host profile of the GraphedDecodeStep flush and re-capture steps (experiment script)."""
import os, sys, time, cProfile, pstats
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
toks = [(torch.randn(B, H, D, device="cuda").half(), torch.randn(B, H, D, device="cuda").half()) for _ in range(200)]
for t in range(62):
    step(toks[t][0], toks[t][1], q)
torch.cuda.synchronize()
for name, t in (("s63", 63), ("flush", 64), ("recapture", 65), ("s66", 66)):
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    step(toks[t][0], toks[t][1], q)
    pr.disable()
    torch.cuda.synchronize()
    print(f"== {name}: {1e3 * (time.perf_counter() - t0):.3f} ms  nblk {st[0].nblk_h} nres {st[0].nres_h}")
    pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
