"""Host profile of single-token appends (experiment script)."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_2512_24449_b200.kv_store import CompressedStore
B, H, D = 8, 8, 128
st = CompressedStore(1, H, D, batch=B, max_tokens=4096, check=False)
kk = torch.randn(300, B, H, D, device="cuda").half()
vv = torch.randn(300, B, H, D, device="cuda").half()
for t in range(10):
    st.append_token(0, kk[t], vv[t])
torch.cuda.synchronize()
t0 = time.perf_counter()
for t in range(10, 138):
    st.append_token(0, kk[t], vv[t])
torch.cuda.synchronize()
print(f"append: {1e6 * (time.perf_counter() - t0) / 128:.1f} us/token (wall)")
pr = cProfile.Profile(); pr.enable()
for t in range(138, 266):
    st.append_token(0, kk[t], vv[t])
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
