"""Prefill compressor timing (experiment script): config-B shapes, 4096 tokens x batch 8 x
8 kv-heads, K and V, arena reserved; median CUDA-event time of compress_batch."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2512_24449_b200.kv_store import CompressedStore
from paper_2512_24449_b200.tensor_model import gauss_outlier
B, H, D, T = 8, 8, 128, 4096
k = gauss_outlier((B, T, H, D), n_outlier=4, seed=1).cuda()
v = gauss_outlier((B, T, H, D), n_outlier=1, seed=2).cuda()
ts = []
ref = None
for rep in range(12):
    st = CompressedStore(1, H, D, batch=B, max_tokens=T + 128, check=False)
    ls = st[0]
    ls._ensure(T // 64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.compress_batch(0, k, v)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    t = int(ls.tail.item())  # total padded bytes: order-independent
    ref = t if ref is None else ref
    assert ref == t and int(ls.err.item()) == 0, (ref, t)
ts = sorted(ts[2:])
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'lib'}: prefill median {ts[len(ts)//2]*1e3:.1f} us min {ts[0]*1e3:.1f} us "
      f"({2*B*H*T*D*2/ (ts[len(ts)//2]*1e-3) / 1e9:.0f} GB/s fp16 in)")
