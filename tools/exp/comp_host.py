"""Host-side breakdown of a prefill compress (experiment script)."""
import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2512_24449_b200.kv_store import CompressedStore
from paper_2512_24449_b200.tensor_model import gauss_outlier
from paper_2512_24449_b200 import _native as N
B, H, D, T = 8, 8, 128, 4096
k = gauss_outlier((B, T, H, D), n_outlier=4, seed=1)
v = gauss_outlier((B, T, H, D), n_outlier=1, seed=2)
for rep in range(4):
    st = CompressedStore(1, H, D, batch=B, max_tokens=T + 128, check=False)
    ls = st[0]
    ls._ensure(T // 64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    st.compress_batch(0, k, v)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: host call {1e3*(t1-t0):.3f} ms, until done {1e3*(t2-t0):.3f} ms, gpu events {e0.elapsed_time(e1):.3f} ms")
# raw C call on a warm store (no python around it)
st = CompressedStore(1, H, D, batch=B, max_tokens=T + 128, check=False)
ls = st[0]; ls._ensure(T // 64)
st.compress_batch(0, k[:, :64].contiguous(), v[:, :64].contiguous())
torch.cuda.synchronize()
L = ls.struct(); lib = N.lib()
from paper_2512_24449_b200.kv_store import ctypes_ref
kc, vc = k[:, :4032].contiguous(), v[:, :4032].contiguous()
torch.cuda.synchronize()
e0.record(); t0 = time.perf_counter()
rc = lib.pkv_compress_tokens(ctypes_ref(L), N.ptr(kc), N.ptr(vc), 4032, 0, 1, 0.1, 0.2, 0, N.ptr(ls.scratch), int(ls.scratch.numel()), N.stream())
t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
print(f"raw C call: rc {rc} host {1e3*(t1-t0):.3f} ms gpu {e0.elapsed_time(e1):.3f} ms scratch {ls.scratch.numel()>>20} MB")
