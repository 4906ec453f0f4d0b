"""Small workload covering every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): the single-pass compressor (decoupled
look-back, tickets), the device-side flush + staging (pkv_append_flush), the
fused fast K / V kernels (per-warp TMA rings, mbarriers), the single-pass
attention and its merge, the three-launch attention, and the generic path.
usage: compute-sanitizer --tool memcheck python tools/sanitize_workload.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_24449_b200 import fused_kernels as F  # noqa: E402
from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop, attention_decode_batched  # noqa: E402
from paper_2512_24449_b200.kv_store import CompressedStore  # noqa: E402

rng = np.random.default_rng(1)
B, H, D, G, T = 2, 2, 128, 4, 64 * 9 + 37
k = torch.from_numpy(rng.standard_normal((B, T, H, D)).astype(np.float16)).cuda()
v = torch.from_numpy(rng.standard_normal((B, T, H, D)).astype(np.float16)).cuda()
st = CompressedStore(1, H, D, batch=B, check=False)
st.compress_batch(0, k[:, :300], v[:, :300])
for t in range(300, 330):
    st.append_token(0, k[:, t], v[:, t])
q = torch.randn((B, H * G, D), device="cuda")
w = torch.softmax(torch.randn((B, H * G, st[0].tokens), device="cuda"), -1)
F.fused_k_scores_batched(st, 0, q)
F.fused_v_output_batched(st, 0, w)
attention_decode_batched(st, 0, q, single_pass=True)
attention_decode_batched(st, 0, q, single_pass=False)
q8 = torch.randn((B, H * 8, D), device="cuda")
attention_decode_batched(st, 0, q8, single_pass=True)
# wide packs / scalar paths (tight rel)
st2 = CompressedStore(1, H, D, batch=B, rel_scale_k=0.02, rel_scale_v=0.03, check=False)
st2.compress_batch(0, k, v)
F.fused_k_scores_batched(st2, 0, q)
attention_decode_batched(st2, 0, q, single_pass=True)
# generic format (pack 8)
st3 = CompressedStore(1, H, D, batch=B, pack_size=8, check=False)
st3.compress_batch(0, k[:, :200], v[:, :200])
F.fused_k_scores_batched(st3, 0, q)
# decode loop: stage + flush in one launch, then attention
st4 = CompressedStore(1, H, D, batch=B, check=False)
st4.compress_batch(0, k[:, :60], v[:, :60])
loop = GraphedDecodeLoop(st4, H * G, headroom=2)
for t in range(60, 72):
    loop.step(k[None, :, t:t + 1], v[None, :, t:t + 1], q[None])
# ragged: prefill by lengths (masked append-flush), then a masked decode loop
st5 = CompressedStore(1, H, D, batch=B, check=False)
st5.compress_batch(0, k[:, :140], v[:, :140], lengths=[140, 70])
loop5 = GraphedDecodeLoop(st5, H * G, headroom=2)
for t in range(8):
    loop5.step(k[None, :, t:t + 1], v[None, :, t:t + 1], q[None], active=[t % 2 == 0, True])
torch.cuda.synchronize()
for s in (st, st2, st3, st4, st5):
    s.check_errors()
print("sanitize workload ok")
