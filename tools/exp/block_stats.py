"""Per-block fast-path eligibility of a K layer at a given rel (diagnostic)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2512_24449_b200.kv_store import CompressedStore
from paper_2512_24449_b200.tensor_model import gauss_outlier
B, H, D, L = 2, 8, 128, 2048
rk = float(sys.argv[1])
k = gauss_outlier((B, L, H, D), n_outlier=4, seed=1)
v = gauss_outlier((B, L, H, D), n_outlier=1, seed=2)
st = CompressedStore(1, H, D, batch=B, rel_scale_k=rk, rel_scale_v=0.2, max_tokens=L, check=False)
st.compress_batch(0, k, v)
arena = st[0].arena.cpu().numpy()
off, ln, _ = st[0].tables()
bad_w = bad_min = 0; maxlen = 0; n = 0; mins_max = []
for u in range(B * H):
    for j in range(st[0].nblk_h):
        o, l = int(off[0, u, j]), int(ln[0, u, j])
        blk = arena[o:o + l]
        nib = blk[8:8 + 256]
        w = np.stack([nib & 15, nib >> 4], 1).ravel()
        mins = blk[264:264 + 1024].view(np.uint16)
        n += 1; maxlen = max(maxlen, l)
        bad_w += int((w > 4).any()); bad_min += int((mins > 240).any())
        mins_max.append(int(mins.max()))
print(f"rel_k {rk}: blocks {n}, any w>4: {bad_w}, any min>240: {bad_min}, max len {maxlen}, max min {max(mins_max)}")
