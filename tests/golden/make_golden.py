"""Generates tests/golden/packkv_golden.npz from the CPU oracle (SPEC.md
restatement, pinned to the SPEC known-answer examples).  The reference ships
no implementation to run, so these frozen vectors are the de-facto reference
outputs: the CPU suite checks the oracle still reproduces them bit-for-bit and
the GPU suite checks the CUDA path against them.  Re-run only on purpose:

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import packkv_oracle as O  # noqa: E402


def main():
    rng = np.random.default_rng(20251224)
    g = {}
    # quantizer: SPEC example rows, ties, constant rows, random rows at 3 scales
    qx = (rng.standard_normal((3, 64, 128)) * rng.uniform(0.01, 20, (3, 64, 1))).astype(np.float16)
    qx[0, 0, :3] = [0.0, 0.34, 1.0]
    qx[0, 1, :] = 5.0
    qx[0, 2, :3] = [0, 0.25, 1]
    g["quant_x"] = qx
    for rel in (0.05, 0.1, 0.2):
        tag = str(rel).replace(".", "p")
        q = [O.quantize_token_wise(x, rel) for x in qx]
        g[f"quant_q_{tag}"] = np.stack([b.q for b in q]).astype(np.uint16)
        g[f"quant_scale_{tag}"] = np.stack([b.scale for b in q])
        g[f"quant_zp_{tag}"] = np.stack([b.zp for b in q])
    # codec: every pack size x layout, random codes/params, incl. 15-bit packs
    for k in O.PACK_SIZES:
        for layout in (0, 1):
            cols = 37 if k in (2, 8, 32) else 48   # ragged K-interleave generalisation too
            codes = rng.integers(0, 1 << int(rng.integers(1, 12)), (64, cols))
            codes[0, 0] = 32767
            scale = rng.uniform(0.01, 2, 64).astype(np.float32)
            zp = rng.uniform(-3, 3, 64).astype(np.float16).astype(np.float32)
            blk = O.encode_block(O.QuantBlock(codes, scale, zp, layout), k, layout, layout)
            g[f"enc_codes_k{k}_l{layout}"] = codes.astype(np.uint16)
            g[f"enc_scale_k{k}_l{layout}"] = scale
            g[f"enc_zp_k{k}_l{layout}"] = zp
            g[f"enc_bytes_k{k}_l{layout}"] = np.frombuffer(blk, np.uint8)
            g[f"enc_cr_k{k}_l{layout}"] = np.float64(O.compression_ratio(blk))
    # store + fused: gaussian-with-outliers KV, 3 repack strategies, residue 17 tokens
    H, D, T, G = 2, 128, 64 * 3 + 17, 4
    K = np.stack([O.gen_gauss_outlier(rng, T, D, 4) for _ in range(H)], 1)
    V = np.stack([O.gen_gauss_outlier(rng, T, D, 1) for _ in range(H)], 1)
    q = rng.standard_normal((H * G, D)).astype(np.float32)
    w = rng.random((H * G, T)).astype(np.float32)
    g["store_K"], g["store_V"], g["store_q"], g["store_w"] = K, V, q, w
    for rp in ("none", "v_median", "greedy"):
        st = O.OracleStore(1, H, D, repack=rp)
        st.compress_batch(0, K, V)
        g[f"store_stream_{rp}"] = np.frombuffer(st.layer_stream(0), np.uint8)
        g[f"store_perm_{rp}"] = np.stack([e.permutation for e in st.directory if e.kind == 0 and e.head == 0])
        g[f"store_scores_{rp}"] = np.stack([O.naive_k_scores(st, 0, hq // G, q[hq]) for hq in range(H * G)])
        g[f"store_out_{rp}"] = np.stack([O.naive_v_output(st, 0, hq // G, w[hq]) for hq in range(H * G)])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "packkv_golden.npz")
    np.savez_compressed(path, **g)
    print(path, os.path.getsize(path), "bytes", len(g), "arrays")


if __name__ == "__main__":
    main()
