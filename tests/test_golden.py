"""Frozen golden vectors (tests/golden/make_golden.py): the CPU oracle must keep
reproducing them bit-for-bit; the CUDA path must match them (bytes exactly,
GEMV outputs within 1e-3 of ||ref||_inf)."""
import os

import numpy as np
import pytest

from oracle import packkv_oracle as O

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "packkv_golden.npz"))
RELS = (0.05, 0.1, 0.2)


def _tag(rel):
    return str(rel).replace(".", "p")


@pytest.mark.parametrize("rel", RELS)
def test_oracle_quantizer_golden(rel):
    for i, x in enumerate(GOLD["quant_x"]):
        qb = O.quantize_token_wise(x, rel)
        assert np.array_equal(qb.q, GOLD[f"quant_q_{_tag(rel)}"][i].astype(np.int64))
        assert np.array_equal(qb.scale, GOLD[f"quant_scale_{_tag(rel)}"][i])
        assert np.array_equal(qb.zp, GOLD[f"quant_zp_{_tag(rel)}"][i])


@pytest.mark.parametrize("k", O.PACK_SIZES)
@pytest.mark.parametrize("layout", [0, 1])
def test_oracle_codec_golden(k, layout):
    t = f"k{k}_l{layout}"
    qb = O.QuantBlock(GOLD[f"enc_codes_{t}"].astype(np.int64), GOLD[f"enc_scale_{t}"], GOLD[f"enc_zp_{t}"], layout)
    blk = O.encode_block(qb, k, layout, layout)
    assert blk == GOLD[f"enc_bytes_{t}"].tobytes()
    assert O.compression_ratio(blk) == float(GOLD[f"enc_cr_{t}"])
    assert np.array_equal(O.decode_block(blk).q, qb.q)


@pytest.mark.parametrize("repack", ["none", "v_median"])
def test_oracle_store_golden(repack):
    st = O.OracleStore(1, 2, 128, repack=repack)
    st.compress_batch(0, GOLD["store_K"], GOLD["store_V"])
    assert st.layer_stream(0) == GOLD[f"store_stream_{repack}"].tobytes()


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("rel", RELS)
def test_gpu_quantizer_golden(rel):
    import torch
    from paper_2512_24449_b200 import quantizer as Q
    qb = Q.quantize_token_wise(torch.from_numpy(GOLD["quant_x"]).cuda(), rel)
    assert np.array_equal(qb.q.cpu().numpy(), GOLD[f"quant_q_{_tag(rel)}"])
    assert np.array_equal(qb.scale.cpu().numpy(), GOLD[f"quant_scale_{_tag(rel)}"])
    assert np.array_equal(qb.zp.cpu().numpy(), GOLD[f"quant_zp_{_tag(rel)}"])


@pytest.mark.gpu
@pytest.mark.parametrize("k", O.PACK_SIZES)
@pytest.mark.parametrize("layout", [0, 1])
def test_gpu_codec_golden(k, layout):
    import torch
    from paper_2512_24449_b200 import bitpack_codec as C, quantizer as Q
    t = f"k{k}_l{layout}"
    qb = Q.QuantBlock(torch.from_numpy(GOLD[f"enc_codes_{t}"].astype(np.int32)).to(torch.uint16).cuda(),
                      torch.from_numpy(GOLD[f"enc_scale_{t}"]).cuda(), torch.from_numpy(GOLD[f"enc_zp_{t}"]).cuda(),
                      layout)
    blk = C.encode_block(qb, k, layout)
    assert blk.to_bytes() == GOLD[f"enc_bytes_{t}"].tobytes()
    assert C.compression_ratio(blk) == float(GOLD[f"enc_cr_{t}"])
    dec = C.decode_block(C.PackedBlock.from_bytes(GOLD[f"enc_bytes_{t}"].tobytes()))
    assert np.array_equal(dec.q.cpu().numpy(), GOLD[f"enc_codes_{t}"])


@pytest.mark.gpu
@pytest.mark.parametrize("repack", ["none", "v_median", "greedy"])
def test_gpu_store_and_fused_golden(repack):
    import torch
    from paper_2512_24449_b200 import fused_kernels as F
    from paper_2512_24449_b200.kv_store import CompressedStore
    st = CompressedStore(1, 2, 128, repack=repack)
    st.compress_batch(0, GOLD["store_K"], GOLD["store_V"])
    assert st[0].stream_bytes(0) == GOLD[f"store_stream_{repack}"].tobytes()
    q = torch.from_numpy(GOLD["store_q"])[None]
    w = torch.from_numpy(GOLD["store_w"])[None]
    s = F.fused_k_scores_batched(st, 0, q)[0].cpu().numpy().astype(np.float64)
    o = F.fused_v_output_batched(st, 0, w)[0].cpu().numpy().astype(np.float64)
    rs, ro = GOLD[f"store_scores_{repack}"], GOLD[f"store_out_{repack}"]
    assert np.abs(s - rs).max() <= 1e-3 * np.abs(rs).max()
    assert np.abs(o - ro).max() <= 1e-3 * np.abs(ro).max()
