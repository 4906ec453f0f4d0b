"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/packkv_b200.h declares; the Python surface
mirrors the reference module/function names; no CPU fallback exists."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "packkv_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pkv_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for s in ("pkv_quantize", "pkv_encode", "pkv_decode", "pkv_compress_tokens", "pkv_fused_k_scores",
              "pkv_fused_v_output", "pkv_last_error", "pkv_version"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2512_24449_b200 import _native as N
    if not os.path.exists(N.LIB_PATH):
        import subprocess
        subprocess.run(["make", "-C", ROOT, "-j", "8"], check=True)
    lib = ctypes.CDLL(N.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} not exported"
    assert set(declared_symbols()) == set(N.exported_symbols())
    N.load()
    assert lib.pkv_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_24449_b200 import _native as N
    from paper_2512_24449_b200.kv_store import CompressedStore
    with pytest.raises(RuntimeError):
        CompressedStore(1, 2, 64)
    with pytest.raises(RuntimeError):
        N.lib()


def test_reference_module_names_present():
    import importlib
    for m in ("errors", "quantizer", "bitpack_codec", "kv_store", "fused_kernels", "attention_sim"):
        importlib.import_module(f"paper_2512_24449_b200.{m}")
    from paper_2512_24449_b200 import errors as E
    for cls in ("PackKVError", "DumpFormatError", "BadMagicError", "TruncatedDumpError", "NonFiniteValueError",
                "ShapeMismatchError", "WidthOverflowError", "MalformedBlockError", "InstanceTooLargeError",
                "StoreFormatError"):
        assert issubclass(getattr(E, cls), E.PackKVError)
    from paper_2512_24449_b200 import fused_kernels as F, kv_store as S, bitpack_codec as C, quantizer as Q
    for f in ("fused_k_scores", "fused_v_output", "naive_k_scores", "naive_v_output", "bench_throughput"):
        assert callable(getattr(F, f))
    for f in ("append_token", "compress_batch", "iterate_blocks", "snapshot_stats"):
        assert callable(getattr(S, f))
    for f in ("encode_block", "decode_block", "decode_pack_at", "compression_ratio", "kivi_baseline_cr"):
        assert callable(getattr(C, f))
    for f in ("quantize_token_wise", "dequantize", "max_abs_error"):
        assert callable(getattr(Q, f))


def test_native_error_mapping():
    from paper_2512_24449_b200 import _native as N, errors as E
    with pytest.raises(E.ShapeMismatchError):
        N.check(N.PKV_E_SHAPE)
    with pytest.raises(E.MalformedBlockError):
        N.raise_flags(N.FLAG_MALFORMED)
    with pytest.raises(E.NonFiniteValueError):
        N.raise_flags(N.FLAG_NONFINITE | N.FLAG_WIDTH)
    with pytest.raises(IndexError):
        N.check(N.PKV_E_INDEX)
