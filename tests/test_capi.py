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


def test_packkv_alias_resolves_to_the_implementation():
    import packkv
    import packkv.errors
    import packkv.fused_kernels
    import paper_2512_24449_b200.errors as E
    import paper_2512_24449_b200.fused_kernels as F
    assert packkv.errors is E and packkv.fused_kernels is F
    assert hasattr(packkv.kv_store, "CompressedStore") and hasattr(packkv.fused_kernels, "fused_k_scores")


def test_errors_subclass_the_installed_reference_classes(tmp_path):
    """With the reference package importable as `packkv` (baseline/_ref, the
    offline install of /root/reference/pkg), every error class of this
    implementation is also the reference class of the same name, so existing
    `except packkv.errors.X` handlers catch it (errors.py:4-41)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.exists(os.path.join(ref, "packkv", "errors.py")):
        pytest.skip("reference package not installed in baseline/_ref")
    import subprocess
    import sys
    pk = tmp_path / "pk"
    pk.mkdir()
    (pk / "paper_2512_24449_b200").symlink_to(os.path.join(ROOT, "paper_2512_24449_b200"))
    code = ("import packkv.errors as R\n"
            "from paper_2512_24449_b200 import errors as E\n"
            "assert R.__file__.startswith(%r)\n"
            "names = ['PackKVError', 'DumpFormatError', 'BadMagicError', 'TruncatedDumpError', 'NonFiniteValueError',\n"
            "         'ShapeMismatchError', 'WidthOverflowError', 'MalformedBlockError', 'InstanceTooLargeError',\n"
            "         'StoreFormatError']\n"
            "for n in names:\n"
            "    assert issubclass(getattr(E, n), getattr(R, n)), n\n"
            "try:\n"
            "    raise E.BadMagicError('x')\n"
            "except R.DumpFormatError:\n"
            "    pass\n"
            "print('ok')\n") % ref
    env = dict(os.environ, PYTHONPATH=f"{ref}{os.pathsep}{pk}")
    r = subprocess.run([sys.executable, "-c", code], cwd=str(tmp_path), env=env, capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr
