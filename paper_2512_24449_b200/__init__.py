"""B200-native PackKV decode-time hot path (arXiv 2512.24449).

Drop-in for the reference ``packkv`` package's hot-path modules:
``quantizer``, ``repacker``, ``bitpack_codec``, ``kv_store``, ``fused_kernels``,
``attention_sim``, ``tensor_model``, ``errors``.  Compute runs in libpackkv_b200.so (sm_100a
CUDA kernels behind the C ABI in include/packkv_b200.h); there is no CPU
fallback.  ``import paper_2512_24449_b200 as packkv`` gives the reference's
module names.
"""
from . import errors
from . import _native

__all__ = ["errors", "quantizer", "repacker", "bitpack_codec", "kv_store", "fused_kernels", "attention_sim",
           "tensor_model", "sharding"]
__version__ = "0.1.0"


def __getattr__(name):
    if name in __all__:
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
