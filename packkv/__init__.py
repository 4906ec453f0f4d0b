"""``packkv`` import alias for the B200-native hot path.

The reference ships its API as the ``packkv`` package (``pkg/src/packkv``,
SPEC.md module names); a caller that switches to this implementation keeps
its imports: ``import packkv.kv_store``, ``from packkv.fused_kernels import
fused_k_scores``, ``except packkv.errors.ShapeMismatchError`` resolve to the
modules of ``paper_2512_24449_b200`` (the same module objects, so classes and
isinstance checks agree).  Put the repository root on ``sys.path`` ahead of
any installed reference package to select it.
"""
import importlib
import sys

import paper_2512_24449_b200 as _impl

_MODULES = ("errors", "quantizer", "repacker", "bitpack_codec", "kv_store", "fused_kernels", "attention_sim",
            "tensor_model", "sharding")

for _m in _MODULES:
    _mod = importlib.import_module(f"paper_2512_24449_b200.{_m}")
    sys.modules[f"{__name__}.{_m}"] = _mod
    globals()[_m] = _mod

__version__ = _impl.__version__
__all__ = list(_MODULES)
