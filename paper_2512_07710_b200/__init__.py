"""paper_2512_07710_b200 — the ESPO policy-loss pass (arXiv 2512.07710 §2.4) on B200.

The compute path is libespo.so (hand-written sm_100a CUDA behind the C ABI in
include/espo.h); ``espo`` is its thin ctypes binding. ``build`` compiles the library.
"""
from .build import build_library, LIB_PATH  # noqa: F401

__all__ = ["build_library", "LIB_PATH"]


def __getattr__(name):
    # the binding imports torch; load it lazily so `build` works without touching CUDA
    if name in ("espo", "Espo", "espo_loss", "EspoLossFunction", "EspoError"):
        from . import espo as _e
        return _e if name == "espo" else getattr(_e, name)
    raise AttributeError(name)
