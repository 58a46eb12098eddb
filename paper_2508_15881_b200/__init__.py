"""TPLA decode hot path for B200 (sm_100a): Python binding of libtpla.so.

    from paper_2508_15881_b200 import abi, runtime

``abi`` is the thin ctypes binding of include/tpla.h (same function names);
``runtime.TplaRank`` allocates one rank's device buffers with PyTorch and calls it.
Loading ``abi`` (or ``runtime``) raises if libtpla.so has not been built: there is no
CPU fallback.  ``build`` compiles the library and needs neither.
"""
import importlib

__all__ = ["abi", "runtime", "build"]


def __getattr__(name):
    if name == "abi":
        return importlib.import_module("._abi", __name__)
    if name in ("runtime", "build"):
        return importlib.import_module("." + name, __name__)
    raise AttributeError(name)
