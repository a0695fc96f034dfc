"""Kernel seam: the one backend is the sm_100a CUDA library.

Drop-in for the reference's ``shockhash._kernels`` module
(/root/reference/pkg/src/shockhash/_kernels/__init__.py:10-38): ``kernels``,
``BACKEND_NAME``, ``HAS_COMPILED`` and ``get_backend`` keep their meaning, but
there is no pure-Python or Cython alternative to select — asking for one
fails loudly rather than silently running on the CPU.
"""

from . import _cuda

kernels = _cuda
BACKEND_NAME = _cuda.NAME
HAS_COMPILED = True  # the backend is native (CUDA) code


def get_backend(name=None):
    """Return the kernel module ('cuda' / 'compiled' / None = active)."""
    if name in (None, "cuda", "compiled"):
        return _cuda
    raise ValueError(f"unknown backend {name!r}: this package has exactly one backend (CUDA, sm_100a)")
