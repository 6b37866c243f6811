"""gCCTB-B200: B200-native batched OLTP concurrency control (arXiv 2406.10158 hot path).

``gcctb`` is the ctypes binding of the C ABI (include/gcctb.h); ``api`` wraps it with
torch-tensor result buffers.  The product path never imports ``oracle`` and has no
CPU fallback: if libgcctb.so is missing, ``gcctb.lib()`` raises.
"""
from . import gcctb  # noqa: F401
from .gcctb import SCHEMES, SCHEME_ID, CCError  # noqa: F401
