"""B200-native (sm_100a) fused training hot path of arXiv 2110.10802 (DaCeML).

The package is the drop-in execution layer for the reference ``dfir``
operator API: ``library_eval`` (the interp.py:337-368 seam), fused-operator
specs mirroring ``frontend.OpSpec`` (frontend.py:73-89), the BERT encoder
layer and MBConv training steps, and the data-parallel runtime — all
calling hand-written CUDA kernels through the C ABI in ``include/dfx.h``.
"""

from .errors import ExecError, ModelError, ShapeError, UnsupportedOp  # noqa: F401

__all__ = ["ExecError", "ModelError", "ShapeError", "UnsupportedOp"]
