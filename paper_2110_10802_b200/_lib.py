"""ctypes binding of the C ABI in ``include/dfx.h`` (``_lib/libdfx_b200.so``).

This is the whole host<->device boundary: every call passes raw device
pointers, extents and a CUDA stream handle.  There is deliberately no CPU
fallback — if the library is missing or the device is not sm_100, importing
the product path raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_void_p

from .errors import ExecError, ShapeError, UnsupportedOp

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libdfx_b200.so")

DFX_F32, DFX_F64, DFX_I64, DFX_BOOL, DFX_BF16, DFX_U8 = 0, 1, 2, 3, 4, 5
EPI_NONE, EPI_BIAS, EPI_BIAS_GELU, EPI_GELU_BWD, EPI_ADD = 0, 1, 2, 3, 4

_STATUS = {1: "shape", 2: "dtype", 3: "align", 4: "cuda", 5: "unsupported", 6: "workspace"}


class GemmArgs(ctypes.Structure):
    """Mirror of ``struct dfx_gemm_args`` (include/dfx.h)."""

    _fields_ = [
        ("in_dtype", c_int32), ("out_dtype", c_int32), ("epilogue", c_int32), ("force_simt", c_int32),
        ("m", c_int64), ("n", c_int64), ("k", c_int64), ("batch1", c_int64), ("batch2", c_int64),
        ("a", c_void_p), ("a_stride_m", c_int64), ("a_stride_k", c_int64),
        ("a_stride_b1", c_int64), ("a_stride_b2", c_int64),
        ("b", c_void_p), ("b_stride_n", c_int64), ("b_stride_k", c_int64),
        ("b_stride_b1", c_int64), ("b_stride_b2", c_int64),
        ("d", c_void_p), ("d_stride_m", c_int64), ("d_stride_b1", c_int64), ("d_stride_b2", c_int64),
        ("alpha", c_float), ("beta", c_float),
        ("bias", c_void_p),
        ("aux", c_void_p), ("aux_stride_m", c_int64), ("aux_stride_b1", c_int64),
        ("aux_stride_b2", c_int64),
        ("aux_out", c_void_p), ("aux_out_stride_m", c_int64), ("aux_out_stride_b1", c_int64),
        ("aux_out_stride_b2", c_int64),
        ("workspace", c_void_p), ("workspace_bytes", c_size_t),
    ]


# (name, restype, argtypes)
_SIGS = [
    ("dfx_last_error", c_char_p, []),
    ("dfx_version", c_int, []),
    ("dfx_device_check", c_int, []),
    ("dfx_launch_count", c_int64, []),
    ("dfx_reset_launch_count", None, []),
    ("dfx_bdrln_fwd", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_float,
                              c_void_p, c_void_p, c_void_p, c_float, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p]),
    ("dfx_bdrln_fwd_kb", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_float,
                                 c_void_p, c_void_p, c_void_p, c_float, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p]),
    ("dfx_bdrln_bwd_workspace", c_size_t, [c_int64, c_int64]),
    ("dfx_bdrln_bwd_kb", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_float, c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_size_t, c_void_p]),
    ("dfx_bdrln_bwd", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_float, c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_size_t, c_void_p]),
    ("dfx_softmax_fwd", c_int, [c_int, c_int64, c_int64, c_int64, c_int64, c_void_p, c_float,
                                c_void_p, c_void_p, c_float, c_void_p, c_void_p, c_void_p]),
    ("dfx_softmax_bwd", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_float,
                                c_float, c_void_p, c_void_p]),
    ("dfx_bias_gelu_fwd", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    ("dfx_bias_gelu_bwd", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_size_t, c_void_p]),
    ("dfx_colsum_workspace", c_size_t, [c_int64, c_int64]),
    ("dfx_colsum", c_int, [c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int, c_void_p,
                           c_size_t, c_void_p]),
    ("dfx_gemm", c_int, [POINTER(GemmArgs), c_void_p]),
    ("dfx_gemm_uses_tensor_cores", c_int, [POINTER(GemmArgs)]),
    ("dfx_gemm_workspace", c_size_t, [POINTER(GemmArgs)]),
    ("dfx_gemm_excite", c_int, [c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dfx_mbconv_workspace", c_size_t, [c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_void_p, c_int]),
    ("dfx_mbconv_fwd_stats", c_int, [c_int, c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_void_p,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                     c_void_p]),
    ("dfx_bn_finalize", c_int, [c_int64, c_int, c_void_p, c_float, c_float, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dfx_mbconv_fwd_se", c_int, [c_int, c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_void_p, c_int64,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_size_t, c_void_p]),
    ("dfx_mbconv_bwd_reduce", c_int, [c_int, c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_void_p,
                                      c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_size_t, c_void_p]),
    ("dfx_mbconv_bwd_dx", c_int, [c_int, c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, ctypes.c_double,
                                  c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("dfx_layernorm_act_fwd", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_float,
                                      c_int, c_void_p, c_void_p]),
    ("dfx_layernorm_act_bwd", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_float, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                      c_void_p]),
    ("dfx_batchnorm_workspace", c_size_t, [c_int64, c_int64]),
    ("dfx_batchnorm_stats", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_size_t,
                                    c_void_p]),
    ("dfx_batchnorm_act_apply", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_int, c_void_p, c_void_p]),
    ("dfx_batchnorm_act_bwd_reduce", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                             c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                             c_size_t, c_void_p]),
    ("dfx_batchnorm_act_bwd_dx", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_int, c_void_p, ctypes.c_double, c_void_p,
                                         c_void_p]),
    ("dfx_batchnorm_stats_finalize", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_float, c_float,
                                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                             c_size_t, c_void_p]),
    ("dfx_batchnorm_act_bwd_reduce_grads", c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                                   c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                                   c_void_p, c_void_p, c_size_t, c_void_p]),
    ("dfx_attn_fwd", c_int, [c_int64, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                             c_float, c_float, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dfx_attn_bwd_workspace", c_size_t, [c_int64, c_int64, c_int64]),
    ("dfx_attn_bwd", c_int, [c_int64, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                             c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_float, c_void_p,
                             c_int64, c_void_p, c_size_t, c_void_p]),
    ("dfx_attn_bwd_bias_grad", c_int, [c_int64, c_int64, c_int64, c_void_p, c_size_t, c_void_p, c_int, c_void_p]),
    ("dfx_im2col3x3", c_int, [c_int, c_int64, c_int64, c_int64, c_int64, c_int, c_void_p, c_int64, c_void_p,
                              c_void_p, c_void_p]),
    ("dfx_avgpool_fwd", c_int, [c_int, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    ("dfx_avgpool_bwd", c_int, [c_int, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    ("dfx_softmax_xent", c_int, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                                 c_void_p]),
    ("dfx_add", c_int, [c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dfx_bdrln_bwd_finalize", c_int, [c_int, c_int64, c_int64, c_void_p, c_size_t, c_void_p, c_void_p, c_void_p,
                                       c_void_p]),
    ("dfx_sgd_update", c_int, [c_int64, c_void_p, c_void_p, c_float, c_void_p, c_void_p]),
    ("dfx_scale_f32", c_int, [c_int64, c_void_p, c_float, c_void_p]),
    ("dfx_cast", c_int, [c_int64, c_int, c_void_p, c_int, c_void_p, c_void_p]),
    ("dfx_cast2", c_int, [c_int64, c_int, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
]

EXPORTED = [name for name, _, _ in _SIGS]

_lib = None
_lock = threading.Lock()


def load(check_device: bool = False):
    """Load the library (once).  Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"dfx CUDA library not found at {LIB_PATH}; run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, res, args in _SIGS:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if check_device:
        rc = _lib.dfx_device_check()
        if rc:
            raise ExecError(_lib.dfx_last_error().decode())
    return _lib


def check(rc: int, what: str = "dfx") -> None:
    if rc == 0:
        return
    msg = _lib.dfx_last_error().decode() if _lib is not None else what
    kind = _STATUS.get(rc, "error")
    if kind in ("shape", "align", "workspace", "dtype"):
        raise ShapeError(f"{msg} [{kind}]")
    if kind == "unsupported":
        raise UnsupportedOp(msg)
    raise ExecError(f"{msg} [{kind}]")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)
