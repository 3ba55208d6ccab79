"""``library_eval`` — the drop-in execution seam of the reference interpreter.

The reference executes every LibraryNode through

    _Execution.run_library -> self.library_eval(node.op, node.attrs, inputs)
                                                        interp.py:337-368
    default: frontend.reference_apply(op, attrs, inputs) frontend.py:146-150

with ``inputs`` a list of numpy arrays (possibly views into interpreter
storage) and the result a list of arrays that the interpreter casts and
writes back.  ``library_eval`` below has exactly that signature, so

    dfir.interp.execute(g, inputs, bindings, library_eval=library_eval)

runs the hot-path operators of a dfir graph on the B200.  Each call copies
its host arrays to HBM, runs the device implementation of the operator
(device_ops.py — the same code ``dfm.DeviceGraph`` runs device-resident) on
the sm_100a kernels through the C ABI (include/dfx.h) and copies the results
back.  Operators outside the hot path
raise ``UnsupportedOp`` — there is no CPU fallback.  Attribute
handling follows ``frontend.normalize_attrs`` (registry.py).

Arithmetic is fp32 (the tensor cores are used for bf16 only).  The reference
evaluates every operator in float64 and casts back to the input dtype
(frontend.py:146-150, 216-218); for f32 graphs that is what happens here too
(fp32 arithmetic, f32 results).  f64 graphs are REJECTED by default — the B200
path has no f64 arithmetic and silently computing in fp32 would change the
reference's numerics; ``make_library_eval(f64="as_f32")`` opts in explicitly
(results are cast back to f64).

``Reshape`` / ``Flatten`` are pure metadata in row-major storage (no bytes
move, no arithmetic); they are answered with a view of the input so a graph
that keeps them as library nodes still runs.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device_ops import DEVICE_OPS, run_op
from .errors import ShapeError, UnsupportedOp
from .registry import get_op, normalize_attrs

__all__ = ["library_eval", "SUPPORTED_OPS"]


_POLICY = {"f64": "reject"}


def _dev(a, dtype=torch.float32):
    arr = np.asarray(a)
    if arr.dtype == np.float64 and _POLICY["f64"] != "as_f32":
        raise ShapeError("B200 path computes in fp32: f64 operands are rejected (the reference evaluates f64; "
                         "use make_library_eval(f64='as_f32') to accept fp32 arithmetic explicitly)")
    if arr.dtype not in (np.float32, np.float64):
        raise ShapeError(f"B200 path takes f32 tensors, got {arr.dtype}")
    # a private, writable, contiguous fp32 copy: the interpreter hands in
    # read-only views of its storage (interp.py:348)
    host = torch.from_numpy(np.array(arr, dtype=np.float32, order="C", copy=True))
    return host.to("cuda", dtype=dtype)


def _host(t, like):
    return t.float().cpu().numpy().astype(np.asarray(like).dtype, copy=False)


def _reshape_host(attrs, inputs):
    """Reshape / Flatten are metadata on row-major storage (frontend.py:713-829):
    answered with a view of the host array, no device traffic."""
    x = np.asarray(inputs[0])
    if "axis" in attrs:  # Flatten
        ax = int(attrs["axis"]) % max(x.ndim, 1)
        return [x.reshape(int(np.prod(x.shape[:ax], dtype=np.int64)), -1)]
    shape = [int(v) for v in attrs["shape"]]
    shape = [x.shape[i] if v == 0 else v for i, v in enumerate(shape)]
    return [x.reshape(shape)]


SUPPORTED_OPS = sorted(DEVICE_OPS)


def library_eval(op: str, attrs, inputs):
    """Evaluate one operator on the B200 (same contract as
    frontend.reference_apply).  Raises UnsupportedOp for operators that are
    not on the hot path — never falls back to the CPU."""
    if op not in DEVICE_OPS:
        raise UnsupportedOp(op)
    spec = get_op(op)
    if not (spec.min_inputs <= len(inputs) <= spec.max_inputs):
        raise ShapeError(f"{op}: takes {spec.min_inputs}..{spec.max_inputs} inputs, got {len(inputs)}")
    norm = normalize_attrs(spec, attrs)
    if op in ("Reshape", "Flatten"):
        return _reshape_host(norm, inputs)
    _lib.load(check_device=True)
    outs = run_op(op, norm, [_dev(x) for x in inputs])
    # results come back as host arrays in the first input's dtype (the seam's
    # contract, frontend.py:216-218); the D2H copies order them after the kernels
    return [_host(o, inputs[0]) for o in outs]


def make_library_eval(f64: str = "reject"):
    """A ``library_eval`` with an explicit f64 policy: ``"reject"`` (default,
    raise ShapeError) or ``"as_f32"`` (compute in fp32, cast results back)."""
    if f64 not in ("reject", "as_f32"):
        raise ValueError("f64 policy must be 'reject' or 'as_f32'")

    def evaluate(op, attrs, inputs):
        saved = _POLICY["f64"]
        _POLICY["f64"] = f64
        try:
            return library_eval(op, attrs, inputs)
        finally:
            _POLICY["f64"] = saved

    return evaluate
