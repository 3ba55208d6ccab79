"""Operator specs of the B200 path, mirroring ``dfir.frontend.OpSpec``.

The reference keeps one registry entry per operator (frontend.py:73-89):
name, attribute schema, input/output arity, shape inference, a numpy
reference, and later-attached lowering/backward builders.  ``register_op``
refuses duplicates (frontend.py:95-98) and ``normalize_attrs`` fills
defaults, rejects unknown attribute names and requires mandatory ones
(frontend.py:112-129).  This module restates that contract for

* the reference operators the B200 path executes (``HOT_OPS``), with the
  reference's own attribute schemas and defaults, and
* the fused operators it adds (``FUSED_OPS``), each documented by the chain
  of registry operators it replaces.

``register_with_dfir(frontend)`` installs the fused operators into a live
``dfir`` registry (when the reference package is importable): their
``reference`` evaluator composes the reference's own ``reference_apply``
calls, so the reference interpreter, passes and tests see ordinary
operators, and ``library_eval`` (library_eval.py) executes them on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

from .errors import ShapeError, UnsupportedOp

REQUIRED = object()  # frontend.py:65


@dataclass
class OpSpec:
    name: str
    attr_schema: dict
    min_inputs: int
    max_inputs: int
    min_outputs: int = 1
    max_outputs: int = 1
    replaces: str = ""          # the reference operator chain this op executes
    infer: Optional[Callable] = None  # concrete shapes -> [(shape, dtype-like index)]
    notes: str = ""
    extra: dict = field(default_factory=dict)


_REGISTRY: dict[str, OpSpec] = {}


class DuplicateOp(Exception):
    """frontend.DuplicateOp (frontend.py:57-58)."""


def register_op(spec: OpSpec) -> None:
    if spec.name in _REGISTRY:
        raise DuplicateOp(f"operator {spec.name!r} is already registered")
    _REGISTRY[spec.name] = spec


def get_op(name: str) -> OpSpec:
    spec = _REGISTRY.get(name)
    if spec is None:
        raise UnsupportedOp(name)
    return spec


def registered_ops() -> list:
    return sorted(_REGISTRY)


def normalize_attrs(op, attrs) -> dict:
    """Same contract as frontend.normalize_attrs (frontend.py:112-129)."""
    spec = get_op(op) if isinstance(op, str) else op
    given = dict(attrs or {})
    given.pop("implementation", None)  # per-node lowering selector (lowering.py:1045-1075)
    out = {}
    for key, default in spec.attr_schema.items():
        if key in given:
            out[key] = given.pop(key)
        elif default is REQUIRED:
            raise ShapeError(f"{spec.name}: missing required attribute {key!r}")
        else:
            out[key] = default
    if given:
        raise ShapeError(f"{spec.name}: unknown attribute(s) {sorted(given)}; known: {sorted(spec.attr_schema)}")
    return out


# -- reference operators executed on the B200 path (schemas = the reference's)
HOT_OPS = [
    OpSpec("LayerNormalization", {"axis": -1, "epsilon": 1e-5}, 2, 3, replaces="frontend.py:504-541"),
    OpSpec("Softmax", {"axis": -1}, 1, 1, replaces="frontend.py:488-501"),
    OpSpec("Gemm", {"alpha": 1.0, "beta": 1.0, "transA": 0, "transB": 0}, 2, 3, replaces="frontend.py:369-405"),
    OpSpec("MatMul", {}, 2, 2, replaces="frontend.py:335-366"),
    OpSpec("Einsum", {"equation": REQUIRED}, 2, 2, replaces="frontend.py:408-481 (two operands)"),
    OpSpec("BatchNormalization", {"epsilon": 1e-5, "momentum": 0.9}, 5, 5, 1, 3,
           replaces="frontend.py:544-591 (training mode)"),
    OpSpec("Conv", {"strides": None, "pads": None, "group": 1, "kernel_shape": None}, 2, 2,
           replaces="frontend.py:598-678 (depthwise 3x3, group = C)"),
    OpSpec("ReduceSum", {"axes": None, "keepdims": 1}, 1, 1, replaces="frontend.py:302-328 (Gemm bias VJP)"),
    OpSpec("ReduceMean", {"axes": None, "keepdims": 1}, 1, 1, replaces="frontend.py:302-328"),
    OpSpec("Reshape", {"shape": None}, 1, 1, replaces="frontend.py:713-829 (metadata only)"),
    OpSpec("Flatten", {"axis": 1}, 1, 1, replaces="frontend.py:713-829 (metadata only)"),
]

# -- fused operators (the subgraphs the reference's fusion recipe collapses,
#    SURVEY.md §3D; masks are the reference's float keep/(1-p) tensors)
FUSED_OPS = [
    OpSpec("BiasDropoutResidualLayerNorm", {"epsilon": 1e-5}, 6, 6, 1, 2,
           replaces="s = Add(Mul(Add(h, bias), mask), residual); y = LayerNormalization(s, gamma, beta)",
           notes="inputs (h, bias, mask, residual, gamma, beta) -> (y, s)"),
    OpSpec("BiasDropoutResidualLayerNormGrad", {"epsilon": 1e-5}, 4, 4, 5, 5,
           replaces="LayerNormalization VJP (autodiff.py:1490-1545) + Mul/Add VJPs",
           notes="inputs (dy, s, gamma, mask) -> (ds, dh, dbias, dgamma, dbeta)"),
    OpSpec("ScaledMaskedSoftmax", {"divisor": 1.0}, 3, 3, 1, 2,
           replaces="p = Softmax(Add(Div(scores, divisor), add_mask)); pd = Mul(p, drop_mask)",
           notes="inputs (scores [B,NH,Q,K], add_mask [B,1,1,K], drop_mask) -> (pd, p)"),
    OpSpec("ScaledMaskedSoftmaxGrad", {"divisor": 1.0}, 3, 3, 1, 1,
           replaces="Mul VJP + Softmax VJP (autodiff.py:1465-1484) + Div VJP",
           notes="inputs (dpd, p, drop_mask) -> dscores"),
    OpSpec("BiasGelu", {}, 2, 2, 1, 2,
           replaces="x = Add(f, bias); tanh-GELU chain of Pow/Mul/Add/Tanh (frontend.py:223-295)",
           notes="inputs (f, bias) -> (y, pre)"),
    OpSpec("BiasGeluGrad", {}, 2, 2, 1, 2,
           replaces="symexpr derivative of the GELU chain (symexpr.py:672-738) + Add VJP",
           notes="inputs (dy, pre) -> (dpre, dbias)"),
    OpSpec("MBConvBlock", {"strides": None, "pads": None, "epsilon": 1e-5, "momentum": 0.9}, 10, 10, 1, 3,
           replaces="Conv(group=C) -> BatchNormalization -> Mul(u, Sigmoid(u)) -> GlobalAveragePool -> "
                    "Gemm -> swish -> Gemm -> Sigmoid -> Mul (SURVEY.md:512-514)",
           notes="inputs (x NCHW, w_dw, gamma, beta, run_mean, run_var, w_r, b_r, w_e, b_e) -> "
                 "(y, new_run_mean, new_run_var)"),
    OpSpec("MBConvBlockGrad", {"strides": None, "pads": None, "epsilon": 1e-5, "momentum": 0.9}, 11, 11, 8, 8,
           replaces="VJPs of the MBConvBlock chain (autodiff.py:1551-1629 + tasklet VJPs)",
           notes="inputs (dy, x, w_dw, gamma, beta, run_mean, run_var, w_r, b_r, w_e, b_e) -> "
                 "(dx, dw_dw, dgamma, dbeta, dw_r, db_r, dw_e, db_e)"),
    OpSpec("LayerNormAct", {"epsilon": 1e-5, "activation": "swish"}, 3, 3, 1, 1,
           replaces="act(LayerNormalization(x, gamma, beta, axis=-1))"),
    OpSpec("LayerNormActGrad", {"epsilon": 1e-5, "activation": "swish"}, 4, 4, 3, 3,
           replaces="act VJP + LayerNormalization VJP (autodiff.py:1490-1545)",
           notes="inputs (dy, x, gamma, beta) -> (dx, dgamma, dbeta)"),
    OpSpec("BatchNormAct", {"epsilon": 1e-5, "momentum": 0.9, "activation": "swish"}, 5, 5, 1, 3,
           replaces="act(BatchNormalization(x, gamma, beta, run_mean, run_var)) (training)"),
    OpSpec("BatchNormActGrad", {"epsilon": 1e-5, "activation": "swish"}, 4, 4, 3, 3,
           replaces="act VJP + BatchNormalization VJP (autodiff.py:1551-1617), batch statistics recomputed",
           notes="inputs (dy, x, gamma, beta) -> (dx, dgamma, dbeta)"),
]

for _s in HOT_OPS + FUSED_OPS:
    register_op(_s)


# ---------------------------------------------------------------------------
# installation into a live dfir registry


def register_with_dfir(frontend=None) -> list:
    """Install the fused operators (spec + reference + lowering + manual VJP)
    and the ``fuse_to_b200`` transformation into the importable ``dfir``
    (dfir_plugin.install).  Returns the operator names newly registered."""
    from .dfir_plugin import install

    return install()["ops"]
