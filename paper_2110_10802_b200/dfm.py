"""``dfm-0.1`` model documents on the B200 path (§8f row 3).

The reference's native model format (``frontend.parse_model_json``,
frontend.py:886-964): ``{"version": "dfm-0.1", "inputs": [{name, shape,
dtype}], "outputs": [...], "initializers": [...], "nodes": [{op, inputs,
outputs, attrs}]}``, initializers given inline (dtype/dims/data), as base64
DTNS bytes, or as a DTNS file.  ``parse_model`` restates its validation with
the same ``ModelError`` messages; ``DeviceGraph`` executes such a model with
every tensor resident in HBM: node by node through ``device_ops`` (the same
operator implementations ``library_eval`` uses), on the current stream, with
no host round trip between operators.  Graphs made of the fused operators
(e.g. the ``model_fused.json`` fixtures, or what ``dfir_plugin.fuse_to_b200``
makes of the reference's graphs) run end to end; any operator outside the hot
path raises ``UnsupportedOp`` when the graph is built (no CPU fallback).
"""

from __future__ import annotations

import base64
import json
import os
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np
import torch

from . import dtns
from .device_ops import DEVICE_OPS, run_op
from .errors import ModelError, ShapeError, UnsupportedOp
from .registry import get_op, normalize_attrs

__all__ = ["ModelNode", "ModelDoc", "parse_model", "DeviceGraph"]

_DTYPES = {"f32": np.float32, "f64": np.float64, "i64": np.int64, "bool": np.bool_}


@dataclass
class ModelNode:
    op: str
    name: str
    attrs: dict
    inputs: list
    outputs: list


@dataclass
class ModelDoc:
    name: str
    inputs: list  # (name, shape, dtype)
    outputs: list
    initializers: dict = field(default_factory=dict)
    nodes: list = field(default_factory=list)


def _require_keys(entry, keys, where):
    if not isinstance(entry, dict) or not keys <= set(entry):
        raise ModelError(f"{where}: missing required keys {sorted(keys)}")


def parse_model(source: Union[str, dict], base_dir: Optional[str] = None) -> ModelDoc:
    """Parse a ``dfm-0.1`` document (path or dict), frontend.py:886-964."""
    if isinstance(source, str):
        base_dir = base_dir or os.path.dirname(os.path.abspath(source))
        try:
            with open(source) as fh:
                doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise ModelError(f"malformed model JSON: {exc}") from exc
    else:
        doc = source
    if not isinstance(doc, dict) or doc.get("version") != "dfm-0.1":
        got = doc.get("version") if isinstance(doc, dict) else None
        raise ModelError(f"unsupported model version {got!r}; expected 'dfm-0.1'")
    inputs = []
    for entry in doc.get("inputs", []):
        _require_keys(entry, {"name", "shape", "dtype"}, "inputs[]")
        if entry["dtype"] not in _DTYPES:
            raise ModelError(f"input {entry['name']}: unknown dtype {entry['dtype']!r}")
        for d in entry["shape"]:
            if not isinstance(d, (int, str)) or (isinstance(d, int) and d < 0):
                raise ModelError(f"input {entry['name']}: dims must be non-negative ints or symbol names, got {d!r}")
        inputs.append((entry["name"], list(entry["shape"]), entry["dtype"]))
    outputs = []
    for entry in doc.get("outputs", []):
        outputs.append(entry["name"] if isinstance(entry, dict) else entry)
        if not isinstance(outputs[-1], str):
            raise ModelError(f"outputs[] entries must be names, got {entry!r}")
    inits = {}
    for entry in doc.get("initializers", []):
        if "name" not in entry:
            raise ModelError("initializers[] entry missing 'name'")
        name = entry["name"]
        if "file" in entry:
            path = entry["file"] if os.path.isabs(entry["file"]) else os.path.join(base_dir or ".", entry["file"])
            try:
                arr = dtns.read_tensor(path)
            except (OSError, dtns.TensorFormatError) as exc:
                raise ModelError(f"initializer {name}: {exc}") from exc
        elif "base64" in entry:
            try:
                arr = dtns.decode(base64.b64decode(entry["base64"]))
            except (ValueError, dtns.TensorFormatError) as exc:
                raise ModelError(f"initializer {name}: {exc}") from exc
        elif {"dtype", "dims", "data"} <= set(entry):
            if entry["dtype"] not in _DTYPES:
                raise ModelError(f"initializer {name}: unknown dtype {entry['dtype']!r}")
            arr = np.asarray(entry["data"], dtype=_DTYPES[entry["dtype"]]).reshape([int(d) for d in entry["dims"]])
        else:
            raise ModelError(f"initializer {name}: needs 'file', 'base64', or dtype/dims/data")
        inits[name] = arr
    nodes = []
    for i, entry in enumerate(doc.get("nodes", [])):
        _require_keys(entry, {"op", "inputs", "outputs"}, f"nodes[{i}]")
        nodes.append(ModelNode(entry["op"], entry.get("name") or f"{entry['op']}_{i}", dict(entry.get("attrs", {})),
                               list(entry["inputs"]), list(entry["outputs"])))
    return ModelDoc(doc.get("name", "model"), inputs, outputs, inits, nodes)


class DeviceGraph:
    """A parsed ``dfm-0.1`` model bound to one device: initializers uploaded
    once, attributes normalised by the registry (frontend.py:112-129), rank-0
    Pow/Div constants and Reshape shape operands folded into attributes as
    ``build_graph`` does (frontend.py:1034-1053).  ``run(inputs)`` executes the
    nodes in document order (every input is a graph input, initializer or an
    earlier output — the reference's own construction rule, frontend.py:1055-1061)."""

    def __init__(self, source: Union[str, dict, ModelDoc], device="cuda", f64: str = "reject"):
        self.doc = source if isinstance(source, ModelDoc) else parse_model(source)
        self.device = torch.device(device)
        if f64 not in ("reject", "as_f32"):
            raise ValueError("f64 policy must be 'reject' or 'as_f32'")
        self.f64 = f64
        defined = {n for n, _, _ in self.doc.inputs} | set(self.doc.initializers)
        self.plan = []
        for node in self.doc.nodes:
            if node.op not in DEVICE_OPS:
                raise UnsupportedOp(node.op)
            spec = get_op(node.op)
            attrs, ins = dict(node.attrs), list(node.inputs)
            if node.op == "Reshape" and len(ins) == 2:
                arr = self.doc.initializers.get(ins[1])
                if arr is None:
                    raise ModelError(f"node {node.name}: Reshape target shape must be a constant")
                attrs.setdefault("shape", [int(v) for v in arr.reshape(-1)])
                ins = ins[:1]
            for t in ins:
                if t not in defined:
                    raise ModelError(f"node {node.name}: input {t!r} is not a graph input, initializer, or earlier "
                                     "node output")
            if not (spec.min_outputs <= len(node.outputs) <= spec.max_outputs):
                raise ModelError(f"node {node.name}: {node.op} produces {spec.min_outputs}..{spec.max_outputs} "
                                 f"outputs, model lists {len(node.outputs)}")
            try:
                attrs = normalize_attrs(spec, attrs)
            except ShapeError as exc:
                raise ShapeError(f"node {node.name}: {exc}") from exc
            self.plan.append((node.op, attrs, ins, list(node.outputs)))
            defined.update(node.outputs)
        for o in self.doc.outputs:
            if o not in defined:
                raise ModelError(f"declared output {o!r} is never produced")
        self.constants = {k: self._upload(v) for k, v in self.doc.initializers.items()}

    def _upload(self, a):
        if isinstance(a, torch.Tensor):
            t = a.to(self.device, non_blocking=True)
        else:
            arr = np.asarray(a)
            if arr.dtype == np.float64 and self.f64 != "as_f32":
                raise ShapeError("DeviceGraph computes in fp32: f64 tensors are rejected (f64='as_f32' opts in)")
            t = torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().to(self.device, non_blocking=True)
        if t.dtype == torch.float64:
            if self.f64 != "as_f32":
                raise ShapeError("DeviceGraph computes in fp32: f64 tensors are rejected (f64='as_f32' opts in)")
            t = t.float()
        return t

    def run(self, inputs: dict, outputs=None) -> dict:
        """inputs: name -> host array or device tensor.  Returns device tensors
        of the requested (default: declared) outputs, produced on the current
        stream."""
        env = dict(self.constants)
        for name, _, _ in self.doc.inputs:
            if name not in inputs and name not in env:
                raise ModelError(f"missing input {name!r}")
        for name, val in inputs.items():
            env[name] = self._upload(val)
        for op, attrs, ins, outs in self.plan:
            res = run_op(op, attrs, [env[i] for i in ins])
            env.update(zip(outs, res))
        return {o: env[o] for o in (outputs or self.doc.outputs)}
