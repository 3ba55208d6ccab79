"""Exception types mirroring the reference's error behaviour.

* ``ModelError`` / ``UnsupportedOp`` / ``ShapeError`` — frontend.py:45-62
* ``ExecError`` carrying state/node — interp.py:56-61
The C ABI returns status codes; ``_lib.check`` maps them onto these.
"""


class ModelError(Exception):
    """Malformed model or graph-construction failure (frontend.py:45-46)."""


class UnsupportedOp(ModelError):
    """Operator type the B200 path does not implement (frontend.py:49-54).

    Raised instead of falling back to the CPU: there is no CPU fallback."""

    def __init__(self, op: str):
        super().__init__(f"unsupported operator type {op!r}")
        self.op = op


class ShapeError(ModelError):
    """Shape/attribute/dtype rejected (frontend.py:61-62)."""


class ExecError(Exception):
    """Execution failure (interp.py:56-61)."""

    def __init__(self, message: str, state=None, node=None):
        where = f" [state {state}, node {node}]" if state is not None else ""
        super().__init__(message + where)
        self.state = state
        self.node = node
