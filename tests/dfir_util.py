"""Locate the reference ``dfir`` package for integration tests: the
pip-installed copy under baseline/_ref (travels to the GPU box) or, in the
build container only, /root/reference/pkg/src.  Returns None if absent."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def import_dfir():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "dfir")):
            if path not in sys.path:
                sys.path.insert(0, path)
            from dfir import autodiff, frontend, interp  # noqa: F401

            return frontend, interp
    return None
