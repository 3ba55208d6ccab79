"""DTNS tensor container I/O, with a direct path into device memory.

The reference's on-disk / on-wire tensor encoding (``dfir/dtns.py``, §8f row 3)
so inputs, weights and golden vectors move byte-exactly between the reference
tools and this GPU path.  The container (all integers little-endian)::

    0   4          magic b"DTNS"
    4   1          version (1)
    5   1          dtype code
    6   1          rank
    7   1          reserved (0)
    8   8 * rank   dims, u64
    ..  payload    row-major, little-endian

Codes 0-3 are the reference's (f32, f64, i64, bool — dtns.py:30-44) and are
written bit-identically to it.  Codes 4 (bf16) and 5 (u8) are this package's
extension, matching the C ABI dtype codes (include/dfx.h); the reference
rejects them on read, so ``encode`` only emits them when ``extended=True``.

``to_device`` decodes straight into a CUDA tensor: the payload is staged once
through pinned memory and copied asynchronously on the current stream, with an
optional dtype cast done on the GPU (e.g. the reference's f64 golden tensors ->
bf16 operands).

Error behaviour mirrors the reference: malformed bytes raise
``TensorFormatError`` (a ``ValueError``) naming the broken field.
"""

from __future__ import annotations

import struct
from typing import BinaryIO, Union

import numpy as np

MAGIC = b"DTNS"
VERSION = 1
_HDR = struct.Struct("<4sBBBB")

# code -> (little-endian numpy payload dtype, name); bf16 travels as raw u16
_CODES = {
    0: (np.dtype("<f4"), "f32"),
    1: (np.dtype("<f8"), "f64"),
    2: (np.dtype("<i8"), "i64"),
    3: (np.dtype("|b1"), "bool"),
    4: (np.dtype("<u2"), "bf16"),  # raw bit patterns
    5: (np.dtype("|u1"), "u8"),
}
_REFERENCE_CODES = (0, 1, 2, 3)
NAME_TO_CODE = {name: code for code, (_, name) in _CODES.items()}
CODE_TO_NAME = {code: name for name, code in NAME_TO_CODE.items()}


class TensorFormatError(ValueError):
    """Bytes that do not decode as a valid tensor container."""


def _code_of(arr: np.ndarray, extended: bool) -> int:
    dt = arr.dtype.newbyteorder("=")
    table = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int64): 2, np.dtype(np.bool_): 3}
    if extended:
        table[np.dtype(np.uint8)] = 5
    code = table.get(dt)
    if code is None:
        supported = "f32, f64, i64, bool" + (", u8 (bf16 via torch tensors)" if extended else "")
        raise TensorFormatError(f"unsupported dtype {arr.dtype!r}; supported: {supported}")
    return code


def _header(code: int, shape) -> bytes:
    if len(shape) > 255:
        raise TensorFormatError(f"rank {len(shape)} exceeds the format maximum of 255")
    return _HDR.pack(MAGIC, VERSION, code, len(shape), 0) + struct.pack(f"<{len(shape)}Q", *shape)


def encode(array, extended: bool = False) -> bytes:
    """Container bytes of a numpy array or torch tensor (CPU or CUDA).

    bf16 torch tensors need ``extended=True`` (code 4); every other accepted
    dtype round-trips bit for bit and, for codes 0-3, byte-identically to the
    reference encoder."""
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is a hard dependency of the package
        torch = None
    if torch is not None and isinstance(array, torch.Tensor):
        t = array.detach()
        if t.dtype == torch.bfloat16:
            if not extended:
                raise TensorFormatError("unsupported dtype bfloat16; supported: f32, f64, i64, bool "
                                        "(pass extended=True for the bf16 extension code)")
            raw = t.contiguous().cpu().view(torch.int16).numpy().view("<u2")
            return _header(4, raw.shape) + raw.tobytes()
        array = t.cpu().numpy()
    arr = np.asarray(array)
    code = _code_of(arr, extended)
    return _header(code, arr.shape) + np.ascontiguousarray(arr, dtype=_CODES[code][0]).tobytes()


def _parse(data) -> tuple[int, tuple, int]:
    """(code, shape, payload offset) of container bytes, validating sizes."""
    n = len(data)
    if n < 8:
        raise TensorFormatError(f"truncated header: {n} bytes, need at least 8")
    magic, version, code, rank, reserved = _HDR.unpack_from(data, 0)
    if magic != MAGIC:
        raise TensorFormatError(f"bad magic {bytes(magic)!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise TensorFormatError(f"unsupported version {version}, expected {VERSION}")
    if code not in _CODES:
        raise TensorFormatError(f"unknown dtype code {code}")
    if reserved != 0:
        raise TensorFormatError(f"reserved byte must be 0, got {reserved}")
    off = 8 + 8 * rank
    if n < off:
        raise TensorFormatError(f"truncated dims: {n} bytes, header promises {rank} dims")
    shape = struct.unpack_from(f"<{rank}Q", data, 8) if rank else ()
    count = 1
    for d in shape:
        count *= d
    need = off + count * _CODES[code][0].itemsize
    if n != need:
        raise TensorFormatError(f"payload size mismatch: file has {n} bytes, shape {tuple(shape)} with dtype "
                                f"{CODE_TO_NAME[code]} needs {need}")
    return code, tuple(shape), off


def decode(data, allow_extended: bool = True) -> np.ndarray:
    """numpy array (native byte order) of container bytes.  bf16 payloads
    come back as their raw uint16 bit patterns (numpy has no bf16)."""
    code, shape, off = _parse(data)
    if not allow_extended and code not in _REFERENCE_CODES:
        raise TensorFormatError(f"unknown dtype code {code}")
    dt = _CODES[code][0]
    count = int(np.prod(shape, dtype=np.int64)) if shape else 1
    arr = np.frombuffer(data, dtype=dt, count=count, offset=off)
    return arr.reshape(shape).astype(dt.newbyteorder("="), copy=True)


def _read_bytes(source) -> bytes:
    if isinstance(source, str):
        with open(source, "rb") as fh:
            return fh.read()
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    return source.read()


def write_tensor(target: Union[str, BinaryIO], array, extended: bool = False) -> None:
    blob = encode(array, extended)
    if isinstance(target, str):
        with open(target, "wb") as fh:
            fh.write(blob)
    else:
        target.write(blob)


def read_tensor(source: Union[str, bytes, BinaryIO]) -> np.ndarray:
    return decode(_read_bytes(source))


def to_device(source, device="cuda", dtype=None):
    """Decode a container (path, bytes or file object) into a torch tensor on
    ``device``.  The payload is staged once into pinned host memory and copied
    with ``non_blocking=True`` on the current stream (torch's pinned-memory
    allocator keeps the staging block alive until the copy completes); a
    ``dtype`` cast (e.g. f64 golden values -> torch.bfloat16) runs on the GPU
    after the copy."""
    import torch

    data = bytearray(_read_bytes(source))
    code, shape, off = _parse(data)
    count = int(np.prod(shape, dtype=np.int64)) if shape else 1
    dt = np.dtype("<i2") if code == 4 else _CODES[code][0]
    view = np.frombuffer(data, dtype=dt, count=count, offset=off).reshape(shape)
    if not view.dtype.isnative:
        view = view.astype(view.dtype.newbyteorder("="))
    host = torch.from_numpy(view)
    if code == 4:
        host = host.view(torch.bfloat16)
    if str(device).startswith("cuda"):
        host = host.pin_memory()
    out = host.to(device, non_blocking=True)
    if dtype is not None and out.dtype != dtype:
        out = out.to(dtype)
    return out
