"""DTNS container I/O (paper_2110_10802_b200/dtns.py) against containers the
reference encoder wrote (tests/golden/dtns, oracle/make_dtns_golden.py), the
reference's error cases (its tests/test_dtns.py), and — on the GPU — operands
loaded straight into device memory feeding the BDRLN kernel."""

import io
import os
import struct

import numpy as np
import pytest
import torch

from paper_2110_10802_b200 import dtns

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "dtns")
VALUES = np.load(os.path.join(GOLD, "values.npz"))
NAMES = sorted(VALUES.files)


def blob(name):
    with open(os.path.join(GOLD, name + ".dtns"), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name", NAMES)
def test_decode_reference_containers(name):
    got = dtns.read_tensor(os.path.join(GOLD, name + ".dtns"))
    want = VALUES[name]
    assert got.dtype == want.dtype and got.shape == want.shape
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("name", NAMES)
def test_encode_byte_identical_to_reference(name):
    assert dtns.encode(VALUES[name]) == blob(name)


def test_torch_and_extended_codes_round_trip():
    t = torch.randn(3, 5).bfloat16()
    with pytest.raises(dtns.TensorFormatError, match="unsupported dtype"):
        dtns.encode(t)
    b = dtns.encode(t, extended=True)
    assert b[5] == dtns.NAME_TO_CODE["bf16"]
    assert torch.equal(dtns.to_device(b, device="cpu"), t)
    u = np.arange(12, dtype=np.uint8).reshape(3, 4)
    with pytest.raises(dtns.TensorFormatError, match="unsupported dtype"):
        dtns.encode(u)
    assert np.array_equal(dtns.decode(dtns.encode(u, extended=True)), u)
    with pytest.raises(dtns.TensorFormatError, match="dtype code"):
        dtns.decode(dtns.encode(u, extended=True), allow_extended=False)
    # a torch f32 tensor encodes exactly like the numpy array
    x = VALUES["f32_4x5"]
    assert dtns.encode(torch.from_numpy(x)) == blob("f32_4x5")


def test_file_objects_and_paths(tmp_path):
    x = VALUES["f64_3x2x2"]
    path = str(tmp_path / "t.dtns")
    dtns.write_tensor(path, x)
    assert dtns.read_tensor(path).tobytes() == x.tobytes()
    buf = io.BytesIO()
    dtns.write_tensor(buf, x)
    buf.seek(0)
    assert dtns.read_tensor(buf).tobytes() == x.tobytes()


def test_header_errors():
    good = bytearray(blob("f32_4x5"))
    bad = bytearray(good)
    bad[0:4] = b"XXXX"
    with pytest.raises(dtns.TensorFormatError, match="magic"):
        dtns.decode(bytes(bad))
    bad = bytearray(good)
    bad[4] = 2
    with pytest.raises(dtns.TensorFormatError, match="version"):
        dtns.decode(bytes(bad))
    bad = bytearray(good)
    bad[5] = 9
    with pytest.raises(dtns.TensorFormatError, match="dtype code"):
        dtns.decode(bytes(bad))
    bad = bytearray(good)
    bad[7] = 1
    with pytest.raises(dtns.TensorFormatError, match="reserved"):
        dtns.decode(bytes(bad))


def test_truncation_and_size_mismatch():
    b = blob("f64_3x2x2")
    with pytest.raises(dtns.TensorFormatError, match="truncated header"):
        dtns.decode(b[:6])
    with pytest.raises(dtns.TensorFormatError, match="truncated dims"):
        dtns.decode(b[:12])
    with pytest.raises(dtns.TensorFormatError, match="size mismatch"):
        dtns.decode(b[:-1])
    with pytest.raises(dtns.TensorFormatError, match="size mismatch"):
        dtns.decode(b + b"\x00")


def test_big_endian_input_normalized():
    arr = np.arange(6, dtype=">f8").reshape(2, 3)
    back = dtns.decode(dtns.encode(arr))
    assert back.dtype == np.dtype("<f8").newbyteorder("=")
    np.testing.assert_array_equal(back, arr.astype("<f8"))
    hdr = dtns.encode(arr)[:8 + 16]
    assert struct.unpack("<4sBBBB2Q", hdr) == (b"DTNS", 1, 1, 2, 0, 2, 3)


@pytest.mark.gpu
def test_to_device_feeds_the_bdrln_kernel():
    """Reference-encoded operands decode straight into device memory (pinned
    staging, async copy, GPU-side cast) and run through the fused BDRLN path
    with the keep mask bit-packed on the device."""
    from oracle import oracle as O  # checker only
    from paper_2110_10802_b200 import kernels as K

    path = lambda n: os.path.join(GOLD, n + ".dtns")  # noqa: E731
    x = dtns.to_device(path("bert_x_8x768_f32"))
    keep_bool = dtns.to_device(path("bert_keep_8x768_bool"))
    assert x.is_cuda and x.dtype == torch.float32 and keep_bool.dtype == torch.bool
    assert torch.equal(x.cpu(), torch.from_numpy(VALUES["bert_x_8x768_f32"]))
    xb = dtns.to_device(path("bert_x_8x768_f32"), dtype=torch.bfloat16)
    assert torch.equal(xb.cpu(), torch.from_numpy(VALUES["bert_x_8x768_f32"]).bfloat16())
    H = x.shape[1]
    g = torch.ones(H, device="cuda")
    b = torch.zeros(H, device="cuda")
    kb = K.pack_keep_bits(keep_bool.to(torch.uint8))
    y = K.bdrln_fwd(x, None, kb, 1 / 0.9, None, g, b, 1e-12)
    torch.cuda.synchronize()
    keep = VALUES["bert_keep_8x768_bool"]
    want = O.bdrln_fwd(VALUES["bert_x_8x768_f32"].astype(np.float64), np.zeros(H),
                       O.mask_values(keep, 0.1, np.float64), np.zeros_like(keep, dtype=np.float64), np.ones(H),
                       np.zeros(H), 1e-12)["y"]
    err = np.abs(y.cpu().numpy() - want).max() / max(np.abs(want).max(), 1.0)
    assert err < 1e-4, err
