"""NNCP file format (tensor_io.py) -- host-side parts run on CPU; device streaming on the GPU."""

import struct

import numpy as np
import pytest

from paper_1909_01149_b200.tensor_io import (MAGIC, BadMagicError, PayloadMismatchError, TensorFileError,
                                             TruncatedFileError, read_matrix, read_tensor, write_matrix,
                                             write_tensor)
from paper_1909_01149_b200.tensor_ops import DenseTensor


def test_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    for k, dims in enumerate([(3, 4, 5), (2, 2), (1, 5, 1, 2)]):
        x = DenseTensor(dims, rng.standard_normal(int(np.prod(dims))))
        path = tmp_path / f"x{k}.bin"
        write_tensor(path, x)
        back = read_tensor(path)
        assert back.dims == x.dims
        assert back.data.tobytes() == x.data.tobytes()


def test_matrix_round_trip(tmp_path):
    h = np.random.default_rng(1).standard_normal((7, 3))
    write_matrix(tmp_path / "h.bin", h)
    assert np.array_equal(read_matrix(tmp_path / "h.bin"), h)


def test_malformed_files(tmp_path):
    path = tmp_path / "good.bin"
    write_tensor(path, DenseTensor((2, 2), np.arange(4.0)))
    raw = path.read_bytes()
    (tmp_path / "magic.bin").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(BadMagicError):
        read_tensor(tmp_path / "magic.bin")
    (tmp_path / "trunc.bin").write_bytes(raw[:-3])
    with pytest.raises(TruncatedFileError):
        read_tensor(tmp_path / "trunc.bin")
    (tmp_path / "head.bin").write_bytes(MAGIC + b"\x01")
    with pytest.raises(TruncatedFileError):
        read_tensor(tmp_path / "head.bin")
    header = struct.pack("<4sHH", MAGIC, 1, 2) + struct.pack("<2Q", 2, 2)
    (tmp_path / "mismatch.bin").write_bytes(header + struct.pack("<3d", 1.0, 2.0, 3.0))
    with pytest.raises(PayloadMismatchError):
        read_tensor(tmp_path / "mismatch.bin")
    header = struct.pack("<4sHH", MAGIC, 9, 2) + struct.pack("<2Q", 1, 1)
    (tmp_path / "v9.bin").write_bytes(header + struct.pack("<1d", 1.0))
    with pytest.raises(TensorFileError):
        read_tensor(tmp_path / "v9.bin")
    assert not issubclass(BadMagicError, TruncatedFileError)
    assert issubclass(BadMagicError, TensorFileError)


@pytest.mark.gpu
def test_device_streaming_read_write(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200.tensor_io as tio

    rng = np.random.default_rng(3)
    x = DenseTensor((40, 30, 20), rng.random(24000))
    path = tmp_path / "x.bin"
    write_tensor(path, x)
    old = tio._CHUNK
    tio._CHUNK = 1000  # force several staged transfers
    try:
        d = read_tensor(path, device=True)
        assert d.on_device and np.array_equal(d.data.cpu().numpy(), x.data)
        write_tensor(tmp_path / "y.bin", d)
    finally:
        tio._CHUNK = old
    assert (tmp_path / "y.bin").read_bytes() == path.read_bytes()


@pytest.mark.gpu
def test_generate_synthetic_truth_matches_reference(golden):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1909_01149_b200.tensor_io import SyntheticSpec, generate_synthetic

    g = golden("synthetic.npz")
    dims = tuple(int(d) for d in g["dims"])
    x, truth = generate_synthetic(SyntheticSpec(dims, int(g["rank"]), int(g["seed"])))
    for n in range(len(dims)):
        assert np.array_equal(truth.factors[n], g[f"h{n}"])     # bit-identical truth draws
    got = np.asarray(x.data)
    assert np.linalg.norm(got - g["x"]) <= 1e-14 * np.linalg.norm(g["x"])
    with pytest.raises(ValueError):
        generate_synthetic(SyntheticSpec((1024, 1024, 256), 2))
