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


@pytest.mark.gpu
def test_parallel_from_file_path_and_device_tensor(tmp_path, golden):
    """nncp_parallel takes a tensor-file path (each rank reads only its block) or a
    device-resident DenseTensor (blocks sliced in HBM): same run as from host memory."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import warnings

    import paper_1909_01149_b200 as P
    from paper_1909_01149_b200.tensor_io import write_tensor

    g = golden("runs.npz")
    dims = tuple(int(d) for d in g["hals_odd_dims"])
    r, iters, iseed = (int(v) for v in g["hals_odd_meta"])
    x = P.DenseTensor(dims, g["hals_odd_x"])
    path = str(tmp_path / "x.nncp")
    write_tensor(path, x)
    cfg = dict(rank=r, algorithm="hals", max_iters=iters, tol=0.0, seed=iseed, grid=(2, 2, 1))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        host = P.nncp_parallel(x, P.RunConfig(**cfg))
        from_file = P.nncp_parallel(path, P.RunConfig(**cfg))
        from_dev = P.nncp_parallel(x.to_device(), P.RunConfig(**cfg))
    assert host.errors == from_file.errors == from_dev.errors
    for a, b, c in zip(host.model.factors, from_file.model.factors, from_dev.model.factors):
        assert np.array_equal(a, b) and np.array_equal(a, c)
    assert np.max(np.abs(np.array(host.errors) - g["grid_hals_odd_2x2x1_errors"])) <= 1e-9
