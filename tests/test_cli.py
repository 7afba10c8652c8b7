"""CLI mirror (cli.py): usage errors on CPU; full runs on the GPU."""

import csv

import numpy as np
import pytest

from paper_1909_01149_b200.cli import CSV_FIELDS, run_cli


def _run(tmp_path, *args):
    prefix = tmp_path / "out"
    return run_cli(list(args) + ["--output-prefix", str(prefix)]), prefix


def _rows(prefix):
    with open(f"{prefix}_convergence.csv") as fh:
        return list(csv.DictReader(fh))


def test_usage_errors(tmp_path):
    with pytest.raises(SystemExit) as info:
        _run(tmp_path, "--input", "x.bin", "--dims", "4,4", "--rank", "2")
    assert info.value.code == 2
    with pytest.raises(SystemExit) as info:
        _run(tmp_path, "--dims", "4,4", "--rank", "2")
    assert info.value.code == 2


def test_missing_input_file_fails_cleanly(tmp_path):
    code, _ = _run(tmp_path, "--input", str(tmp_path / "nope.bin"), "--rank", "2")
    assert code == 1


@pytest.mark.gpu
def test_cli_runs(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1909_01149_b200 import (FactorSet, RunConfig, SyntheticSpec, generate_synthetic, nncp_sequential,
                                       read_matrix)
    from oracle import nncp_oracle as O

    code, prefix = _run(tmp_path, "--dims", "6,5,4", "--synthetic-rank", "2", "--rank", "2", "--algo", "hals",
                        "--iters", "8", "--seed", "2", "--tol", "0")
    assert code == 0
    rows = _rows(prefix)
    assert list(rows[0].keys()) == list(CSV_FIELDS) and len(rows) == 9
    factors = [read_matrix(f"{prefix}_factors_{n}.bin") for n in (1, 2, 3)]
    lam = np.atleast_1d(np.loadtxt(f"{prefix}_lambda.txt"))
    x, _ = generate_synthetic(SyntheticSpec((6, 5, 4), 2, seed=2))
    xd = np.asarray(x.data)
    direct = np.linalg.norm(xd - O.reconstruct(factors, lam)) / np.linalg.norm(xd)
    assert abs(direct - float(rows[-1]["relerr"])) <= 1e-10
    rep = nncp_sequential(x, RunConfig(rank=2, algorithm="hals", max_iters=8, tol=0.0, seed=2))
    assert [float(r["relerr"]) for r in rows] == rep.errors
    assert all(int(r["words_communicated"]) == 0 for r in rows)
    with pytest.raises(SystemExit) as info:
        _run(tmp_path, "--dims", "4,4,4", "--synthetic-rank", "2", "--rank", "2", "--grid", "2,2")
    assert info.value.code == 2
    (tmp_path / "s").mkdir()
    (tmp_path / "p").mkdir()
    args = ["--dims", "6,6,6", "--synthetic-rank", "2", "--rank", "2", "--algo", "mu", "--iters", "5", "--seed", "3",
            "--tol", "0"]
    code_s, ps = _run(tmp_path / "s", *args)
    code_p, pp = _run(tmp_path / "p", *args, "--grid", "2,2,1")
    assert code_s == 0 and code_p == 0
    for a, b in zip(_rows(ps), _rows(pp)):
        assert abs(float(a["relerr"]) - float(b["relerr"])) <= 1e-10
    assert all(int(r["words_communicated"]) > 0 for r in _rows(pp))
    code, prefix = _run(tmp_path, "--dims", "8,8,8", "--synthetic-rank", "2", "--rank", "2", "--algo", "bpp",
                        "--iters", "50", "--seed", "9")
    assert code == 0 and float(_rows(prefix)[-1]["relerr"]) <= 1e-4
    del FactorSet
