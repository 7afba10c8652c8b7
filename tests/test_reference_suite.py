"""The reference package's own unit tests, run against this package.

tests/reference_suite.py binds the module name ``nncp`` to paper_1909_01149_b200
and runs the reference's test files (copied by build() into the git-ignored
baseline/_ref/tests; skipped where they are absent).  test_grid.py needs no GPU
(Grid.run / Worker / DistMap); every other file calls the device kernels.

Deselected reference tests, each a documented, deliberate deviation:
DESELECT below (DESIGN.md §6 "Known deviations")."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "tests")

# reference test id -> why it cannot hold for the device mirror
DESELECT = {
    "test_acceptance.py::test_c04c_mu_converges_on_exact_data":
        "known red in the reference itself (pkg/README.md:33-37): plain MU needs ~2x the iteration budget; "
        "the device run reaches the reference's own 9.27e-02",
    "test_driver.py::TestSequentialDriver::test_nnls_failure_carries_context":
        "monkeypatches driver.bpp_update, a Python call the fused device sweep does not make per mode; the "
        "error wrapping itself is covered by tests/test_gpu_spmd.py failure tests",
    "test_driver.py::TestParallelDriver::test_stateful_updaters_communicate_extra":
        "asserts HALS issues more All-Reduces than BPP: the reference's per-column HALS hook All-Reduce returns "
        "a value nobody reads (updaters.py:117) and the device path elides it (DESIGN.md §6)",
    "test_io_cli.py::TestCli::test_category_columns_cover_iteration_wall_time":
        "category seconds are device time from CUDA events, not host wall-clock sections: on a 48^3 tensor the "
        "~0.1 ms device iteration is below the host's per-iteration overhead, which the CSV reports as 'other'",
}


def _run(files, timeout=1500):
    if not os.path.isdir(SUITE):
        pytest.skip("reference tests not installed (baseline/_ref/tests; build() copies them)")
    args = [sys.executable, os.path.join(ROOT, "tests", "reference_suite.py")] + list(files)
    skip = [tid.split("::")[-1] for tid in DESELECT if tid.split("::")[0] in files]
    if skip:
        args += ["-k=" + " and ".join(f"not {name}" for name in skip)]
    res = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
    print(res.stdout[-6000:], res.stderr[-3000:])
    return res


def test_reference_grid_tests_pass_against_mirror():
    res = _run(["test_grid.py"])
    assert res.returncode == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_tensor_ops.py", "test_dimtree.py", "test_updaters.py", "test_driver.py",
                                  "test_io_cli.py", "test_acceptance.py"])
def test_reference_tests_pass_against_mirror(name):
    res = _run([name])
    assert res.returncode == 0
