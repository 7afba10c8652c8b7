"""Run the reference package's OWN unit tests against this package (test infrastructure).

    python tests/reference_suite.py [pytest args...]

`build()` copies the reference's tests (`/root/reference/pkg/tests`) into the
git-ignored `baseline/_ref/tests` next to the reference install, so they travel to
the GPU box but never enter the repository.  Here the module name `nncp` (and its
submodules) is bound to `paper_1909_01149_b200` before pytest imports the test
files: every `from nncp import ...` in them resolves to the device-backed mirror,
and every numeric call in those tests runs through libnncp_b200.so.
"""

import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "tests")


def alias_reference_modules():
    sys.path.insert(0, ROOT)
    import paper_1909_01149_b200 as P
    from paper_1909_01149_b200 import cli, dimtree, driver, grid, tensor_io, tensor_ops, updaters

    sys.modules["nncp"] = P
    for name, mod in (("dimtree", dimtree), ("driver", driver), ("grid", grid), ("tensor_io", tensor_io),
                      ("tensor_ops", tensor_ops), ("updaters", updaters), ("cli", cli)):
        sys.modules[f"nncp.{name}"] = mod
        setattr(P, name, mod)
    return P


def main(argv):
    if not os.path.isdir(SUITE):
        print(f"reference tests not present at {SUITE} (build() copies them where /root/reference exists)")
        return 5
    alias_reference_modules()
    import pytest

    files = [a for a in argv if not a.startswith("-")]
    opts = [a for a in argv if a.startswith("-")]
    paths = [os.path.join(SUITE, f) for f in files] or [SUITE]
    with tempfile.TemporaryDirectory() as tmp:       # hypothesis writes its database to the cwd
        os.chdir(tmp)
        return pytest.main(["-p", "no:cacheprovider", "--rootdir", tmp, "--confcutdir", SUITE, "-q", "-rfE"]
                           + opts + paths)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
