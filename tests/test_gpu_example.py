"""The plain-C example (examples/chase_example.c) solves the 1-2-1 matrix on the GPU through the
C ABI alone and matches the closed-form spectrum (Table 1) to 1e-10 ||H||."""
import subprocess

import pytest

from test_library_abi import _build_example

pytestmark = pytest.mark.gpu


def test_plain_c_example_runs(tmp_path):
    exe = _build_example(str(tmp_path / "chase_example"))
    r = subprocess.run([exe, "800"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max |lambda - exact|" in r.stdout
