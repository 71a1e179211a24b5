"""Run the reference's own unit tests (tests/test_{geometry,octree,features}.cpp,
30 cases) compiled unmodified against the reference library with the
doctest shim (oracle/ref/doctest.h). These pin the checker itself: the
reference build used as the oracle passes its own KATs. Skipped where
oracle/_ref was not built."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("name", ["test_geometry_ref", "test_octree_ref", "test_features_ref"])
def test_reference_unit_tests(name):
    exe = os.path.join(REF, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
