"""The reference's whole unit-test suite (tests/CMakeLists.txt: test_geometry,
test_lsh, test_nystrom, test_sparse, test_sinkhorn, test_metrics, test_runner;
compiled
from /root/reference where they lie, unmodified) linked against the drop-in
shim (integration/lcn_shim.cpp): their build_sparse / build_correction /
select_landmarks / build_factors / lsh_neighbor_pairs / sinkhorn calls run on
the B200 through the C-ABI, their assertions are the reference's. Built by
integration/Makefile in the build container (it needs the reference sources);
the binary travels to the GPU box with the tree."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "ref_tests_gpu")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="integration/_build/ref_tests_gpu not built (needs /root/reference)")
def test_reference_unit_tests_through_the_shim():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200)
    summary = [ln for ln in r.stdout.splitlines() if ln.startswith("[doctest]")]
    print(r.stdout[-4000:])
    print(r.stderr[-8000:])
    assert r.returncode == 0, "\n".join(summary) + "\n" + r.stderr[-4000:]
    assert summary and "| 0 failed" in summary[0]
    assert "lcn shim: B200 context" in r.stderr  # the shimmed stages ran on the GPU
