"""The INTEGRATION.md sparsekit-side shim (integration/sparsekit_b200.hpp),
compiled against the reference headers by `make -C oracle shim` (the build
container) and run here: reference SparseTensor / Features / WeightTensor /
DataflowConfig objects through the C ABI, checked against the compiled
reference's conv_ref / conv_dgrad / conv_wgrad on the Fig. 2 golden instance
and the test_exec.cpp random instances (fp32 path, 1e-5), plus the
ValidationError mapping. Test infrastructure: the binary lives in oracle/_ref."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_check")


@pytest.mark.gpu
def test_sparsekit_shim_against_reference():
    assert os.path.exists(BIN), "oracle/_ref/shim_check missing: run __graft_entry__.build()"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "shim ok" in r.stdout, r.stdout + r.stderr
