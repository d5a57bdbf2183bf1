"""The reference-side binding (integration/miga_phi.hpp), compiled against the
reference's own headers into integration/_build/test_binding by
integration/Makefile (run by __graft_entry__.build() where /root/reference
exists; the binary travels to the GPU box).  It runs the reference's
MgritSolver / ThetaStepper and the binding's DeviceMgritSolver /
DeviceThetaStepper -- constructed exactly like the reference classes, from a
miga::SpatialDiscretization and ProblemSpec with std::function sources --
on identical inputs and requires bit-identical results."""
import os
import subprocess

import pytest

from tests.conftest import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "integration", "_build", "test_binding")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def test_binding_bit_identical_to_reference_classes():
    if not os.path.exists(EXE):
        pytest.skip("integration/_build/test_binding not built (make -C integration, needs /root/reference)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all cases bit-identical" in r.stdout
