"""Host-side check of the block-recurrence sweep schedules (setup_host.hpp
BlkStream) used by the reassociated mode: tests/cpp/blk_emulate.cpp decodes
the stream images and runs them block by block on the CPU (old sums, fresh
sums, dense block inverse), against the sequential ILUT substitutions
(ilut.hpp:146-163) and Gauss-Seidel sweeps (solvers.hpp:80-99)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2107_05337_b200", "csrc")


@pytest.fixture(scope="module")
def emulator(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("blk") / "blk_emulate")
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{CSRC}", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "blk_emulate.cpp"), os.path.join(CSRC, "setup_host.cpp"),
                    "-o", exe], check=True, capture_output=True)
    return exe


# (grid m, stencil half-width w): IgA-like patterns of degree 1..5, ragged
# last blocks (n % 32 != 0), tiny systems (one block)
@pytest.mark.parametrize("m,w", [(40, 3), (33, 1), (70, 1), (17, 2), (5, 1), (3, 1), (30, 5)])
def test_block_sweeps_match_sequential(emulator, m, w):
    r = subprocess.run([emulator, str(m), str(w)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
