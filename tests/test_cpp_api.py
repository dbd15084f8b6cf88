"""The C++ drop-in API (include/bcad/*.hpp) on the GPU: reference-style test
programs in tests/cpp/, built by __graft_entry__.build() against
libbcad_cu.so, run here and must report every check passing."""
import glob
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "bin")
PROGRAMS = sorted(glob.glob(os.path.join(BIN, "test_*")))


def test_programs_built():
    assert len(PROGRAMS) >= 2, "run __graft_entry__.build() first"


@pytest.mark.parametrize("exe", PROGRAMS, ids=[os.path.basename(p) for p in PROGRAMS])
def test_cpp_program(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
