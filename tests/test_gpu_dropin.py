"""The C++ drop-in (paper_1709_04145_b200/dropin: pbad::gpu::batch_simulate /
simulate with the reference's own KinematicModel / ForceModel / SimConfig /
Trajectory types) against the reference's own batch_simulate / simulate on
the same inputs: tests/dropin/dropin_check.cpp, built by oracle/ref/Makefile
where /root/reference exists and shipped with the tree.  Every Trajectory
field must be equal, error texts included."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK = os.path.join(ROOT, "oracle", "_ref", "pbad_dropin_check")


def test_dropin_matches_reference_batch_simulate():
    if not os.path.exists(CHECK):
        pytest.fail(f"{CHECK} was not built (needs /root/reference headers at build time)")
    r = subprocess.run([CHECK], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "DROPIN ALL EQUAL" in r.stdout
