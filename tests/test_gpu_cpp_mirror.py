"""The C++ host mirror (include/dynsurf_b200.hpp) driven like the reference's
process_sequence loop: config/dimension errors rethrown as the reference's
exception types, frames processed, model downloaded."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(REPO, "paper_1904_13073_b200", "build", "pipeline_demo")


def test_cpp_mirror_pipeline_demo():
    if not os.path.exists(DEMO):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "paper_1904_13073_b200")],
                       check=True)
    out = subprocess.run([DEMO, "rigid_orbit", "4"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 4
    assert lines[0]["surfel_count"] == lines[0]["valid_pixels"] > 500
    assert all(l["correspondences"] > 500 for l in lines[1:])
    assert out.stdout.strip().splitlines()[-1].startswith("ok ")
