"""The C++ drop-in (tools/porolb_gpu_demo.cpp over include/porolb_gpu/porolb_gpu.hpp):
reference acceptance criteria 1 (Poiseuille exactness) and 10 (bench sanity,
CLI >= 0.75 x SBB MLUPS on the 128^3 sphere-in-box) run through the C++ API,
plus the scenario files (profile / sphere CSV, voxel file) written and read back."""
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
DEMO = Path(__file__).resolve().parent.parent / "tools" / "porolb_gpu_demo"


def test_cpp_demo_acceptance(gpu):
    assert DEMO.exists(), "build with python paper_1507_06565_b200/build.py"
    res = subprocess.run([str(DEMO)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    out = json.loads(res.stdout)
    assert out["poiseuille_converged"] and out["poiseuille_max_rel_err"] <= 1e-8
    assert out["cli_over_sbb"] >= 0.75
    assert out["bench_cells"] == 128 ** 3
    assert out["io_round_trip"]  # profile/sphere CSV + voxel file through the io.hpp mirror
