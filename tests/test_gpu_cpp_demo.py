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


def test_dns_dropin_resolve_drive(gpu, ref):
    """The reference's make_simulation/run_to_steady (dns.cpp:11-22) compiled
    unchanged against the C++ mirror: a pressure-gradient drive resolved by
    resolve_drive() runs to the same steady state as the reference."""
    exe = Path(__file__).resolve().parent / "cpp" / "dns_dropin"
    assert exe.exists(), "build with python paper_1507_06565_b200/build.py"
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    got = dict(kv.split("=") for kv in res.stdout.split())
    g = ref.resolve_drive(1, (4e-8, 0.0, 0.0), 0, 4.0)
    assert float(got["g"]) == g[0] == 1e-8
    geom = ref.make_box_geometry((4, 4, 18), (True, True, False), True, True)
    wp, wm = ref.relaxation_from_magic(1.0 / 6.0, 3.0 / 16.0)
    r = ref.simulation(geom, 1.0 / 6.0, wp, wm, 3.0 / 16.0, g, 0)
    st = r.run_to_steady_state(1e-10, 500, 20000)
    assert int(got["steps"]) == st["steps"] and int(got["converged"]) == int(st["converged"])
    assert float(got["u_max"]) == r.planar_profile()["u_max"]
    assert float(got["eps_wall"]) == 0.0 and float(got["eps_mid"]) == 1.0


def test_dist_demo_cpp_multi_gpu_host_path(gpu):
    """DistSimulation (C++ over csrc/dist.cpp): 2 and 3 slabs through the local
    transport, and the NCCL transport at world size 1 (periodic self-exchange,
    CUDA-graph replay) -- both bit-identical to the single domain."""
    exe = Path(__file__).resolve().parent / "cpp" / "dist_demo"
    assert exe.exists(), "build with python paper_1507_06565_b200/build.py"
    for args in (["256", "64", "96", "2", "23"], ["192", "40", "64", "3", "16"]):
        res = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stdout + res.stderr
        # (NCCL may print its version banner on stdout first)
        out = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
        assert out["local_bitwise"] and out["local_profile"] and out["local_vmax_equal"], out
        assert out["nccl_error"] == "", out["nccl_error"]
        assert out["nccl_bitwise"] and out["nccl_profile"] and out["nccl_vmax_equal"], out


def test_dist_demo_cpp_ipc_world2(gpu):
    """DistSimulation::ipc (C++): two processes (fork, blobs through pipes) on
    one B200, the edge kernels storing into each other's ghost buffers; each
    slab bit-identical to the single domain, profile and max speed equal."""
    exe = Path(__file__).resolve().parent / "cpp" / "dist_demo"
    res = subprocess.run([str(exe), "ipc", "128", "32", "48", "15"], capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    out = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["error"] == "" and out["rank0_ok"] and out["rank1_ok"], (out, res.stderr[-2000:])
