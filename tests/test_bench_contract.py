"""bench.py's driver contract that can be checked without a GPU: the reference
arm (`--impl reference`, the reference solver built from its sources into
oracle/_ref) prints one JSON line with the agreed keys on the arm's config."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(*args, timeout=600):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line(ref):
    d = _run("--impl", "reference", "--config", "C1", "--steps", "3", "--warmup", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["metric"] == "D3Q19 TRT fp64 fluid MLUPS" and d["unit"] == "MLUPS"
    assert d["steps"] == 3 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C1") and d["config"]["fluid_cells"] == 61440
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_never_loads_the_product(ref):
    """--impl reference builds its workload from oracle code only (spheres,
    voxelizer checked against the reference-made golden geometry) and times
    oracle/_ref: libporolb_cuda.so must not be mapped in that process."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'C2', "
            "'--steps', '2', '--warmup', '3', '--ref-budget', '1']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\n"
            "except SystemExit:\n    pass\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('PRODUCT_LOADED' if 'libporolb_cuda' in maps else 'PRODUCT_ABSENT')\n"
            "print('REF_LOADED' if 'libporolb_ref' in maps else 'REF_ABSENT')\n")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "PRODUCT_ABSENT" in res.stdout and "REF_LOADED" in res.stdout, res.stdout
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][0])
    assert line["geometry"].startswith("sha256 == tests/golden/C2.json")
    assert line["cpu_baseline"]["cores"] >= 1


def test_both_arms_print_the_same_config(ref, pg):
    """The config dict of --impl reference equals what our arm prints (same
    keys and values), built here from the product workload definition."""
    import bench
    from paper_1507_06565_b200 import configs
    d = _run("--impl", "reference", "--config", "C3", "--steps", "2", "--warmup", "3",
             "--ref-budget", "1")
    w = configs.ALL["C3"]()
    g = w.geometry()
    ours = bench.config_dict(w.name, g.fluid_cells, g.cells, g.n_links, w.scheme.name, 1, w.meta)
    assert d["config"] == json.loads(json.dumps(ours))


def test_unknown_config_is_rejected():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "C9"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert res.returncode != 0


@pytest.mark.gpu
def test_ours_json_line_small(gpu):
    d = _run("--config", "C1", "--steps", "50", "--warmup", "5", "--no-cpu-baseline")
    assert d["value"] > 0 and d["gpu_launches"] >= 1
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"]
    assert d["math"] == "fast"
    pc = d["per_config"]
    assert set(pc) == {"C2", "C3", "C5"}
    for v in pc.values():
        assert v["value"] > 0 and 0 < v["frac"] and v["layout"] in ("dense", "fluid-only",
                                                                       "dense-persistent")
