"""Timing of the file-format row against the reference's own
io.cpp (oracle/_ref, all host threads for its OpenMP parts; its writers and
readers are single-threaded by construction).

  * write_vtk on the C2 workload (128x64x128) after 200 steps: ours (device
    moments + threaded formatting) vs reference (same state via set_pdfs);
    the two files must be byte-identical.
  * write_voxel_file / read_voxel_file on the C4 flag field (512x256x512).

Prints one JSON object.  Usage: python tools/bench_io.py [--out FILE]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def _sha(p):
    h = hashlib.sha256()
    with open(p, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 24), b""):
            h.update(chunk)
    return h.hexdigest()


def _timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return time.perf_counter() - t0, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--tmp", default=None)
    args = ap.parse_args()

    import paper_1507_06565_b200 as pg
    from paper_1507_06565_b200 import configs
    from oracle.oracle import load_ref

    ref = load_ref()
    threads = ref.set_threads(os.cpu_count() or 1)
    tmp = Path(args.tmp or tempfile.mkdtemp(prefix="pgpu_io_"))
    res = {"host_threads": os.cpu_count(), "ref_threads": threads, "tmpdir": str(tmp)}

    # --- VTK on C2 ------------------------------------------------------------
    w = configs.c2()
    geom = w.geometry()
    sim = configs.make_simulation(w, geom)
    sim.step(200)
    sim.synchronize()
    p = w.params()
    rs = ref.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.lambda_magic, p.body_force,
                        int(w.scheme))
    rs.set_pdfs(sim.get_pdfs())
    ours, theirs = tmp / "c2_ours.vtk", tmp / "c2_ref.vtk"
    pg.write_vtk(ours, sim)  # warm (page cache, device buffers)
    t_ours = min(_timed(lambda: pg.write_vtk(ours, sim))[0] for _ in range(3))
    t_ref, _ = _timed(lambda: rs.write_vtk(theirs))
    size = ours.stat().st_size
    same = ours.stat().st_size == theirs.stat().st_size and _sha(ours) == _sha(theirs)
    res["write_vtk"] = {"workload": "C2 128x64x128, 200 steps", "cells": geom.cells,
                        "bytes": size, "ours_s": t_ours, "ref_s": t_ref,
                        "speedup": t_ref / t_ours, "ours_MBps": size / t_ours / 1e6,
                        "identical": bool(same)}
    ours.unlink()
    theirs.unlink()
    del rs

    # --- voxel file on C4 -----------------------------------------------------
    w4 = configs.c4()
    g4 = pg.voxelize_device(w4.pack, w4.dims, **w4.voxelize_options())
    vo, vr = tmp / "c4_ours.vox", tmp / "c4_ref.vox"
    t_wo, _ = _timed(lambda: pg.write_voxel_file(vo, g4))
    t_wr, _ = _timed(lambda: ref.write_voxel_file(vr, g4))
    same_w = _sha(vo) == _sha(vr)
    t_ro, q = _timed(lambda: pg.read_voxel_file(vr))
    t_rr, r = _timed(lambda: ref.read_voxel_file(vr))
    same_r = (np.array_equal(q.link_fluid_cell, r.link_fluid_cell)
              and np.array_equal(q.link_second_fluid, r.link_second_fluid)
              and np.array_equal(q.link_direction, r.link_direction)
              and np.array_equal(q.porosity, r.porosity) and q.fluid_cells == r.fluid_cells)
    res["voxel_file"] = {"workload": "C4 512x256x512 flags", "cells": g4.cells,
                         "links": q.n_links, "write_ours_s": t_wo, "write_ref_s": t_wr,
                         "write_identical": bool(same_w), "read_ours_s": t_ro,
                         "read_ref_s": t_rr, "read_speedup": t_rr / t_ro,
                         "read_identical": bool(same_r)}
    vo.unlink()
    vr.unlink()
    line = json.dumps(res)
    print(line)
    if args.out:
        Path(args.out).write_text(line + "\n")


if __name__ == "__main__":
    main()
