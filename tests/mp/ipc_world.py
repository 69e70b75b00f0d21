"""One rank of the IPC-transport check (tests/test_gpu_dist_ipc.py): launched
by torch.distributed.run with WORLD_SIZE ranks (gloo carries only the IPC
blobs and the result hashes).  Every rank runs its x-slab on cuda:0 through
the native IPC transport -- the edge kernel stores its 5 outgoing PDFs per
face into the neighbours' ghost buffers (CUDA IPC), interprocess events and
the shared-memory handshake order the ranks -- and rank 0 compares every
slab bit for bit with a single-domain run, plus the global profile and max
speed.  Prints one JSON line on rank 0."""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.getcwd()))


def main():
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    import paper_1507_06565_b200 as pg
    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import SlabSimulation, slab_ranges

    nx = int(os.environ.get("IPC_NX", "128"))
    scheme = int(os.environ.get("IPC_SCHEME", "1"))
    rng = np.random.default_rng(5)
    n = 30
    c = np.c_[rng.uniform(0, nx, n), rng.uniform(0, 24, n), rng.uniform(1, 16, n)]
    r = rng.uniform(2.0, 5.0, n)
    pack = pg.SpherePack(c, r, (float(nx), 24.0, 32.0))
    w = configs.Workload("ipc_test", (nx, 24, 32), pg.WallScheme(scheme), 0.07,
                         (3e-6, -1e-6, 2e-7), 23, pack=pack)
    ss = SlabSimulation(w, rank, world, device=0, transport="ipc")
    ss.step(7)
    prof_mid = ss.planar_profile()  # an observable between step batches (KP + reductions)
    ss.step(w.steps - 7)
    prof = ss.planar_profile()
    vmax = ss.max_speed()
    g = ss.me.geometry
    f = ss.sim.get_pdfs()
    fl = g.flags.reshape(g.dims[::-1]) == 0
    mine = hashlib.sha256(np.ascontiguousarray(f[:, fl]).tobytes()).hexdigest()
    hashes = [None] * world
    dist.all_gather_object(hashes, mine)
    if rank == 0:
        full = w.geometry()
        sim = configs.make_simulation(w, full, device=0)
        sim.step(7)
        ref_mid = sim.planar_profile()
        sim.step(w.steps - 7)
        ref = sim.planar_profile()
        fr = sim.get_pdfs()
        flags = full.flags.reshape(w.dims[::-1]) == 0
        ok = []
        for q, (x0, x1) in enumerate(slab_ranges(nx, world)):
            h = hashlib.sha256(np.ascontiguousarray(fr[..., x0:x1][:, flags[..., x0:x1]]).tobytes())
            ok.append(h.hexdigest() == hashes[q])

        def close(a, b):
            return bool(np.allclose(a, b, rtol=1e-12, atol=1e-12 * max(1e-300, np.abs(b).max())))

        out = {"world": world, "slabs_equal": ok,
               "profile_ok": close(prof.u_superficial, ref.u_superficial)
               and close(prof_mid.u_superficial, ref_mid.u_superficial)
               and np.array_equal(prof.z, ref.z) and prof.height == ref.height,
               "max_speed_ok": abs(vmax - sim.max_speed()) <= 1e-12 * abs(sim.max_speed())}
        print(json.dumps(out), flush=True)
    dist.barrier()
    ss.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
