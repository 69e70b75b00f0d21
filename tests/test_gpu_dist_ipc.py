"""The IPC transport of the multi-GPU driver (csrc/dist.cpp) at world sizes
2 and 3 with one process per rank -- the only multi-process data path that
can run on a single B200 (NCCL refuses two ranks on one device): the
edge-column kernel stores its 5 outgoing PDFs per face straight into the
neighbour's ghost buffer through a CUDA IPC mapping, and the ranks order
each other with interprocess events and the shared-memory handshake (stream
waits only: no kernel spins on another rank).  Every slab must equal the
single-domain run bit for bit (tests/mp/ipc_world.py)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("world,nx,scheme", [(2, 128, 1), (2, 96, 0), (3, 96, 1)])
def test_ipc_transport_world(gpu, world, nx, scheme):
    env = dict(os.environ, IPC_NX=str(nx), IPC_SCHEME=str(scheme), PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", "--master-port=29533",
           str(ROOT / "tests" / "mp" / "ipc_world.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    line = [l for l in res.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    assert out["world"] == world
    assert all(out["slabs_equal"]), out
    assert out["profile_ok"] and out["max_speed_ok"], out


def test_bench_two_ranks_one_device(gpu):
    """The N > 1 bench path end to end (torchrun, slab geometry, IPC halo
    transport, timing, e2e, --verify) with both ranks on cuda:0 and gloo for
    the host-side collectives: every slab of C4 after warm-up + timed steps
    equals the single-GPU run bit for bit."""
    env = dict(os.environ, PGPU_BENCH_ONE_DEVICE="1", PGPU_BENCH_BACKEND="gloo",
               PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29545", str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "6", "--warmup", "3", "--scaling", "strong", "--verify", "--transport", "ipc",
           "--no-cpu-baseline"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    d = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["halo_transport"] == "ipc"
    assert d["config"]["parallelism"] == "x-slab2"
    assert d["parity"]["parity_ok"] is True, d["parity"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
