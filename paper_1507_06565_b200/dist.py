"""x-slab domain decomposition across GPUs.

The global domain is cut along the flow axis x into P contiguous slabs, one
per rank (one process per GPU).  In pull form a cell at a slab face needs,
from the neighbouring slab, only the post-collision populations whose
velocity points into the receiving slab: directions {1,7,9,11,13} (e_x=+1)
from the left neighbour and {2,8,10,12,14} (e_x=-1) from the right one; a CLI
link's second fluid cell x_f1 - e_k lies in the ghost column only for those
same directions.  So each face carries exactly 5 PDFs per (y, z): the
paper's communication-reducing ghost-layer exchange.

Per step and rank (DistTransport), on two CUDA streams:
  1. edge stream: step_part(0) pulls/collides the edge columns x=0 and
     x=nx-1 and writes their 5 outgoing PDFs to the send buffers, then the
     exchange (NCCL send/recv through torch.distributed) fills the
     neighbours' ghost buffers of the next parity;
  2. compute stream: step_part(1), the interior columns, concurrently;
  3. step_finish(): buffer swap, parity flip.
Interior cells never read ghosts, so the only cross-stream orderings are the
column dependencies between consecutive steps: the edge part of step n+1
waits for the interior of step n (and for the exchange of step n, in stream
order), the interior of step n+1 waits for the edge part of step n.
The exchange is the only data-path collective; observables combine per-rank
partial sums with all_reduce.  LocalTransport runs all slabs in one process on
one device (sequentially, no kernel ever waits on another), which is how the
decomposition is verified bit-for-bit on a single GPU.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import numpy as np

from . import porolb as P

# directions crossing an x face (kernels.cu halo_slot order)
TO_RIGHT = (1, 7, 9, 11, 13)   # e_x = +1: leave through x = nx-1
TO_LEFT = (2, 8, 10, 12, 14)   # e_x = -1: leave through x = 0


def slab_ranges(nx: int, world: int) -> List[tuple]:
    """Equal contiguous x ranges; every slab keeps a multiple of 32 cells
    when possible so rows stay warp-aligned."""
    if nx % world:
        raise P.ConfigError(f"nx={nx} is not divisible by {world} ranks")
    w = nx // world
    return [(r * w, (r + 1) * w) for r in range(world)]


def _on(stream):
    """Context that makes `stream` torch's current stream (no-op on CPU)."""
    import contextlib

    if stream is None:
        return contextlib.nullcontext()
    import torch

    return torch.cuda.stream(stream)


class SlabRank:
    """One slab: a slab-mode Simulation (or a compatible engine) plus its
    send/receive halo buffers (torch tensors on the engine's device)."""

    def __init__(self, workload, rank: int, world: int, device=0, engine: Optional[Callable] = None,
                 stream=None, geometry=None):
        import torch

        self.rank, self.world = rank, world
        self.stream = None
        self.workload = workload
        self.x0, self.x1 = slab_ranges(workload.dims[0], world)[rank]
        self.geometry = geometry if geometry is not None else workload.geometry_slab(self.x0, self.x1)
        if engine is None:
            self.sim = P.Simulation.from_params(self.geometry, workload.params(), workload.scheme,
                                                int(device))
            gp = workload.glbm_params()
            if gp is not None:
                self.sim.set_porous(gp)
            tdev = torch.device("cuda", int(device))
            # kernels, halo copies and NCCL calls are ordered on one torch stream
            self.stream = stream if stream is not None else torch.cuda.Stream(device=tdev)
            self.sim.set_stream(self.stream.cuda_stream)
        else:
            self.sim = engine(self.geometry, workload)
            tdev = torch.device("cpu")
        n = self.sim.halo_elems
        mk = lambda: torch.zeros(n, dtype=torch.float64, device=tdev)  # noqa: E731
        self.send_lo, self.send_hi = mk(), mk()
        self.recv_lo = [mk(), mk()]
        self.recv_hi = [mk(), mk()]
        self.sim.set_halo_buffers(self.send_lo, self.send_hi, self.recv_lo[0], self.recv_lo[1],
                                  self.recv_hi[0], self.recv_hi[1])


class DistTransport:
    """One rank per process; neighbours over torch.distributed (NCCL / gloo)."""

    def __init__(self, rank: SlabRank, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.me = rank
        self.group = group
        self.left = (rank.rank - 1) % rank.world
        self.right = (rank.rank + 1) % rank.world

    def step(self, n: int = 1) -> None:
        if self.me.stream is None:  # CPU engine: one ordered sequence
            self._step_serial(n)
            return
        self._step_two_streams(n)

    def _exchange(self):
        me, dist = self.me, self.dist
        p = me.sim.halo_parity
        if me.world == 1:
            me.recv_hi[p].copy_(me.send_lo)
            me.recv_lo[p].copy_(me.send_hi)
            return []
        ops = [dist.P2POp(dist.isend, me.send_lo, self.left, self.group, tag=0),
               dist.P2POp(dist.isend, me.send_hi, self.right, self.group, tag=1),
               dist.P2POp(dist.irecv, me.recv_hi[p], self.right, self.group, tag=0),
               dist.P2POp(dist.irecv, me.recv_lo[p], self.left, self.group, tag=1)]
        return dist.batch_isend_irecv(ops)

    def _step_serial(self, n: int) -> None:
        me = self.me
        for _ in range(int(n)):
            me.sim.step_part(0)  # edge columns -> send buffers
            reqs = self._exchange()
            me.sim.step_part(1)  # interior columns
            me.sim.step_finish()
            for req in reqs:  # the next step's edge part reads the new ghosts
                req.wait()

    def _step_two_streams(self, n: int) -> None:
        import torch

        me = self.me
        main = me.stream
        if getattr(self, "_edge_stream", None) is None:
            # high priority: the edge part (and the exchange ordered after it)
            # is dispatched ahead of the interior sweep's remaining blocks
            self._edge_stream = torch.cuda.Stream(device=main.device, priority=-1)
        edge = self._edge_stream
        edge.wait_stream(main)  # everything issued before step() on the main stream
        prev_edge = None
        for _ in range(int(n)):
            ev_main = torch.cuda.Event()
            ev_main.record(main)  # interior of the previous step
            with torch.cuda.stream(edge):
                edge.wait_event(ev_main)
                me.sim.step_part(0, edge.cuda_stream)  # edge columns -> send buffers
                ev_edge = torch.cuda.Event()
                ev_edge.record(edge)
                for req in self._exchange():  # in edge-stream order
                    req.wait()
            if prev_edge is not None:  # the interior reads/overwrites the previous
                main.wait_event(prev_edge)  # step's edge columns
            me.sim.step_part(1, main.cuda_stream)  # interior, concurrent with edge + exchange
            me.sim.step_finish()
            prev_edge = ev_edge
        main.wait_stream(edge)  # step() returns with all work ordered on the main stream

    # -- collective observables ---------------------------------------------
    def _allreduce(self, values, op="sum"):
        import torch

        t = torch.tensor(np.asarray(values, dtype=np.float64), device=self.me.send_lo.device)
        if self.me.world > 1:
            rop = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX,
                   "min": self.dist.ReduceOp.MIN}[op]
            self.dist.all_reduce(t, op=rop, group=self.group)
        return t.cpu().numpy()

    def fluid_cells(self) -> int:
        return int(self._allreduce([self.me.sim.fluid_cells])[0])

    def planar_profile(self, stream_axis: int = 0) -> P.ProfileData:
        """simulation.cpp:371-417 over the whole domain (per-rank plane sums
        combined with all_reduce; equal to the reference within rounding)."""
        me = self.me
        g = me.geometry
        nx_loc, ny, nz = g.dims
        sums = self._allreduce(me.sim.plane_sums(stream_axis))
        counts = self._allreduce(np.asarray(g.porosity) * nx_loc * ny)
        plane = float(me.workload.dims[0] * ny)
        nzp = [z for z in range(nz) if round(counts[z]) > 0]
        prof = P.ProfileData()
        if not nzp:
            return prof
        zl, zh = nzp[0], nzp[-1]
        zs = np.arange(zl, zh + 1)
        prof.z = zs + 0.5
        prof.u_superficial = sums[zl:zh + 1] / plane
        cnt = np.round(counts[zl:zh + 1])
        prof.u_intrinsic = np.where(cnt > 0, sums[zl:zh + 1] / np.maximum(cnt, 1), 0.0)
        prof.epsilon = cnt / plane
        i = int(np.argmax(np.abs(prof.u_superficial)))
        prof.u_max = float(prof.u_superficial[i])
        prof.u_normalized = prof.u_superficial / prof.u_max if prof.u_max else 0 * prof.z
        prof.stream_axis = stream_axis
        return prof

    def max_speed(self) -> float:
        v2, fin = self.me.sim.max_speed2()
        v2 = self._allreduce([v2], "max")[0]
        fin = self._allreduce([1.0 if fin else 0.0], "min")[0]
        return float(np.sqrt(v2)) if fin > 0 else float("nan")


class SlabSimulation(DistTransport):
    """The rank-local handle bench.py uses: SlabSimulation(workload, rank, world)."""

    def __init__(self, workload, rank: int, world: int, device=0, group=None, engine=None,
                 geometry=None):
        super().__init__(SlabRank(workload, rank, world, device, engine, geometry=geometry), group)
        self.sim = self.me.sim

    def set_stream(self, stream) -> None:
        self.me.stream = stream
        self.sim.set_stream(stream.cuda_stream)


class LocalTransport:
    """All slabs of a decomposition in ONE process on one device.  Each step
    runs every slab's edge part, then the exchanges (device copies), then the
    interior parts -- sequentially, so no kernel waits on another.  Used to
    verify the decomposition bit-for-bit on one GPU (and on CPU engines)."""

    def __init__(self, workload, world: int, device=0, engine=None):
        import torch

        self.stream = None if engine is not None else torch.cuda.Stream(device=int(device))
        self.ranks = [SlabRank(workload, r, world, device, engine, self.stream)
                      for r in range(world)]
        self.world = world

    def step(self, n: int = 1) -> None:
        with _on(self.stream):
            self._step(n)

    def _step(self, n: int) -> None:
        R, W = self.ranks, self.world
        for _ in range(int(n)):
            for r in R:
                r.sim.step_part(0)
            for i, r in enumerate(R):
                p = r.sim.halo_parity
                left, right = R[(i - 1) % W], R[(i + 1) % W]
                left.recv_hi[p].copy_(r.send_lo)
                right.recv_lo[p].copy_(r.send_hi)
            for r in R:
                r.sim.step_part(1)
            for r in R:
                r.sim.step_finish()

    def gather_pdfs(self) -> np.ndarray:
        """Global f(n) (19, nz, ny, nx) assembled from the slabs."""
        parts = [r.sim.get_pdfs() for r in self.ranks]
        return np.concatenate(parts, axis=3)
