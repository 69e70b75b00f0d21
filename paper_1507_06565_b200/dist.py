"""x-slab domain decomposition across GPUs.

The global domain is cut along the flow axis x into P contiguous slabs, one
per rank.  In pull form a cell at a slab face needs, from the neighbouring
slab, only the post-collision populations whose velocity points into the
receiving slab: directions {1,7,9,11,13} (e_x=+1) from the left neighbour and
{2,8,10,12,14} (e_x=-1) from the right one; a CLI link's second fluid cell
x_f1 - e_k lies in the ghost column only for those same directions.  So each
face carries exactly 5 PDFs per (y, z): the paper's communication-reducing
ghost-layer exchange.

On the GPU the per-step schedule runs natively in libporolb_cuda.so
(csrc/dist.cpp, `pgpu_dist_*`): edge columns on a high-priority stream, then
the exchange, overlapped with the interior columns on the simulation's
stream; NCCL between processes (one rank per GPU, `SlabSimulation`) or peer
copies between the slabs of one process (`LocalTransport`).  NCCL mode
replays the steady-state schedule as a CUDA graph.  This module only builds
the slab simulations and hands them to that driver.

`DistTransport` keeps the same schedule in Python over torch.distributed for
CPU engines (the oracle slab engine), which is how the host-side logic of the
decomposition is tested with gloo at world size 2 without GPUs.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import numpy as np

from . import porolb as P

# directions crossing an x face (kernels.cu halo_slot order)
TO_RIGHT = (1, 7, 9, 11, 13)   # e_x = +1: leave through x = nx-1
TO_LEFT = (2, 8, 10, 12, 14)   # e_x = -1: leave through x = 0


def slab_ranges(nx: int, world: int) -> List[tuple]:
    """Equal contiguous x ranges of nx / world columns (ConfigError if world
    does not divide nx).  Widths need not be multiples of 32: slabs of >= 96
    columns sweep 32-column edge bands, narrower ones the face columns
    (csrc/lattice.cuh edge_band)."""
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
            # CUDA slab: the native driver (pgpu_dist) owns its halo buffers
            self.sim = P.Simulation.from_params(self.geometry, workload.params(), workload.scheme,
                                                int(device))
            gp = workload.glbm_params()
            if gp is not None:
                self.sim.set_porous(gp)
            tdev = torch.device("cuda", int(device))
            # the slab's interior sweeps and observables run on this torch stream
            self.stream = stream if stream is not None else torch.cuda.Stream(device=tdev)
            self.sim.set_stream(self.stream.cuda_stream)
            return
        self.sim = engine(self.geometry, workload)
        n = self.sim.halo_elems
        mk = lambda: torch.zeros(n, dtype=torch.float64)  # noqa: E731
        self.send_lo, self.send_hi = mk(), mk()
        self.recv_lo = [mk(), mk()]
        self.recv_hi = [mk(), mk()]
        self.sim.set_halo_buffers(self.send_lo, self.send_hi, self.recv_lo[0], self.recv_lo[1],
                                  self.recv_hi[0], self.recv_hi[1])


def _profile_meta(prof: P.ProfileData, params: P.FluidParams, geometry, nz: int) -> None:
    """ProfileData metadata exactly as simulation.cpp:386-397 fills it."""
    prof.nu = params.nu
    prof.body_force = tuple(params.body_force)
    lo, hi = geometry.wall_plane_lo, geometry.wall_plane_hi
    if lo is not None and hi is not None:
        prof.z0, prof.height = float(lo), float(hi) - float(lo)
    else:
        prof.z0, prof.height = 0.0, float(nz)


class NativeDist:
    """The native x-slab driver (csrc/dist.cpp) over slab simulations.

    local mode: `sims` are all slabs of the decomposition in this process
    (peer copies); nccl mode: `sims` is this process's one slab and
    `nccl_id`/`rank`/`world` describe the communicator."""

    def __init__(self, sims, nccl_id: Optional[bytes] = None, rank: int = 0,
                 world: Optional[int] = None, ipc_allgather: Optional[Callable] = None):
        import ctypes as C

        from . import _lib
        self._C, self._lib = C, _lib
        self.sims = list(sims)
        self.world = int(world if world is not None else len(self.sims))
        self._h = C.c_void_p()
        if ipc_allgather is not None:
            # IPC transport: the edge kernel stores into the neighbours' ghost
            # buffers; the blobs travel through the caller's all-gather.  Every
            # step is collective, so a failure on one rank fails them all
            # (self.ok) instead of leaving the others waiting.
            L = _lib.lib
            self.ok = False
            blob = None
            try:
                P._check(L.pgpu_dist_create_ipc(self.sims[0]._h, int(rank), self.world,
                                                C.byref(self._h)))
                n = C.c_int64()
                P._check(L.pgpu_dist_ipc_blob_size(C.byref(n)))
                buf = (C.c_uint8 * n.value)()
                P._check(L.pgpu_dist_ipc_export(self._h, buf))
                blob = bytes(buf)
            except Exception as e:  # noqa: BLE001
                self.error = repr(e)
            blobs = ipc_allgather(blob)
            ok = all(b is not None for b in blobs)
            if ok:
                allb = (C.c_uint8 * len(b"".join(blobs))).from_buffer_copy(b"".join(blobs))
                try:
                    P._check(L.pgpu_dist_ipc_connect(self._h, allb))
                except Exception as e:  # noqa: BLE001
                    self.error = repr(e)
                    ok = False
            self.ok = all(ipc_allgather(ok))
            if not self.ok:
                self.close()
            return
        elif nccl_id is None:
            arr = (C.c_void_p * len(self.sims))(*[s._h.value for s in self.sims])
            P._check(_lib.lib.pgpu_dist_create_local(arr, len(self.sims), C.byref(self._h)))
        else:
            buf = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
            P._check(_lib.lib.pgpu_dist_create_nccl(self.sims[0]._h, buf, int(rank), self.world,
                                                    C.byref(self._h)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        import ctypes as C

        from . import _lib
        buf = (C.c_uint8 * 128)()
        P._check(_lib.lib.pgpu_dist_nccl_unique_id(buf))
        return bytes(buf)

    def step(self, n: int = 1) -> None:
        P._check(self._lib.lib.pgpu_dist_step(self._h, int(n)))

    def set_graphs(self, enable: bool) -> None:
        P._check(self._lib.lib.pgpu_dist_set_graphs(self._h, int(bool(enable))))

    def synchronize(self) -> None:
        P._check(self._lib.lib.pgpu_dist_synchronize(self._h))

    def plane_sums(self, stream_axis: int = 0) -> np.ndarray:
        out = np.zeros(self.sims[0].nz)
        P._check(self._lib.lib.pgpu_dist_plane_sums(self._h, int(stream_axis),
                                                    P._p(out, self._C.c_double)))
        return out

    def max_speed2(self):
        v2, fin = self._C.c_double(), self._C.c_int32()
        P._check(self._lib.lib.pgpu_dist_max_speed2(self._h, self._C.byref(v2),
                                                    self._C.byref(fin)))
        return v2.value, bool(fin.value)

    def max_speed(self) -> float:
        v2, fin = self.max_speed2()
        return float(np.sqrt(v2)) if fin else float("nan")

    def planar_profile(self, stream_axis: int = 0) -> P.ProfileData:
        """simulation.cpp:371-417 over the whole domain (per-rank plane sums
        added across ranks: equal to the reference within rounding)."""
        nz = self.sims[0].nz
        bufs = [np.zeros(nz) for _ in range(5)]
        meta = self._lib.ProfileMeta()
        P._check(self._lib.lib.pgpu_dist_planar_profile(
            self._h, int(stream_axis), *[P._p(b, self._C.c_double) for b in bufs],
            self._C.byref(meta)))
        return P._profile(bufs, meta)

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self._lib.lib.pgpu_dist_destroy(self._h)
            self._h = self._C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class DistTransport:
    """CPU engines: the native schedule restated over torch.distributed
    (gloo), one rank per process (host-logic tests of the decomposition)."""

    def __init__(self, rank: SlabRank, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.me = rank
        self.group = group
        self.left = (rank.rank - 1) % rank.world
        self.right = (rank.rank + 1) % rank.world

    def _exchange(self):
        me, dist = self.me, self.dist
        p = me.sim.halo_parity
        if me.world == 1:
            me.recv_hi[p].copy_(me.send_lo)
            me.recv_lo[p].copy_(me.send_hi)
            return []
        # same per-peer order as csrc/dist.cpp (matching does not rely on tags)
        ops = [dist.P2POp(dist.isend, me.send_lo, self.left, self.group, tag=0),
               dist.P2POp(dist.isend, me.send_hi, self.right, self.group, tag=1),
               dist.P2POp(dist.irecv, me.recv_hi[p], self.right, self.group, tag=0),
               dist.P2POp(dist.irecv, me.recv_lo[p], self.left, self.group, tag=1)]
        return dist.batch_isend_irecv(ops)

    def step(self, n: int = 1) -> None:
        me = self.me
        for _ in range(int(n)):
            me.sim.step_part(0)  # edge columns -> send buffers
            reqs = self._exchange()
            me.sim.step_part(1)  # interior columns
            me.sim.step_finish()
            for req in reqs:  # the next step's edge part reads the new ghosts
                req.wait()

    # -- collective observables ---------------------------------------------
    def _allreduce(self, values, op="sum"):
        import torch

        t = torch.tensor(np.asarray(values, dtype=np.float64))
        if self.me.world > 1:
            rop = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX,
                   "min": self.dist.ReduceOp.MIN}[op]
            self.dist.all_reduce(t, op=rop, group=self.group)
        return t.numpy()

    def fluid_cells(self) -> int:
        return int(self._allreduce([self.me.sim.fluid_cells])[0])

    def planar_profile(self, stream_axis: int = 0) -> P.ProfileData:
        """simulation.cpp:371-417 over the whole domain (per-rank plane sums
        combined with all_reduce; equal to the reference within rounding)."""
        me = self.me
        g = me.geometry
        nx_loc, ny, nz = g.dims
        sums = self._allreduce(me.sim.plane_sums(stream_axis))
        counts = self._allreduce(np.round(np.asarray(g.porosity) * nx_loc * ny))
        plane = float(me.workload.dims[0] * ny)
        prof = P.ProfileData()
        prof.stream_axis = stream_axis
        _profile_meta(prof, me.workload.params(), g, nz)
        nzp = [z for z in range(nz) if counts[z] > 0]
        if not nzp:
            return prof
        zl, zh = nzp[0], nzp[-1]
        zs = np.arange(zl, zh + 1)
        prof.z = zs + 0.5
        prof.u_superficial = sums[zl:zh + 1] / plane
        cnt = counts[zl:zh + 1]
        prof.u_intrinsic = np.where(cnt > 0, sums[zl:zh + 1] / np.maximum(cnt, 1), 0.0)
        prof.epsilon = cnt / plane
        u_max = 0.0
        for v in prof.u_superficial:  # profile.cpp:10-19 (first largest |u|)
            if abs(v) > abs(u_max):
                u_max = float(v)
        prof.u_max = u_max
        prof.u_normalized = prof.u_superficial / u_max if u_max != 0.0 else 0 * prof.z
        return prof

    def max_speed(self) -> float:
        v2, fin = self.me.sim.max_speed2()
        v2 = self._allreduce([v2], "max")[0]
        fin = self._allreduce([1.0 if fin else 0.0], "min")[0]
        return float(np.sqrt(v2)) if fin > 0 else float("nan")


class SlabSimulation:
    """One rank's slab (the handle bench.py uses): SlabSimulation(workload,
    rank, world).  CUDA: the native driver in NCCL mode (the unique id travels
    over torch.distributed when it is initialised); CPU engines: DistTransport."""

    def __init__(self, workload, rank: int, world: int, device=0, group=None, engine=None,
                 geometry=None, transport: str = "nccl"):
        self.me = SlabRank(workload, rank, world, device, engine, geometry=geometry)
        self.sim = self.me.sim
        self.workload = workload
        self._cpu = None
        self.native = None
        self.transport = transport if engine is None else "gloo"
        if engine is not None:
            self._cpu = DistTransport(self.me, group)
            return
        nid = None
        import torch.distributed as tdist
        if transport == "ipc":
            def allgather(obj):
                if world == 1:
                    return [obj]
                out = [None] * world
                tdist.all_gather_object(out, obj, group=group)
                return out
            nd = NativeDist([self.sim], rank=rank, world=world, ipc_allgather=allgather)
            if nd.ok:
                self.native = nd
                return
            # CUDA IPC unavailable on some rank: every rank falls back to NCCL
            import warnings
            warnings.warn(f"IPC halo transport unavailable ({getattr(nd, 'error', 'another rank')}); "
                          "using NCCL")
            self.transport = "nccl"
        if world > 1 and tdist.is_available() and tdist.is_initialized():
            obj = [NativeDist.nccl_unique_id() if rank == 0 else None]
            tdist.broadcast_object_list(obj, src=0, group=group)
            nid = obj[0]
        elif world == 1:
            nid = NativeDist.nccl_unique_id()
        else:
            raise P.ConfigError("world > 1 needs torch.distributed initialised (NCCL id exchange)")
        self.native = NativeDist([self.sim], nccl_id=nid, rank=rank, world=world)

    def step(self, n: int = 1) -> None:
        (self._cpu or self.native).step(n)

    def planar_profile(self, stream_axis: int = 0) -> P.ProfileData:
        return (self._cpu or self.native).planar_profile(stream_axis)

    def max_speed(self) -> float:
        return (self._cpu or self.native).max_speed()

    def fluid_cells(self) -> int:
        if self._cpu is not None:
            return self._cpu.fluid_cells()
        return int(self.workload_fluid_total())

    def workload_fluid_total(self) -> int:
        counts = np.round(np.asarray(self.me.geometry.porosity) * self.me.geometry.dims[0]
                          * self.me.geometry.dims[1])
        import torch.distributed as tdist
        if self.me.world > 1 and tdist.is_initialized():
            import torch
            dev = "cpu" if tdist.get_backend() == "gloo" else "cuda"
            t = torch.tensor([counts.sum()], dtype=torch.float64, device=dev)
            tdist.all_reduce(t)
            return int(t.item())
        return int(counts.sum())

    def close(self) -> None:
        if self.native is not None:
            self.native.close()


class LocalTransport:
    """All slabs of a decomposition in ONE process: on the GPU the native
    driver in local mode (peer copies; edge and interior parts on two streams
    per slab), for CPU engines the same steps in order.  Verifies the
    decomposition bit for bit against the single domain on one device."""

    def __init__(self, workload, world: int, device=0, engine=None):
        self.world = world
        self.ranks = [SlabRank(workload, r, world, device, engine) for r in range(world)]
        self.native = None if engine is not None else NativeDist([r.sim for r in self.ranks])

    def step(self, n: int = 1) -> None:
        if self.native is not None:
            self.native.step(n)
            return
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

    def planar_profile(self, stream_axis: int = 0) -> P.ProfileData:
        return self.native.planar_profile(stream_axis)

    def max_speed(self) -> float:
        return self.native.max_speed()

    def gather_pdfs(self) -> np.ndarray:
        """Global f(n) (19, nz, ny, nx) assembled from the slabs."""
        parts = [r.sim.get_pdfs() for r in self.ranks]
        return np.concatenate(parts, axis=3)
