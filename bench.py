"""Benchmark: D3Q19 TRT fp64 fluid MLUPS on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--scaling weak|strong]
    python bench.py --impl reference ...     # the reference CPU solver (oracle/_ref)

Workload: config C4 (512x256x512 pore-scale bed, CLI, the largest single-GPU
BASELINE config and the one its 1/2/4/8-GPU scaling is quoted on); N>1 runs
one rank per GPU over an x-slab split with the 5-PDF halo (weak scaling:
512x256x512 cells per GPU).  The 20 GB of PDFs are far larger than the 126 MB
L2, so no flush is needed between timed steps.

One JSON line on rank 0.  `value` = fluid cells x K / device time (max over
ranks), inputs resident in HBM; `e2e` = the same metric through the C ABI
from host buffers (geometry upload + K steps + download of f(K) and the
profile inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def physical_cores() -> int:
    """Physical cores among the CPUs this process may run on (SMT siblings
    counted once), from /sys topology; falls back to the logical count."""
    try:
        cpus = sorted(os.sched_getaffinity(0))
        seen = set()
        for c in cpus:
            f = Path(f"/sys/devices/system/cpu/cpu{c}/topology/thread_siblings_list")
            seen.add(f.read_text().strip() if f.exists() else str(c))
        return max(1, len(seen))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# CPU legs (cpu_baseline, --impl reference): one OpenMP thread per physical
# core, bound compactly.  Set before any OpenMP runtime starts.
CPU_THREADS = physical_cores()
os.environ.setdefault("OMP_NUM_THREADS", str(CPU_THREADS))
os.environ.setdefault("OMP_PLACES", "cores")
os.environ.setdefault("OMP_PROC_BIND", "close")

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0
BYTES_PER_FLUID_CELL = 304  # 19 fp64 reads + 19 fp64 writes


def hbm_peak():
    try:
        pk = json.loads(PEAKS_FILE.read_text())
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.first = 0

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        """Call right before the timed region: waits for nvidia-smi's first
        sample (its start-up takes longer than a short timed region) and
        drops everything sampled before the region."""
        if not self.proc:
            return
        t_end = time.time() + 3.0
        while not self.lines and time.time() < t_end:
            time.sleep(0.01)
        self.first = len(self.lines)

    def stop(self):
        if not self.proc:
            return None
        late = False
        if len(self.lines) <= self.first:  # timed region shorter than one sampling period
            late = True
            t_end = time.time() + 3.0
            while len(self.lines) <= self.first and time.time() < t_end:
                time.sleep(0.02)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[self.first:]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
               "samples": len(sm)}
        if late:
            out["note"] = "timed region shorter than the 100 ms sampling period; sampled after it"
        return out


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PGPU_BENCH_ONE_DEVICE") == "1":
        local = 0  # test knob: every rank on cuda:0 (the IPC transport's multi-process check)
    return rank, world, local


def all_reduce(dist, t, op=None):
    """torch.distributed all-reduce of a CUDA tensor; through host memory when
    the process group is gloo (the one-device multi-process check)."""
    op = op if op is not None else dist.ReduceOp.SUM
    if dist.get_backend() == "gloo":
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)


def ncu_traffic(config_name: str, math: str, kernel_hash: str):
    """DRAM bytes per launch of the hot kernel from the committed ncu capture
    (profiles/ncu_traffic.json), only when it was measured on this kernel
    build (same kernel_hash, see paper_1507_06565_b200/build.py) and math mode."""
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        e = json.loads(f.read_text()).get(f"{config_name}|{math}")
        if e is None or e.get("kernel_hash") != kernel_hash:
            return None
        return float(e["dram_bytes_per_launch"])
    except Exception:  # noqa: BLE001
        return None


def config_dict(name, fluid, cells, links, scheme, world, meta, slab=None):
    """The `config` of the JSON line, identical in both arms."""
    slab = world > 1 if slab is None else slab
    return {"workload": name, "fluid_cells": int(fluid), "cells": int(cells),
            "links": int(links), "scheme": scheme,
            "l2": "inputs larger than L2 (2 x 19 x cells x 8 B > 126 MB)"
            if 2 * 19 * 8 * cells > 126e6 else "state L2-resident",
            "parallelism": f"x-slab{world}" if slab else "single", **meta}


# ---------------------------------------------------------------------------
# CPU reference timing (oracle/_ref: the reference compiled from its sources)
# ---------------------------------------------------------------------------
def reference_cpu_sample(sim, fluid_cells: int, budget_s: float, warmup: int = 3,
                         max_steps: int = 1_000_000):
    """The one sampler of both CPU legs: `warmup` (>= 3) untimed steps of the
    reference Simulation::step(), then steps timed one by one until ~budget_s
    (at most max_steps); the rate is taken at the MEDIAN step time, so a
    transient disturbance of the shared host does not move either leg.
    Returns (fluid MLUPS, steps, seconds, warmup)."""
    w = max(3, int(warmup))
    sim.step(w)
    times = []
    t_start = time.perf_counter()
    while len(times) < max(1, int(max_steps)):
        t0 = time.perf_counter()
        sim.step(1)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start >= budget_s:
            break
    med = statistics.median(times)
    return fluid_cells / med / 1e6, len(times), sum(times), w


def cpu_sample_text(name, n, w, dt, threads):
    return (f"{name}: {n} time steps of the reference Simulation::step() (timed one by one; oracle/_ref, OpenMP "
            f"{threads} threads = physical cores, OMP_PLACES=cores OMP_PROC_BIND=close) after "
            f"{w} warm-up steps, {dt:.1f} s; rate at the median step time)")


def run_reference_arm(args):
    """The reference CPU solver on the same workload, built and run with
    oracle code only (oracle/ref_workloads.py: harness spheres, the oracle
    voxelizer checked against the reference-made golden geometry, and the
    reference Simulation from oracle/_ref).  The product library is never
    loaded in this process."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import ref_workloads
    from oracle.oracle import RefLib

    w, geom, meta = ref_workloads.build(args.config)
    checked = meta.pop("geometry_checked", None)
    ref = RefLib()
    threads = ref.set_threads(CPU_THREADS)
    sim = ref_workloads.reference_simulation(ref, w, geom)
    mlups, n, dt, wu = reference_cpu_sample(sim, geom.fluid_cells, args.ref_budget,
                                            min(max(args.warmup, 3), 10), args.steps)
    line = {
        "metric": "D3Q19 TRT fp64 fluid MLUPS", "value": mlups, "unit": "MLUPS",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / n * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(w.name, geom.fluid_cells, geom.cells, geom.n_links, w.scheme, 1,
                              meta),
        "cpu_baseline": {"value": mlups, "unit": "MLUPS", "cores": threads, "kind": "reference",
                         "sample": cpu_sample_text(w.name, n, wu, dt, threads)
                         + f" (of the requested {args.steps}, capped at ~{args.ref_budget:.0f} s)"},
        "e2e": {"value": mlups, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "geometry": checked,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # NCCL on high-priority streams: the 5-PDF halo send/recv kernels are
        # scheduled ahead of the interior sweep's pending blocks, so the
        # exchange overlaps the interior instead of queueing behind it
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        if os.environ.get("PGPU_BENCH_BACKEND") == "gloo":  # test knob (with PGPU_BENCH_ONE_DEVICE)
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
    import paper_1507_06565_b200 as pg
    from paper_1507_06565_b200 import configs

    if world > 1 or args.force_slab:
        from paper_1507_06565_b200.dist import SlabSimulation

        w = configs.c4(nx_scale=world) if (args.config == "C4" and args.scaling == "weak") \
            else configs.ALL[args.config]()
        sim_obj = SlabSimulation(w, rank, world, device=local, transport=args.transport)
        halo_transport = sim_obj.transport  # "ipc", or "nccl" (also the fallback)
        sim = sim_obj.sim
        fluid_local = sim.fluid_cells
        stepper = sim_obj.step
        geom = None
    else:
        w = configs.ALL[args.config]()
        if args.scheme:
            w.scheme = pg.WallScheme[args.scheme]
            w.name += f"_{args.scheme.lower()}_override"
        geom = w.geometry()
        sim = configs.make_simulation(w, geom, device=local)
        fluid_local = geom.fluid_cells
        stepper = sim.step
    if world > 1 or args.force_slab:
        stream = sim_obj.me.stream
    else:
        stream = torch.cuda.Stream(device=local)
        sim.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        stepper(args.warmup)
        if not (world > 1 or args.force_slab):
            sim.prepare()  # the step's CUDA graphs exist before the timed region (no steps taken)
    torch.cuda.synchronize()
    fluid_total = fluid_local
    links_local = geom.n_links if geom is not None else sim_obj.me.geometry.n_links
    links_total = links_local
    if dist is not None:
        t = torch.tensor([fluid_local, links_local], dtype=torch.float64, device="cuda")
        all_reduce(dist, t)
        fluid_total, links_total = int(t[0].item()), int(t[1].item())
        dist.barrier()

    device_bytes = sim.device_bytes
    sweep_kernel = getattr(sim, "sweep_kernel", None)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = sim.launch_count
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks.mark()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        stepper(args.steps)
        ev1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = sim.launch_count - launches0
    clk = clocks.stop()
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        all_reduce(dist, t, dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = fluid_total * args.steps / (ms * 1e-3) / 1e6

    # roofline of the hot kernel (one K1 launch per step, timed on its stream)
    peak, peak_src = hbm_peak()
    bytes_per_launch = BYTES_PER_FLUID_CELL * fluid_local
    achieved = bytes_per_launch / (ms_per_step * 1e-3) / 1e9
    khash = pg.build_info().get("kernel_hash", "unknown")
    traffic = ncu_traffic(w.name, args.math, khash) if world == 1 else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": bytes_per_launch, "kernel_hash": khash}

    # e2e through the public API with host buffers.  The device-resident
    # simulation stays alive meanwhile (52 GB of 180 GB on C4): reallocating
    # the 26 GB it would free right away made cudaMalloc take up to 0.7 s in
    # some runs (tools/e2e_probe.py), a driver effect unrelated to the path.
    parity = None
    if (world > 1 or args.force_slab) and args.verify:
        parity = verify_slabs(w, sim_obj, args.warmup + args.steps, rank, world, local, dist,
                              args.scaling)

    e2e = None
    if world == 1 and not args.no_e2e and not args.force_slab:
        e2e = e2e_run(pg, configs, w, geom, args.steps, local, args.e2e_output)
    elif (world > 1 or args.force_slab) and not args.no_e2e:
        slab_geom = sim_obj.me.geometry
        e2e = e2e_run_dist(w, slab_geom, args.steps, rank, world, local, dist, halo_transport)
    del sim, stepper
    if world > 1 or args.force_slab:
        del sim_obj
    torch.cuda.empty_cache()

    per_config = None
    if rank == 0 and world == 1 and not args.force_slab and not args.no_per_config:
        per_config = per_config_run(pg, configs, args.config, local, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.force_slab:
        try:
            from oracle.oracle import RefLib

            ref = RefLib()
            threads = ref.set_threads(CPU_THREADS)
            p = w.params()
            rsim = ref.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.lambda_magic,
                                  p.body_force, int(w.scheme))
            gp = w.glbm_params()
            if gp is not None:
                rsim.set_porous(gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus, 0.0, True)
            mlups, n, dt, wu = reference_cpu_sample(rsim, geom.fluid_cells, args.cpu_budget)
            del rsim
            cpu = {"value": mlups, "unit": "MLUPS", "cores": threads, "kind": "reference",
                   "sample": cpu_sample_text(w.name, n, wu, dt, threads)}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "MLUPS", "cores": CPU_THREADS, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": "D3Q19 TRT fp64 fluid MLUPS", "value": value, "unit": "MLUPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_dict(w.name, fluid_total, int(np.prod(w.dims)) if world == 1
                                  else int(np.prod(w.dims)), links_total, w.scheme.name,
                                  world, w.meta, slab=world > 1 or args.force_slab),
            "math": args.math,
            "sweep_kernel": sweep_kernel,
            "device_bytes_per_gpu": device_bytes,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "total_cell_mlups": int(np.prod(w.dims)) * args.steps / (ms * 1e-3) / 1e6,
            "per_config": per_config,
        }
        if world > 1 or args.force_slab:
            line["halo_transport"] = halo_transport
        if parity is not None:
            line["parity"] = parity
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def verify_slabs(w, sim_obj, total_steps, rank, world, device, dist, scaling):
    """--verify: after the timed region every rank hashes its slab's fluid
    populations f(n); rank 0 reruns the whole domain single-GPU for the same
    number of steps and hashes the same column ranges.  parity_ok = every
    slab bit-identical (strong scaling: the global domain fits one GPU)."""
    import hashlib

    import torch

    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import slab_ranges

    def fluid_hash(pdfs, flags):
        return hashlib.sha256(np.ascontiguousarray(pdfs[:, flags == 0]).tobytes()).hexdigest()

    g = sim_obj.me.geometry
    mine = fluid_hash(sim_obj.sim.get_pdfs(), g.flags.reshape(g.dims[::-1]))
    hashes = [None] * world
    if dist is not None:
        dist.all_gather_object(hashes, mine)
    else:
        hashes = [mine]
    if rank != 0:
        return None
    if scaling != "strong" and world > 1:
        return {"parity_ok": None, "why": "weak scaling: the global domain does not fit one GPU",
                "slab_sha256": hashes}
    full = w.geometry()
    sim = configs.make_simulation(w, full, device=device)
    sim.step(total_steps)
    f = sim.get_pdfs()
    del sim
    torch.cuda.empty_cache()
    flags = full.flags.reshape(w.dims[::-1])
    ok = []
    for r, (x0, x1) in enumerate(slab_ranges(w.dims[0], world)):
        ok.append(fluid_hash(np.ascontiguousarray(f[..., x0:x1]), flags[..., x0:x1]) == hashes[r])
    return {"parity_ok": all(ok), "steps": total_steps, "slabs_equal": ok,
            "what": "sha256 of every slab's fluid f(n) vs the single-GPU run of the same steps"}


def per_config_run(pg, configs, skip, device, peak):
    """The other BASELINE configs timed in the same process (fluid MLUPS and
    the 304-B roofline fraction of their hot kernel), each a device-resident
    run of >= 200 steps (>= ~0.2 s) after 20 warm-up steps."""
    import torch

    out = {}
    for key in ("C1", "C2", "C3", "C4", "C5"):
        if key == skip:
            continue
        if key == "C4":
            continue  # the headline workload (or too large to add to it)
        w = configs.ALL[key]()
        geom = w.geometry()
        sim = configs.make_simulation(w, geom, device=device)
        stream = torch.cuda.Stream(device=device)
        sim.set_stream(stream.cuda_stream)
        sim.step(20)
        sim.prepare()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 200
        while True:
            e0.record(stream)
            sim.step(steps)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if ms > 150.0 or steps >= 20000:
                break
            steps *= 4
        mlups = geom.fluid_cells * steps / (ms * 1e-3) / 1e6
        gbs = BYTES_PER_FLUID_CELL * geom.fluid_cells * steps / (ms * 1e-3) / 1e9
        out[key] = {"workload": w.name, "value": mlups, "unit": "MLUPS", "steps": steps,
                    "ms_per_step": ms / steps, "frac": gbs / peak,
                    "layout": sim.layout, "sweep_kernel": sim.sweep_kernel,
                    "fluid_cells": geom.fluid_cells}
        del sim
    return out


def pinned_geometry(geom):
    """The geometry with its arrays in pinned (page-locked) host memory: the
    e2e leg's inputs come from pinned buffers the caller prepared (untimed),
    so pgpu_create DMAs them directly instead of staging pageable memory."""
    import dataclasses

    import torch

    def pin(a):
        if a is None:
            return None
        t = torch.empty(a.shape, dtype=getattr(torch, a.dtype.name), pin_memory=True)
        out = t.numpy()
        out[...] = a
        return out

    names = ("flags", "link_fluid_cell", "link_second_fluid", "link_direction", "link_q",
             "link_moving", "porosity", "ghost_flags_lo", "ghost_flags_hi")
    return dataclasses.replace(geom, **{n: pin(getattr(geom, n)) for n in names})


def e2e_run(pg, configs, w, geom, steps, device, output="fields"):
    """Timed: create from host geometry (H2D) + steps + the result back (D2H):
    the macroscopic density and velocity fields (the API's field output,
    simulation.hpp macroscopic(); `output="pdfs"`: all of f(N)) into pinned
    memory, and the planar profile."""
    import torch

    cells = geom.cells
    shape = geom.dims[::-1]
    if output == "pdfs":
        host = torch.empty(19 * cells, dtype=torch.float64, pin_memory=True).numpy()
    else:
        host = torch.empty(4 * cells, dtype=torch.float64, pin_memory=True).numpy()
    h2d = (geom.flags.nbytes + geom.n_links * (8 + 8 + 4 + 4 + 1) + geom.porosity.nbytes)
    geom = pinned_geometry(geom)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim = configs.make_simulation(w, geom, device=device)
    tc = time.perf_counter()
    sim.step(steps)
    if output == "pdfs":
        sim.get_pdfs(host.reshape(19, *shape))
    else:
        sim.macroscopic_fields(out=[host[i * cells:(i + 1) * cells].reshape(shape) for i in range(4)])
    td = time.perf_counter()
    prof = sim.planar_profile()
    t1 = time.perf_counter()
    d2h = host.nbytes + 5 * prof.z.nbytes
    del sim
    torch.cuda.empty_cache()
    what = ("pgpu_get_pdfs (pinned)" if output == "pdfs"
            else "pgpu_macroscopic_fields (delta_rho, u; pinned)")
    return {"value": geom.fluid_cells * steps / (t1 - t0) / 1e6, "unit": "MLUPS",
            "h2d_bytes_per_step": h2d / steps, "d2h_bytes_per_step": d2h / steps,
            "seconds": t1 - t0, "create_s": tc - t0, "steps_and_result_s": td - tc,
            "profile_s": t1 - td, "output": output,
            "what": f"pgpu_create from host geometry + K steps + {what} + pgpu_planar_profile"}


def e2e_run_dist(w, geom, steps, rank, world, device, dist, transport="nccl"):
    """N > 1: every rank creates its slab from its host slab geometry, steps
    through DistTransport (NCCL halo), downloads its f(N) into pinned memory
    and joins the global profile; time = max over ranks."""
    import torch

    from paper_1507_06565_b200.dist import SlabSimulation

    cells = geom.cells
    shape = geom.dims[::-1]
    host = torch.empty(4 * cells, dtype=torch.float64, pin_memory=True).numpy()
    h2d = (geom.flags.nbytes + geom.n_links * (8 + 8 + 4 + 4 + 1) + geom.porosity.nbytes
           + 2 * geom.ghost_flags_lo.nbytes)
    geom = pinned_geometry(geom)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    ss = SlabSimulation(w, rank, world, device=device, geometry=geom, transport=transport)
    tc = time.perf_counter()
    ss.step(steps)
    ss.sim.macroscopic_fields(out=[host[i * cells:(i + 1) * cells].reshape(shape) for i in range(4)])
    td = time.perf_counter()
    prof = ss.planar_profile()
    t1 = time.perf_counter()
    loc = torch.tensor([t1 - t0, tc - t0, td - tc, t1 - td], dtype=torch.float64, device="cuda")
    fl = torch.tensor([float(ss.sim.fluid_cells)], dtype=torch.float64, device="cuda")
    if dist is not None:
        all_reduce(dist, loc, dist.ReduceOp.MAX)
        all_reduce(dist, fl)
    tt, tcr, tst, tpr = (float(v) for v in loc.cpu())
    d2h = host.nbytes + 5 * prof.z.nbytes
    del ss
    torch.cuda.empty_cache()
    return {"value": float(fl.item()) * steps / tt / 1e6, "unit": "MLUPS",
            "h2d_bytes_per_step": world * h2d / steps, "d2h_bytes_per_step": world * d2h / steps,
            "seconds": tt, "create_s": tcr, "steps_and_result_s": tst, "profile_s": tpr,
            "output": "fields",
            "what": "per rank: pgpu_create from its host slab geometry + K steps with the NCCL "
                    "halo + pgpu_macroscopic_fields of its slab (pinned) + global planar "
                    "profile; max over ranks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--scheme", default=None, choices=["SBB", "CLI"],
                    help="override the config's wall scheme (experiments only)")
    ap.add_argument("--math", default="fast", choices=["fast", "exact"],
                    help="pgpu_math_mode: fast = FMA-contracted collision "
                         "(<= 1e-12 vs the reference, tests/test_gpu_fast.py); exact = "
                         "bit-identical to the reference")
    ap.add_argument("--cpu-budget", type=float, default=15.0,
                    help="seconds of reference steps in the cpu_baseline leg (after 3 warm-ups)")
    ap.add_argument("--ref-budget", type=float, default=20.0,
                    help="seconds of reference steps per --impl reference run (after >= 3 warm-ups)")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--verify", action="store_true",
                    help="N>1 / --force-slab: check the slabs' f(n) bitwise against a "
                         "single-GPU run of the same steps (strong scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="N > 1 halo exchange: NCCL send/recv, or IPC (the edge kernel stores "
                         "the 5 PDFs per face straight into the neighbours' ghost buffers)")
    ap.add_argument("--e2e-output", default="fields", choices=["fields", "pdfs"],
                    help="the result read back in the e2e leg: the macroscopic density/velocity "
                         "fields (default) or all of f(N)")
    ap.add_argument("--force-slab", action="store_true",
                    help="diagnostic: run the multi-GPU slab path (edge/interior split, halo "
                         "exchange) even at N=1")
    args = ap.parse_args()
    os.environ["PGPU_MATH"] = args.math  # read by pgpu_create
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
