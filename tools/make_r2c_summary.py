"""profiles/r02c_ncu_summary.md + profiles/ncu_traffic.json + the launch list from the files
tools/gpu_final_r2c.sh left in gpurun_out/ (run from the repo root after the gpurun call)."""
import ast
import collections
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

G = Path("gpurun_out")
khash = ast.literal_eval((G / "r02c_build_info.txt").read_text())["kernel_hash"]
tables = subprocess.run([sys.executable, "tools/ncu_csv_summary.py", str(G), khash, "--prefix", "r02c",
                         "--traffic-json", "profiles/ncu_traffic.json"],
                        capture_output=True, text=True, check=True).stdout.rstrip() + "\n"
shutil.copy(G / "r02c_launches_c4.csv", "profiles/r02c_launches_bench_c4.csv")


def row(name):
    for ln in tables.splitlines():
        if ln.startswith(f"| {name} |"):
            c = [x.strip() for x in ln.strip("|").split("|")]
            return {"ms": float(c[2]), "ratio": float(c[4]), "dram_pct": re.search(r"\(([\d.]+) %\)", c[5]).group(1),
                    "frac": re.search(r"\*\*([\d.]+)\*\*", c[6]).group(1)}
    raise KeyError(name)


def bench(name):
    return json.loads((G / name).read_text().strip().splitlines()[-1])


b, bs, br = bench("r02c_bench.json"), bench("r02c_bench_slab.json"), bench("r02c_bench_ref.json")
pc = b["per_config"]
tests = re.findall(r"(\d+) passed", (G / "r02c_gpu_tests.log").read_text())[-1]

rows = list(csv.reader(open(G / "r02c_launches_c4.csv")))
h = next(i for i, x in enumerate(rows) if x and x[0] == "ID")
hdr = rows[h]
iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for x in rows[h + 1:]:
    if len(x) <= iV:
        continue
    ms = float(x[iV].replace(",", "")) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3,
                                          "ms": 1.0, "msecond": 1.0}[x[iU]]
    k = x[iK].split("(")[0].replace("void ", "").split("::")[-1][:40]
    agg[k][0] += 1
    agg[k][1] += ms
tot = sum(v[1] for v in agg.values())
k1 = next(v for k, v in agg.items() if k.startswith("k_sweep_units"))
k0 = next(v for k, v in agg.items() if k.startswith("k_collide_compact"))
rest_n = sum(v[0] for v in agg.values()) - k1[0] - k0[0]
rest = tot - k1[1] - k0[1]
det = ", ".join(f"`{k}` {v[1]:.2f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])
                if not k.startswith(("k_sweep_units", "k_collide_compact")) and v[1] >= 0.2)

c4, c4e, c4s, c2, c3, c5, c5d, cp = (row(n) for n in ("c4_cli_fast", "c4_cli_exact", "c4_sbb_fast", "c2_fast",
                                                     "c3_fast", "c5_fast", "c5_fast_dense",
                                                     "c4_cli_fast_cpipe"))
out = f"""# Round 2 (fourth session) — ncu captures of the final kernels per workload (B200, sm_100a)

Captured by `tools/gpu_r2c_profiles.sh` (inside `tools/gpu_final_r2c.sh`) on one B200 after the
same box ran the GPU suite ({tests} passed), `smoke()`, the default bench, the reference arm and the
slab-path bench: `ncu --set full --clock-control none --import-source on`, one launch after 3
warm-up launches of the same kernel (`bench.py --steps 3 --warmup 3`), exported on the box to CSV
and summarised by `tools/make_r2c_summary.py` (`tools/ncu_csv_summary.py --prefix r02c`).  Kernel
build `kernel_hash={khash}` (`pgpu_build_info`; `profiles/ncu_traffic.json` entries carry it,
and `bench.py` reports `roofline.traffic` only for that build).  Peak = this pool's measured copy
bandwidth, `MEASURED_PEAKS.json` `hbm_gbs` = 6558.7 GB/s.  ncu per-launch times are cold-cache and
serialised: the bench's CUDA-event times of back-to-back launches are the figures of record; the
share of the step is what must agree (launch list below).

What changed since `r02b_ncu_summary.md`: the hot kernel of the fluid-only layout is the **units
sweep** `k_sweep_units` (csrc/sweep_units.cu, DESIGN.md §6): warps sweep runs of up to 32
consecutive *fluid slots* instead of 32-cell chunks, so no lane idles on a solid cell of the
packing; and the fluid-only layout is the default for every domain that is not L2-resident (C5
too).  The chunk sweep `k_sweep_cpipe` (`c4_cli_fast_cpipe`, same box, `PGPU_SWEEP=cpipe`) is the
kernel the earlier summaries describe; `c5_fast_dense` is the dense layout's sweep on C5
(`PGPU_LAYOUT=dense`).

{tables}
Reading:

* **C4 CLI, math FAST (the bench workload): {c4['frac']} of the 304-B roofline per ncu** ({c4['ms']:.3f} ms per
  launch), DRAM at {c4['dram_pct']} % of the measured copy bandwidth, traffic {c4['ratio']:.3f}x the algorithmic bytes
  (CLI coefficients 8 B and descriptors 2 B per link, slot words 4 B per fluid cell, unit records).
  The driver-style bench run on the same box: {b['value']:,.0f} fluid MLUPS = **{b['roofline']['frac']:.4f}** (SM clock
  {b['clocks']['sm_mhz']:.0f} MHz, {', '.join(b['clocks']['reasons']) or 'no throttle reason'}), e2e {b['e2e']['value'] / 1e3:.1f} k.  The chunk sweep on the same
  box: {cp['frac']} per ncu ({cp['ms']:.3f} ms), DRAM at {cp['dram_pct']} %.  Bit-exact mode (EXACT): {c4e['frac']}.
* Why the units sweep is faster at (almost) the same instruction count per warp step: a unit
  carries 32 fluid cells, a warp-plane of the bed 16 -- per fluid cell the bed's warp instructions
  halve (thread instructions per fluid cell read *higher* because the idle lanes of the chunk
  sweep execute nothing and are not counted; the warp-level issue slots are what the SM spends),
  and each warp has a full 4.9 KB of copies in flight instead of ~2.4 KB in the bed.  Top stall is
  the wait for the unit's copies (long scoreboard): the sweep is memory-latency-bound at
  {c4['dram_pct']}-{c4s['dram_pct']} % of the copy bandwidth.
* SBB on the same bed: **{c4s['frac']}** (DRAM {c4s['dram_pct']} % of the copy bandwidth, traffic {c4s['ratio']:.3f}x).
* C2 / C3 (254 MB of state, twice L2, {1e3 * c2['ms']:.0f}-{1e3 * c3['ms']:.0f} us kernels): {c2['frac']} / {c3['frac']} per ncu -- a single
  serialised launch does not see what the bench's back-to-back launches gain from the alternating
  two-ended block order (each sweep starts on the planes the last one wrote) and from programmatic
  dependent launch: bench **{pc['C2']['frac']:.3f} / {pc['C3']['frac']:.3f}**.  Part of the traffic is served from L2
  ({c2['ratio']:.2f} / {c3['ratio']:.2f} of the algorithmic bytes reach DRAM).  C3's units in the bed average 27 fluid
  cells and 44 links; short-scoreboard stalls (the shared-memory chain of the link closures) weigh
  more there than on C4.
* C5 (GLBM channel, all fluid between two wall planes) on the fluid-only layout with the units
  sweep: **{c5['frac']}** per ncu ({pc['C5']['frac']:.3f} in the bench) against {c5d['frac']} of the dense layout's `k_sweep_pipe`
  -- contiguous 256-byte runs per direction, no per-cell solid tests.
* The x-slab path on the same box (`bench.py --force-slab --verify`, C4 as one slab, interior and
  edge bands on the units sweep, IPC transport): {bs['value']:,.0f} MLUPS = {bs['roofline']['frac']:.3f}, `parity_ok`
  {bs['parity']['parity_ok']}.  Reference arm (`bench.py --impl reference`, the reference's OpenMP solver on the box's
  {br['cpu_baseline']['cores']} cores): {br['value']:.1f} MLUPS; the `cpu_baseline` leg of the default bench: {b['cpu_baseline']['value']:.1f}.

Launch list of the default bench command (`profiles/r02c_launches_bench_c4.csv`, ncu
`gpu__time_duration.sum`, `bench.py --steps 3 --warmup 3`): the timed steps are only K1 launches.

| kernel | launches | ms (ncu, serialised) | share |
|---|---|---|---|
| `k_sweep_units<2,0,1,0>` (K1, C4 CLI fast) | {k1[0]} (2 warm-up + 3 timed) | {k1[1]:.3f} | {100 * k1[1] / tot:.1f} % |
| `k_collide_compact<2,0,0,0>` (K0, first step) | {k0[0]} | {k0[1]:.3f} | {100 * k0[1] / tot:.1f} % |
| setup ({det}, others) | {rest_n} | {rest:.2f} | {100 * rest / tot:.1f} % |
"""
Path("profiles/r02c_ncu_summary.md").write_text(out)
print(out[-1800:])
