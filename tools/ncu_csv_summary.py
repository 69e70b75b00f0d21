"""Markdown summary of ncu --set full captures exported to CSV on the GPU box
(tools/gpu_r2_profiles.sh: <name>.raw.csv = --page raw, <name>.sass.csv =
--page source --print-source=sass), plus profiles/ncu_traffic.json entries
keyed by workload|math and the kernel build hash.

usage: ncu_csv_summary.py DIR KERNEL_HASH [--prefix r02] [--traffic-json profiles/ncu_traffic.json]
The peak is MEASURED_PEAKS.json's hbm_gbs when present.
"""
import csv
import io
import json
import re
import sys
from collections import defaultdict
from pathlib import Path

try:  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth, GB/s), driver-written per pool
    PEAK = float(json.loads(Path("MEASURED_PEAKS.json").read_text())["hbm_gbs"])
except Exception:  # noqa: BLE001
    PEAK = 6551.7
# name: (workload key of bench.py, math, fluid cells, warp-planes of the kernel)
RUNS = {
    "c4_cli_fast": ("C4_bed_512x256x512_cli", "fast", 51785984, 16 * 256 * 512),
    "c4_cli_exact": ("C4_bed_512x256x512_cli", "exact", 51785984, 16 * 256 * 512),
    "c4_sbb_fast": ("C4_bed_512x256x512_cli_sbb_override", "fast", 51785984, 16 * 256 * 512),
    "c2_fast": ("C2_bed_128x64x128_sbb", "fast", 834673, 4 * 64 * 128),
    "c3_fast": ("C3_bed_128x64x128_cli", "fast", 834673, 4 * 64 * 128),
    "c5_fast": ("C5_glbm_256x16x512", "fast", 2088960, 8 * 16 * 512),
    "c5_fast_dense": (None, "fast", 2088960, 8 * 16 * 512),
    # the chunk sweep on the headline workload, for comparison (not written to the traffic JSON)
    "c4_cli_fast_cpipe": (None, "fast", 51785984, 16 * 256 * 512),
}
GROUP = {"DADD": "fp64", "DMUL": "fp64", "DFMA": "fp64", "DSETP": "fp64",
         "LDGSTS": "LDGSTS", "LDG": "LDG", "STG": "STG", "LDS": "LDS", "STS": "STS",
         "LDC": "LDC/LDCU", "LDCU": "LDC/LDCU"}


def raw(path):
    rows = list(csv.reader(open(path)))
    h, u, r = rows[0], rows[1], rows[2]
    get = lambda k: (float(r[h.index(k)].replace(",", "")), u[h.index(k)])  # noqa: E731
    stalls = []
    for k, name in enumerate(h):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                stalls.append((float(r[k].replace(",", "")),
                               name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    return r[h.index("Kernel Name")], get, sorted(((100 * s / tot, n) for s, n in stalls),
                                                 reverse=True)


def sass(path):
    rows = list(csv.reader(open(path)))
    hdr = next(x for x in rows if x and x[0] == "Address")
    i_src, i_w = hdr.index("Source"), hdr.index("Instructions Executed")
    i_t = hdr.index("Predicated-On Thread Instructions Executed")
    warp, thr = defaultdict(float), defaultdict(float)
    for x in rows:
        if len(x) <= i_t or not x[0].startswith("0x"):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", x[i_src].strip())
        if not m:
            continue
        try:
            warp[m.group(2)] += float(x[i_w])
            thr[m.group(2)] += float(x[i_t])
        except ValueError:
            pass
    return warp, thr


def main():
    d = Path(sys.argv[1])
    khash = sys.argv[2]
    tj = Path(sys.argv[sys.argv.index("--traffic-json") + 1]) if "--traffic-json" in sys.argv else None
    pre = sys.argv[sys.argv.index("--prefix") + 1] if "--prefix" in sys.argv else "r02"
    out = ["| capture | kernel | time (ms) | DRAM read + write per launch | traffic / algorithmic |"
           f" DRAM GB/s (% of {PEAK:.0f}) | algorithmic GB/s = roofline frac | warps active | regs |"
           " top stalls |", "|---|---|---|---|---|---|---|---|---|---|"]
    hist = []
    traffic = json.loads(tj.read_text()) if tj and tj.exists() else {}
    for name, (wl, math, fluid, wplanes) in RUNS.items():
        rp = d / f"{pre}_{name}.raw.csv"
        if not rp.exists():
            continue
        kname, get, stalls = raw(rp)
        tv, tu = get("gpu__time_duration.sum")
        t_ms = tv * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[tu]
        scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
        rd = get("dram__bytes_read.sum")[0] * scale[get("dram__bytes_read.sum")[1]]  # GB
        wr = get("dram__bytes_write.sum")[0] * scale[get("dram__bytes_write.sum")[1]]
        alg = 304.0 * fluid / 1e9
        dram_gbs = (rd + wr) / (t_ms * 1e-3)
        alg_gbs = alg / (t_ms * 1e-3)
        warps = get("sm__warps_active.avg.pct_of_peak_sustained_active")[0]
        regs = int(get("launch__registers_per_thread")[0])
        k = re.sub(r"\(KParams.*", "", kname.replace("void unnamed>::", ""))
        st = ", ".join(f"{n} {p:.0f}%" for p, n in stalls[:3])
        out.append(f"| {name} | `{k}` | {t_ms:.4f} | {rd:.4f} + {wr:.4f} GB | {(rd + wr) / alg:.3f} |"
                   f" {dram_gbs:.0f} ({100 * dram_gbs / PEAK:.1f} %) | {alg_gbs:.0f} = **{alg_gbs / PEAK:.3f}** |"
                   f" {warps:.0f} % | {regs} | {st} |")
        if "k_sweep_units" in kname:  # warps sweep units (<= 32 fluid slots): 4 warps x 4 units per block
            wplanes = int(get("launch__grid_size")[0]) * 16
        per = "unit" if "k_sweep_units" in kname else "warp-plane"
        if wl is not None:
          traffic[f"{wl}|{math}"] = {
            "kernel": k, "kernel_hash": khash, "dram_bytes_per_launch": (rd + wr) * 1e9,
            "dram_read_bytes": rd * 1e9, "dram_write_bytes": wr * 1e9, "duration_ms_ncu": t_ms,
            "algorithmic_bytes_per_launch": 304 * fluid,
            "source": f"profiles/{pre}_ncu_summary.md (ncu --set full, 1 launch, {name})"}  # noqa: E126
        sp = d / f"{pre}_{name}.sass.csv"
        if sp.exists():
            warp, thr = sass(sp)
            tw = sum(warp.values())
            grp = defaultdict(float)
            for op, v in thr.items():
                grp[GROUP.get(op, "integer/control/other")] += v
            top = sorted(warp.items(), key=lambda kv: -kv[1])[:12]
            hist.append(f"**{name}** — {tw / wplanes:.0f} warp instructions per {per}; thread "
                        "instructions per fluid cell by group: " +
                        ", ".join(f"{g} {v / fluid:.1f}" for g, v in
                                  sorted(grp.items(), key=lambda kv: -kv[1])) +
                        f"  \n  top opcodes (warp instr / {per}): " +
                        ", ".join(f"{op} {v / wplanes:.1f}" for op, v in top) + "\n")
    print("\n".join(out))
    print("\n### SASS instruction histograms (executed, from the source page)\n")
    print("\n".join(hist))
    if tj:
        tj.write_text(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
