"""SASS instruction histogram of an ncu report's kernel (--set full with
--import-source): executed instructions per opcode, as warp instructions per
warp-plane and predicated-on thread instructions per fluid cell.
usage: ncu_sass_hist.py REPORT FLUID_CELLS WARP_PLANES [--md]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, fluid, wplanes = sys.argv[1], float(sys.argv[2]), float(sys.argv[3])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
name = rows[0][1] if rows and rows[0][0] == "Kernel Name" else "?"
hdr = next(r for r in rows if r and r[0] == "Address")
i_src, i_warp = hdr.index("Source"), hdr.index("Instructions Executed")
i_thr = hdr.index("Predicated-On Thread Instructions Executed")
warp, thr = defaultdict(float), defaultdict(float)
GROUP = {"DADD": "fp64", "DMUL": "fp64", "DFMA": "fp64", "DSETP": "fp64",
         "LDGSTS": "global->shared copy", "LDG": "global load", "STG": "global store",
         "LDS": "shared load", "STS": "shared store", "LDC": "constant load",
         "LDGDEPBAR": "copy commit/wait", "DEPBAR": "copy commit/wait"}
for r in rows:
    if len(r) <= i_thr or not r[0].startswith("0x"):
        continue
    src = r[i_src].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
    if not m:
        continue
    op = m.group(2)
    try:
        warp[op] += float(r[i_warp])
        thr[op] += float(r[i_thr])
    except ValueError:
        pass
tw, tt = sum(warp.values()), sum(thr.values())
md = "--md" in sys.argv
if md:
    print(f"kernel: `{name[:110]}`\n")
    print(f"total: {tw / wplanes:.0f} warp instructions per warp-plane, "
          f"{tt / fluid:.0f} thread instructions per fluid cell\n")
    print("| opcode | warp instr / warp-plane | thread instr / fluid cell | share |")
    print("|---|---|---|---|")
for op, v in sorted(warp.items(), key=lambda kv: -kv[1])[:28]:
    if md:
        print(f"| {op} | {v / wplanes:.1f} | {thr[op] / fluid:.1f} | {100 * v / tw:.1f} % |")
    else:
        print(f"{op:10s} {v / wplanes:8.1f} /warp-plane {thr[op] / fluid:8.1f} /fluid-cell "
              f"{100 * v / tw:5.1f} %")
grp = defaultdict(float)
for op, v in thr.items():
    grp[GROUP.get(op, "other")] += v
print("\ngroups (thread instr / fluid cell): " +
      ", ".join(f"{g} {v / fluid:.1f}" for g, v in sorted(grp.items(), key=lambda kv: -kv[1])))
