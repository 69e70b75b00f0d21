"""Top stalled SASS instructions of an ncu report (needs --import-source / -lineinfo)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ia, iw = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iw]), i, r[ia].strip()) for i, r in enumerate(rows[2:]) if len(r) > iw and r[iw].isdigit()]
tot = sum(d[0] for d in data)
for s, i, src in sorted(data, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% [{i:4d}] {src[:100]}")
