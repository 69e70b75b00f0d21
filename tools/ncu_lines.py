"""Stall samples and executed instructions per CUDA source line of an ncu report
(needs --import-source and -lineinfo).  usage: ncu_lines.py REPORT [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out, path = [], None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0].isdigit() and r[2] == "-":
        try:
            out.append((int(r[4]), int(r[7]), f"{path}:{r[0]}", r[1].strip()))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out) or 1
print(f"total samples {tot}, instructions {toti}")
for s, ins, loc, src in sorted(out, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% smp {100*ins/toti:5.1f}% ins  {loc:22s} {src[:90]}")
