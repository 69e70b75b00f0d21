"""Top stalled SASS instructions with their CUDA line and top stall reasons.
usage: ncu_sass.py REPORT [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, out, cur = None, [], None
for r in csv.reader(io.StringIO(txt)):
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[2] == "-":
        cur = r[0]
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    st = sorted(((int(r[k]), hdr[k][6:]) for k in range(len(hdr))
                 if hdr[k].startswith("stall_") and r[k].isdigit() and int(r[k]) > 0), reverse=True)[:3]
    out.append((s, cur, r[3], st))
tot = sum(o[0] for o in out) or 1
for s, l, t, st in sorted(out, key=lambda o: -o[0])[:n]:
    print(f"{100*s/tot:5.1f}% L{l:5s} {t[:58]:58s} {st}")
