"""Producer / link-warp / consumer split of an ncu source-page CSV of
k_sweep_tma (stall samples and executed instructions per source line).
usage: tma_prof_summary.py SRC_CSV RAW_CSV"""
import csv
import sys

src = open("paper_1507_06565_b200/csrc/sweep_tma.cu").read().split("\n")
mark = {name: [i + 1 for i, l in enumerate(src) if name in l and "----" in l][0]
        for name in ("producers", "link warp", "consumers")}
rows = list(csv.reader(open(sys.argv[1])))
hdr = path = cur = None
seen = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 7 and r[0].isdigit() and r[2] == "-":
        cur = (path, int(r[0]), r[1].strip()[:64])
        continue
    if hdr and len(r) > 7 and r[2].startswith("0x"):
        a = int(r[2], 16)
        if a in seen:
            continue
        d = dict(zip(hdr, r))
        seen[a] = (int(r[4]), int(r[7]), cur,
                   {k[6:]: float(d[k] or 0) for k in hdr if k.startswith("stall_") and "Not" not in k})


def side(c):
    f, l, _ = c
    if f != "sweep_tma.cu":
        return "?"
    if mark["producers"] <= l < mark["link warp"]:
        return "P"
    if mark["link warp"] <= l < mark["consumers"]:
        return "L"
    if l >= mark["consumers"]:
        return "C"
    return "?"


agg = {}
for a, (smp, ins, c, st) in seen.items():
    key = (side(c),) + c
    g = agg.setdefault(key, [0, 0, {}])
    g[0] += smp
    g[1] += ins
    for k, x in st.items():
        g[2][k] = g[2].get(k, 0) + x
tot = sum(g[0] for g in agg.values())
n = int(sys.argv[3]) if len(sys.argv) > 3 else 14
for sd in "PLC?":
    items = [(k, g) for k, g in agg.items() if k[0] == sd]
    s = sum(g[0] for _, g in items)
    i = sum(g[1] for _, g in items)
    print(f"{sd}: samples {100 * s / tot:.1f}%  instructions {i}")
    for k, g in sorted(items, key=lambda kg: -kg[1][0])[:n]:
        top = sorted(g[2].items(), key=lambda kv: -kv[1])[:2]
        print(f"   {100 * g[0] / tot:5.1f}% {g[1]:>11}  {k[1]}:{k[2]} {k[3]}  {[(a, round(b)) for a, b in top]}")
rows = list(csv.reader(open(sys.argv[2])))
h, u, r = rows[0], rows[1], rows[2]
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__t_sector_op_read_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread"]:
    if k in h:
        print(k, r[h.index(k)], u[h.index(k)])
