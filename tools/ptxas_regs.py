"""Print registers/spills per kernel of csrc/kernels.cu (ptxas -v), demangled."""
import re, subprocess, sys
from pathlib import Path
src = Path(__file__).resolve().parent.parent / "paper_1507_06565_b200" / "csrc" / "kernels.cu"
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                      "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-c", str(src), "-o", "/tmp/_k.o"],
                     capture_output=True, text=True).stderr
cur = None
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["cu++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = m.group(0)
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        if pat in cur:
            print(f"{m2.group(1):>4} regs  {spill if 'spill' in locals() else ''}  {cur[:110]}")
        cur = None
