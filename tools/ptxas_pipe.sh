#!/bin/bash
# Register / spill summary of every k_sweep_pipe instantiation (ptxas -v).
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xptxas -v -c paper_1507_06565_b200/csrc/kernels.cu -o /tmp/k.o "$@" 2>&1 |
python3 -c '
import re, sys
name = None
for line in sys.stdin:
    m = re.search(r"Function properties for (\S+)", line)
    if m: name = m.group(1); continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and name and "k_sweep_pipe" in name:
        t = re.search(r"pipeILb(\d)ELb(\d)ELb(\d)ELb(\d)ELi(\d)", name).groups()
        print("RHO1=%s GLBM=%s REC=%s SLAB=%s OP=%s" % t, "stack", m.group(1), "spill", m.group(2))
'
