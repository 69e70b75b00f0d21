#!/bin/bash
# A/B of the product build against experiment variants (PGPU_LIB), per config.
# usage: tools/ab_bench.sh "C4 C3" variant1 variant2 ...
cfgs=$1; shift
for cfg in $cfgs; do
  for v in product "$@"; do
    if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi
    for rep in 1 2 3; do
      st=200; [ $cfg != C4 ] && st=2000
      r=$(python bench.py --config $cfg --steps $st --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))')
      echo "$cfg $v $r"
    done
  done
done
