#!/bin/bash
# A/B of variant builds per config and math mode: tools/ab_variants.sh "C4 C3" "fast" "product minb5" [reps] [extra bench args]
cfgs=$1; maths=$2; vars=$3; reps=${4:-2}; extra=$5
for cfg in $cfgs; do for m in $maths; do for rep in $(seq $reps); do for v in $vars; do
  if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi
  st=200; [ $cfg != C4 ] && st=2000
  r=$(python bench.py --config $cfg --steps $st --warmup 20 --no-cpu-baseline --no-e2e --math $m $extra 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"] if d["clocks"] else None)')
  echo "$cfg $m $v $r"
done; done; done; done
