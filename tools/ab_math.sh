#!/bin/bash
# A/B of the math modes per config within one call: tools/ab_math.sh "C4 C3" [reps]
cfgs=$1; reps=${2:-2}
for cfg in $cfgs; do
  for m in exact fast; do
    for rep in $(seq $reps); do
      st=200; [ $cfg != C4 ] && st=2000
      r=$(python bench.py --config $cfg --steps $st --warmup 20 --no-cpu-baseline --no-e2e --math $m 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"] if d["clocks"] else None)')
      echo "$cfg $m $r"
    done
  done
done
