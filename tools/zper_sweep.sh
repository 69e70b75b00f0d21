#!/bin/bash
# z-planes-per-block sweep of the fluid-only K1 sweep (device-resident metric, math fast).
# usage: tools/zper_sweep.sh "C2 C3" "0 3 8 15 16 22 32"
cfgs=${1:-"C2 C3"}; zs=${2:-"0 3 8 15 16 22 32"}
for cfg in $cfgs; do
  for z in $zs; do
    if [ $z = 0 ]; then unset PGPU_ZPER; else export PGPU_ZPER=$z; fi
    st=2000; [ $cfg = C4 ] && st=200
    v=$(python bench.py --config $cfg --steps $st --warmup 20 --no-cpu-baseline --no-e2e --no-per-config 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"] if d["clocks"] else None)')
    echo "$cfg zper=$z $v"
  done
done
