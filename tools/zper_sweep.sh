#!/bin/bash
# z-planes-per-block sweep of the K1 sweep on the small configs (device-resident metric).
for cfg in C2 C3 C5; do
  for z in 0 1 2 4 6 8; do
    if [ $z = 0 ]; then unset PGPU_ZPER; else export PGPU_ZPER=$z; fi
    v=$(python bench.py --config $cfg --steps 400 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))')
    echo "$cfg zper=$z $v"
  done
done
