#!/bin/bash
# A/B of environment settings per config: tools/ab_env.sh "C2 C5" "PGPU_LAYOUT=dense" "PGPU_LAYOUT=compact" ...
cfgs=$1; shift
for cfg in $cfgs; do
  for v in "$@"; do
    for rep in 1 2; do
      st=200; [ $cfg != C4 ] && st=2000
      r=$(env $v python bench.py --config $cfg --steps $st --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3))')
      echo "$cfg $v $r"
    done
  done
done
