mkdir -p gpurun_out
timeout 300 python tools/lid_probe.py > gpurun_out/lid_probe.log 2>&1; cat gpurun_out/lid_probe.log | tail -40
for cfg in C4 C3; do for rep in 1 2; do
  for v in "exact 1" "fast 1" "fast 0"; do set -- $v
    r=$(PGPU_FOLD=$2 python bench.py --config $cfg --steps $([ $cfg = C4 ] && echo 200 || echo 2000) --warmup 20 --no-cpu-baseline --no-e2e --math $1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"] if d["clocks"] else None)')
    echo "$cfg $1 fold=$2 $r"
  done
done; done
