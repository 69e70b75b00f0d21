# z-block order A/B on the CLI workloads (PGPU_ZREV alternation with heavy-first)
mkdir -p gpurun_out
for cfg in C3 C4; do
for v in 1 0 1 0; do
  st=400; [ $cfg = C4 ] && st=100
  PGPU_ZREV=$v timeout 300 python bench.py --steps $st --warmup 20 --no-cpu-baseline --no-e2e --no-per-config --config $cfg > gpurun_out/zo.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/zo.json')); print('$cfg zrev=$v', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
