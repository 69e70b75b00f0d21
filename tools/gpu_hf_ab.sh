# boundary z-blocks first (PGPU_HEAVYFIRST) A/B
mkdir -p gpurun_out
for cfg in C3 C2 C4; do
for v in 0 1 0 1; do
  st=400; [ $cfg = C4 ] && st=100
  PGPU_HEAVYFIRST=$v timeout 300 python bench.py --steps $st --warmup 20 --no-cpu-baseline --no-e2e --no-per-config --config $cfg > gpurun_out/hf.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/hf.json')); print('$cfg hf=$v', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
