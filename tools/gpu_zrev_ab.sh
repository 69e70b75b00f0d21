# z-order alternation + store policy A/B on the per-config workloads (C2, C3, C4)
mkdir -p gpurun_out
B="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-per-config"
for cfg in C2 C3; do
for v in "PGPU_ZREV=0 PGPU_STREAM_STORES=1" "PGPU_ZREV=0 PGPU_STREAM_STORES=0" "PGPU_ZREV=1 PGPU_STREAM_STORES=1" "PGPU_ZREV=1 PGPU_STREAM_STORES=0"; do
  env $v timeout 300 python bench.py $B --config $cfg > gpurun_out/zr.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/zr.json')); print('$cfg', '$v', round(d['value']), round(d['roofline']['frac'],3))"
done; done
for v in "PGPU_ZREV=0" "PGPU_ZREV=1"; do
  env $v timeout 300 python bench.py $B > gpurun_out/zr.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/zr.json')); print('C4', '$v', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
