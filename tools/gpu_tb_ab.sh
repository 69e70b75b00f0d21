# two-step (temporal blocking) sweep vs the one-step cpipe sweep
mkdir -p gpurun_out
B="--steps 100 --warmup 6 --no-cpu-baseline --no-e2e --no-per-config"
for cfg in C4 C2 C3; do
for k in cpipe tb2; do
  PGPU_SWEEP=$k timeout 300 python bench.py $B --config $cfg > gpurun_out/tb_$k.json 2> gpurun_out/tb_$k.err; echo "$cfg $k rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/tb_$k.json')); print('$cfg $k', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['gpu_launches'])" 2>&1 | tail -1
done; done
