# programmatic dependent launch of the whole-domain sweeps: parity + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py tests/test_gpu_fast.py tests/test_gpu_configs.py -x -q -m "gpu" > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pdl_tests.log
B="--steps 400 --warmup 20 --no-cpu-baseline --no-e2e --no-per-config"
for cfg in ${CFGS:-C2 C3 C4}; do
for v in 0 1 0 1; do
  st=400; [ $cfg = C4 ] && st=100
  PGPU_PDL=$v timeout 300 python bench.py --steps $st --warmup 20 --no-cpu-baseline --no-e2e --no-per-config --config $cfg > gpurun_out/pdl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pdl.json')); print('$cfg pdl=$v', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
