# quick parity (compact + parity + fast suites) and the per-config bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py tests/test_gpu_fast.py tests/test_gpu_tma.py -x -q -m "gpu and not slow" > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/qb.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/qb.json')); print('C4', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], {k: (round(v['value']), round(v['frac'],3)) for k,v in d['per_config'].items()})"
