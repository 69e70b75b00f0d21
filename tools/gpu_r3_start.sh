# session-3 start: confirm the rebuilt tree on a B200 (GPU suite, smoke, quick bench with per-config)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/qb.json 2>gpurun_out/qb.err; python -c "
import json; d=json.load(open('gpurun_out/qb.json')); print('C4', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], {k: (round(v['value']), round(v['frac'],3)) for k,v in d['per_config'].items()})"
