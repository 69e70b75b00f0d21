# session re-entry check: GPU suite + default bench on the rebuilt tree
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m "gpu" -x > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/gpu_tests.log | tail -8
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); print(round(d['value']), round(d['roofline']['frac'],3), d['device_bytes_per_gpu']/1e9, round(d['e2e']['value']), d['cpu_baseline']['value'], d['clocks'], {k: (round(v['value']), round(v['frac'],3)) for k,v in d['per_config'].items()})"
