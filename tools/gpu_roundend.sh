# What the driver runs at round end, in one call: GPU suite, smoke, default bench, reference arm.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_roundend.json 2>gpurun_out/bench_roundend.err; python -c "import json; d=json.load(open('gpurun_out/bench_roundend.json')); print(round(d['value']), round(d['roofline']['frac'],3), round(d['e2e']['value']), d['cpu_baseline']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_ref.json')); print('ref', round(d['value'],1), d['cpu_baseline']['cores'])"
