mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_setup.py tests/test_gpu_compact.py tests/test_gpu_configs.py -q -x > gpurun_out/t4.log 2>&1; echo rc=$? >> gpurun_out/t4.log; tail -2 gpurun_out/t4.log
PGPU_TRACE=1 timeout 600 python tools/e2e_probe.py compact 2>&1 | grep -E "rep|upload"
timeout 300 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
