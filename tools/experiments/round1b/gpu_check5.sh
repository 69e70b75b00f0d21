mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
for i in 1 2; do PGPU_TRACE=1 timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>&1 | grep -E "pgpu\] create (upload|alloc)|e2e" | sed "s/.*\"e2e\": \({[^}]*}\).*/\1/" | cut -c1-160; done
PGPU_TRACE=1 timeout 600 python tools/e2e_probe.py compact 2>&1 | grep -E "rep|alloc"
