mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log; tail -2 gpurun_out/t11.log
bash tools/ab_bench.sh "C4 C3" base 2>&1 | tee gpurun_out/ab11.log
