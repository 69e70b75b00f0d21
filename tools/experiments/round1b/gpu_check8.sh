mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/ab_bench.sh "C4" base 2>&1 | tee gpurun_out/ab19.log
