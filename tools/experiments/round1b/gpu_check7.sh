mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compact.py -q -x > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log; tail -2 gpurun_out/t7.log
bash tools/ab_bench.sh "C4" lf 2>&1 | tee gpurun_out/ab18.log
