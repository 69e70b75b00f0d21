mkdir -p gpurun_out
bash tools/ab_bench.sh "C5" d1s4 d2s3 2>&1 | tee gpurun_out/ab14.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
