mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
PGPU_LIB=paper_1507_06565_b200/_variants/bounds/libporolb_cuda.so timeout 1500 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_drivers.py -q -x > gpurun_out/t_bounds.log 2>&1; echo bounds rc=$? >> gpurun_out/t_bounds.log; tail -2 gpurun_out/t_bounds.log
bash tools/ab_bench.sh "C4 C3" base 2>&1 | tee gpurun_out/ab17.log
