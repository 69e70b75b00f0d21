mkdir -p gpurun_out
PGPU_LIB=paper_1507_06565_b200/_variants/ra/libporolb_cuda.so timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py -q -x -k "compact" > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log; tail -3 gpurun_out/t13.log
bash tools/ab_bench.sh "C4 C3" ra 2>&1 | tee gpurun_out/ab13.log
