mkdir -p gpurun_out
PGPU_LIB=paper_1507_06565_b200/_variants/cw2/libporolb_cuda.so timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_compact.py -q -x > gpurun_out/t22.log 2>&1; echo rc=$? >> gpurun_out/t22.log; tail -2 gpurun_out/t22.log
bash tools/ab_bench.sh "C4 C3 C2" cw2 2>&1 | tee gpurun_out/ab22.log
