mkdir -p gpurun_out
PGPU_LIB=paper_1507_06565_b200/_variants/cw16/libporolb_cuda.so timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_compact.py -q -x > gpurun_out/t23.log 2>&1; echo rc=$? >> gpurun_out/t23.log; tail -2 gpurun_out/t23.log
bash tools/ab_bench.sh "C4 C2" cw16 2>&1 | tee gpurun_out/ab23.log
for v in product cw16; do if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi; for r in 1 2; do python bench.py --scheme SBB --steps 200 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"C4-SBB $v\", round(d[\"value\"]))"; done; done
