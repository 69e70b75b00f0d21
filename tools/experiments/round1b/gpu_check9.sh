mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_compact.py -q -x > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log; tail -2 gpurun_out/t9.log
for v in product base; do
  if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi
  for rep in 1 2; do timeout 300 python bench.py --force-slab --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("slab '$v'", round(d["value"]), round(d["roofline"]["frac"],3))'; done
done
