mkdir -p gpurun_out
PGPU_LAYOUT=compact PGPU_LIB=paper_1507_06565_b200/_variants/bounds/libporolb_cuda.so timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log; tail -2 gpurun_out/t10.log
bash tools/ab_bench.sh "C4 C3 C2" base 2>&1 | tee gpurun_out/ab20.log
for v in product base; do
  if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi
  for rep in 1 2; do python bench.py --scheme SBB --steps 200 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("C4-SBB '$v'", round(d["value"]), round(d["roofline"]["frac"],3))'; done
done
