mkdir -p gpurun_out
bash tools/ab_bench.sh "C4" pol1 pol2 2>&1 | tee gpurun_out/ab24.log
for v in product pol1; do if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi; for r in 1 2; do python bench.py --scheme SBB --steps 200 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"C4-SBB $v\", round(d[\"value\"]))"; done; done
