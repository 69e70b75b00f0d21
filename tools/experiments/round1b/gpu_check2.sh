mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_compact.py -q -x > gpurun_out/gpu_tests2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests2.log
tail -3 gpurun_out/gpu_tests2.log
bash tools/ab_bench.sh "C4" nocs 2>&1 | tee gpurun_out/ab_nocs.log
for l in compact dense; do PGPU_LAYOUT=$l timeout 300 python bench.py --force-slab --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("force-slab '$l'", round(d["value"]), round(d["roofline"]["frac"],3))'; done
