# Final round numbers: per-config bench lines (product defaults), C4 bench JSON, slab path, reference arm.
mkdir -p gpurun_out
for c in C1 C2 C3 C5; do
  st=2000; timeout 600 python bench.py --config $c --steps $st --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$c'", round(d["value"]), round(d["roofline"]["frac"],3), d["ms_per_step"])'
done | tee gpurun_out/final_configs.log
timeout 300 python bench.py --scheme SBB --steps 200 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("C4-SBB", round(d["value"]), round(d["roofline"]["frac"],3))' | tee -a gpurun_out/final_configs.log
timeout 300 python bench.py --force-slab --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("C4-slab", round(d["value"]), round(d["roofline"]["frac"],3))' | tee -a gpurun_out/final_configs.log
timeout 300 python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err; cat gpurun_out/bench_final.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
