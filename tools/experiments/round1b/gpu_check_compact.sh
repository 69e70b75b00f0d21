# Compact-layout check on one B200: smoke, C4 bench (CLI + SBB, compact vs dense), GPU suite forced compact.
mkdir -p gpurun_out
export PGPU_LAYOUT=compact
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_compact.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_compact.log
tail -2 gpurun_out/smoke_compact.log
unset PGPU_LAYOUT
for sch in CLI SBB; do
  timeout 300 python bench.py --scheme $sch --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("compact", d["config"]["scheme"], round(d["value"]), round(d["roofline"]["frac"],3), d["ms_per_step"])'
  PGPU_LAYOUT=dense timeout 300 python bench.py --scheme $sch --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("dense", d["config"]["scheme"], round(d["value"]), round(d["roofline"]["frac"],3), d["ms_per_step"])'
done
export PGPU_LAYOUT=compact
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_compact.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_compact.log
tail -15 gpurun_out/gpu_tests_compact.log
