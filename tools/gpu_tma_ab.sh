# TMA sweep: parity tests, then A/B against the cpipe sweep (C4 CLI + per-config), variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tma.py -x -q > gpurun_out/tma_tests.log 2>&1; echo "tma tests rc=$?"; tail -3 gpurun_out/tma_tests.log
B="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e"
run() {  # label env...
  local l=$1; shift
  env "$@" timeout 300 python bench.py $B > gpurun_out/ab_$l.json 2> gpurun_out/ab_$l.err; echo "$l rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/ab_$l.json')); print('$l', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], {k: (round(v['value']), round(v['frac'],3)) for k,v in d.get('per_config',{}).items()})" 2>&1 | tail -1
}
run cpipe PGPU_SWEEP=cpipe
run tma PGPU_SWEEP=tma



