#!/bin/bash
# Units sweep (k_sweep_units) on one B200: parity tests, then A/B against the
# chunk sweep per config and units-per-warp setting.  Output: gpurun_out/units_ab.txt
mkdir -p gpurun_out
OUT=gpurun_out/units_ab.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_units.py -x -q > gpurun_out/units_tests.log 2>&1
echo "units tests rc=$?" >> $OUT
tail -3 gpurun_out/units_tests.log >> $OUT
B="--no-per-config --no-cpu-baseline --no-e2e --steps 100 --warmup 5"
run() {  # cfg kernel upw
  PGPU_SWEEP=$2 PGPU_UPW=$3 timeout 300 python bench.py $B --config $1 > gpurun_out/u_tmp.json 2> gpurun_out/u_tmp.err
  rc=$?
  python - "$1" "$2" "$3" $rc >> $OUT <<'PY'
import json, sys
cfg, k, upw, rc = sys.argv[1:5]
try:
    d = json.loads(open('gpurun_out/u_tmp.json').read().strip().splitlines()[-1])
    print(cfg, k, 'upw=' + upw, round(d['value']), round(d['roofline']['frac'], 4), d['clocks']['sm_mhz'], d.get('sweep_kernel'))
except Exception as e:
    print(cfg, k, upw, 'rc=' + rc, 'failed', e)
PY
}
for cfg in ${CFGS:-C4 C3 C2}; do
  run $cfg cpipe 0
  for upw in ${UPWS:-0 4 8 16 32}; do run $cfg units $upw; done
done
cat $OUT
