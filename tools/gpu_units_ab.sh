#!/bin/bash
# Units sweep (k_sweep_units) on one B200: parity tests, then A/B against the
# chunk sweep per config and units-per-warp setting.  Output: gpurun_out/units_ab.txt
mkdir -p gpurun_out
OUT=gpurun_out/units_ab.txt
: > $OUT
if [ -z "$NOTESTS" ]; then
timeout 900 python -m pytest tests/test_gpu_units.py -x -q > gpurun_out/units_tests.log 2>&1
echo "units tests rc=$?" >> $OUT
tail -3 gpurun_out/units_tests.log >> $OUT
fi
B="--no-per-config --no-cpu-baseline --no-e2e --steps 100 --warmup 5"
run() {  # cfg kernel upw
  PGPU_SWEEP=$2 PGPU_UPW=$3 timeout 300 python bench.py $B --config $1 > gpurun_out/u_tmp.json 2> gpurun_out/u_tmp.err
  rc=$?
  python - "$1" "$2" "$3" $rc >> $OUT <<'PY'
import json, sys
cfg, k, upw, rc = sys.argv[1:5]
try:
    d = json.loads(open('gpurun_out/u_tmp.json').read().strip().splitlines()[-1])
    import os
    print(cfg, k, 'upw=' + upw, 'group=' + os.environ.get('PGPU_UGROUP', '1'), round(d['value']), round(d['roofline']['frac'], 4), d['clocks']['sm_mhz'], d.get('sweep_kernel'))
except Exception as e:
    print(cfg, k, upw, 'rc=' + rc, 'failed', e)
PY
}
# VARS: variant builds (paper_1507_06565_b200/build.py --variant=...), "product" = the library
for cfg in ${CFGS:-C4 C3 C2}; do
  unset PGPU_LIB
  [ -z "$NOCPIPE" ] && run $cfg cpipe 0
  for v in ${VARS:-product}; do
    if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi
    echo "variant $v" >> $OUT
    for g in ${GROUPS_:-1}; do export PGPU_UGROUP=$g
    for upw in ${UPWS:-0 4 8 16 32}; do run $cfg units $upw; done; done
  done
done
cat $OUT
