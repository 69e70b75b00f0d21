run() { local envs="$1"; shift; timeout 300 env $envs python bench.py "$@" --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs $*', round(d['value']), 'MLUPS', round(d['roofline']['frac'],3), round(d['ms_per_step'],3),'ms')"; }
V=paper_1507_06565_b200/_variants
for v in base stage1 stage1m5 stage2m5 stage1p192; do
  L=""; [ $v != base ] && L="PGPU_LIB=$V/$v/libporolb_cuda.so"
  for zp in 4 8; do run "$L PGPU_ZPER=$zp" --scheme CLI; done
  run "$L PGPU_ZPER=8" --scheme SBB
done
