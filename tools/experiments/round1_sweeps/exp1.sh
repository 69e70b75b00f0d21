# usage: bash tools/exp1.sh  -- env-var sweep of the sweep-kernel variants on C4
run() { local envs="$1"; shift; timeout 300 env $envs python bench.py "$@" --steps 60 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs $*', round(d['value']), 'MLUPS', round(d['roofline']['frac'],3), round(d['ms_per_step'],3),'ms')"; }
for sch in SBB CLI; do
 run "PGPU_SWEEP=plain PGPU_FILL_SECTORS=1" --scheme $sch
 run "PGPU_SWEEP=plain PGPU_FILL_SECTORS=0" --scheme $sch
 for zp in 4 16 64; do for fill in 1 0; do run "PGPU_SWEEP=pipe PGPU_ZPER=$zp PGPU_FILL_SECTORS=$fill" --scheme $sch; done; done
done
