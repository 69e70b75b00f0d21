run() { local envs="$1"; shift; timeout 300 env $envs python bench.py "$@" --steps 60 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs $*', round(d['value']), 'MLUPS', round(d['roofline']['frac'],3), round(d['ms_per_step'],3),'ms')"; }
for sch in CLI SBB; do for zp in 2 4 16; do run "PGPU_ZPER=$zp" --scheme $sch; done; done
for cfg in C1 C2 C3 C5; do run "X=1" --config $cfg; done
