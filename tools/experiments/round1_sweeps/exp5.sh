run() { local envs="$1"; shift; timeout 300 env $envs python bench.py "$@" --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs $*', round(d['value']), 'MLUPS', round(d['roofline']['frac'],3), round(d['ms_per_step'],3),'ms')"; }
run "X=1" --scheme CLI
run "X=1" --scheme SBB
run "PGPU_ZPER=8" --scheme CLI
for cfg in C2 C3 C5; do run "X=1" --config $cfg; done
