run() { local envs="$1"; shift; timeout 300 env $envs python bench.py "$@" --steps 60 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs $*', round(d['value']), 'MLUPS', round(d['roofline']['frac'],3), round(d['ms_per_step'],3),'ms')"; }
V=paper_1507_06565_b200/_variants
run "X=1" --scheme CLI
run "PGPU_LIB=$V/pool48/libporolb_cuda.so" --scheme CLI
run "PGPU_LIB=$V/pool192/libporolb_cuda.so" --scheme CLI
run "PGPU_ZPER=8" --scheme CLI
run "X=1" --scheme SBB
for cfg in C1 C2 C3 C5; do run "X=1" --config $cfg; done
