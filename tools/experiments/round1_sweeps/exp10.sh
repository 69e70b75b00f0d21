run() { local envs="$1"; shift; timeout 300 env $envs python bench.py "$@" --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs $*', round(d['value']), 'MLUPS', round(d['roofline']['frac'],3), round(d['ms_per_step'],3),'ms')"; }
V=paper_1507_06565_b200/_variants
run "X=1" --scheme CLI
run "PGPU_LIB=$V/pool192/libporolb_cuda.so" --scheme CLI
run "PGPU_LIB=$V/pool64/libporolb_cuda.so" --scheme CLI
run "X=1" --config C3
run "PGPU_LIB=$V/pool192/libporolb_cuda.so" --config C3
