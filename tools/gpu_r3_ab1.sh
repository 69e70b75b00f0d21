# session 3: per-config A/B of sweep kernels / schedules (no cpu baseline, no e2e)
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('C4', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], {k: (round(v['value']), round(v['frac'],3)) for k,v in d['per_config'].items()})"; }
run X=1
run PGPU_SWEEP=tma
run PGPU_ZPER=2
run PGPU_ZPER=4
run X=1
