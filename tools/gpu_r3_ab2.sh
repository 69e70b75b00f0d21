# session 3: zper wave target A/B + C4 CLI source-level ncu capture
mkdir -p gpurun_out /tmp/ncu
run() { echo "== $*"; env "$@" timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('C4', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], {k: (round(v['value']), round(v['frac'],3)) for k,v in d['per_config'].items()})"; }
run X=1
run PGPU_ZWAVES2=10
run PGPU_ZWAVES2=18
run PGPU_ZWAVES2=26
B="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o /tmp/ncu/r03_c4 -f python bench.py $B > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/ncu/r03_c4.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/r03_c4.src.csv 2>/dev/null
ncu -i /tmp/ncu/r03_c4.ncu-rep --page raw --csv > gpurun_out/r03_c4.raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o /tmp/ncu/r03_c3 -f python bench.py $B --config C3 > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/ncu/r03_c3.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/r03_c3.src.csv 2>/dev/null
ncu -i /tmp/ncu/r03_c3.ncu-rep --page raw --csv > gpurun_out/r03_c3.raw.csv 2>/dev/null
ls -la gpurun_out
