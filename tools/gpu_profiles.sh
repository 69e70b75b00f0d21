# A/B + profile capture of the product K1 (CLI bench workload and the SBB variant) on C4.
mkdir -p gpurun_out
bash tools/ab_bench.sh "C4" cp128 cp256 2>&1 | tee gpurun_out/ab5.log
for c in C2 C3 C5; do python bench.py --config $c --steps 2000 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$c'", round(d["value"]), round(d["roofline"]["frac"],3))'; done | tee gpurun_out/configs.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/k1_cli -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1_cli.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/k1_sbb -f python bench.py --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1_sbb.log 2>&1
tail -1 gpurun_out/ncu_k1_sbb.log
