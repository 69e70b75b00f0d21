# Final profile capture of the product K1 (CLI bench workload + SBB) and launch list on C4.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/k1_cli_final -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1_cli.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/k1_sbb_final -f python bench.py --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1_sbb.log 2>&1
tail -1 gpurun_out/ncu_k1_sbb.log
