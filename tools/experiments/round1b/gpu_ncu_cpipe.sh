# GPU suite (both layouts) + ncu of the compact K1 (CLI and SBB) on C4.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/cpipe_cli -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cpipe_cli.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/cpipe_sbb -f python bench.py --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cpipe_sbb.log 2>&1
tail -2 gpurun_out/ncu_cpipe_sbb.log
