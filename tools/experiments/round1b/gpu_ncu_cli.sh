mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/cpipe_cli_m4 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cpipe_cli.log 2>&1
tail -1 gpurun_out/ncu_cpipe_cli.log
