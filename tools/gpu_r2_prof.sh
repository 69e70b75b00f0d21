# round 2: fast-mode tests + ncu captures of the C4 K1 (exact / fast, CLI and SBB)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -m "gpu and not slow" > gpurun_out/fast_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/fast_tests.log
for m in exact fast; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/r2_k1_cli_$m -f python bench.py --math $m --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1_cli_$m.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/r2_k1_sbb_fast -f python bench.py --math fast --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1_sbb_fast.log 2>&1
ls -la gpurun_out/*.ncu-rep
