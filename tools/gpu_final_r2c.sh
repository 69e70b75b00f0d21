# round 2 (fourth session) final: GPU suite, smoke, default bench, reference arm, profiles
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02c_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed" gpurun_out/r02c_gpu_tests.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02c_bench_ref.json 2> gpurun_out/r02c_bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --force-slab --verify --no-cpu-baseline > gpurun_out/r02c_bench_slab.json 2> gpurun_out/r02c_bench_slab.err; echo "slab rc=$?"
PREFIX=r02c bash tools/gpu_r2c_profiles.sh
