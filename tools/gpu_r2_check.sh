# round 2: GPU suite (not slow), default bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; cat gpurun_out/bench_default.json | head -c 4000; echo
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json | head -c 2000; echo
