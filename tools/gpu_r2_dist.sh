# round 2: native multi-GPU path on one B200 (local transport, NCCL world 1), C++ demos
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_cpp_demo.py -q -m "gpu and not slow" > gpurun_out/dist_tests.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/dist_tests.log
timeout 1500 python -m pytest tests -q -m "gpu and not slow" > gpurun_out/gpu_tests.log 2>&1; echo "all gpu tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
