mkdir -p gpurun_out
sed -i 's/for cfg in C2 C3 C5; do/for cfg in C2 C3 C4; do/; s/for z in 0 1 2 4 6 8; do/for z in 0 1 2 3 4 6 8 12 16; do/' tools/zper_sweep.sh
bash tools/zper_sweep.sh 2>&1 | tee gpurun_out/zper.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
