mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/k1_cli_prod -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
PGPU_LIB=paper_1507_06565_b200/_variants/nogj/libporolb_cuda.so timeout 600 ncu --set full --clock-control none -k regex:k_sweep_cpipe -s 3 -c 1 -o gpurun_out/k1_cli_nogj -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -2
