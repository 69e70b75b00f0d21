mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_bulk -s 3 -c 1 -o gpurun_out/bulk_c4 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bulk.log 2>&1
tail -5 gpurun_out/ncu_bulk.log
