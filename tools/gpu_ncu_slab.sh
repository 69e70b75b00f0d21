# ncu of the slab path's compact kernels (edge part and interior part) on C4, one B200.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv -k regex:k_sweep_cpipe -s 6 -c 6 python bench.py --force-slab --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_slab.csv 2> gpurun_out/ncu_slab.err
tail -30 gpurun_out/ncu_slab.csv
