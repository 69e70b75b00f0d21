# ncu --set full of the TMA sweep on C4 (CLI fast), exported to CSV on the box
mkdir -p gpurun_out /tmp/ncu
B="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config"
PGPU_SWEEP=tma timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 3 -c 1 -o /tmp/ncu/tma_c4 -f python bench.py $B > gpurun_out/ncu_tma.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/ncu/tma_c4.ncu-rep --page raw --csv > gpurun_out/tma_c4.raw.csv 2>/dev/null
ncu -i /tmp/ncu/tma_c4.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/tma_c4.src.csv 2>/dev/null
ncu -i /tmp/ncu/tma_c4.ncu-rep --page details --csv > gpurun_out/tma_c4.details.csv 2>/dev/null
ls -la gpurun_out/tma_c4*
