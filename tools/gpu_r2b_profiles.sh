# round 2 (second session) final profiles: launch list of the default bench + ncu --set full of the hot kernel per
# workload; the reports are exported to CSV on the box (raw metrics + SASS source page) and only
# the headline workload's .ncu-rep is kept (gpurun_out/ travels back only up to 64 MiB)
mkdir -p gpurun_out /tmp/ncu
B="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_c4.csv python bench.py $B > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
cap() {  # name regex args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o /tmp/ncu/r02b_$1 -f python bench.py $B $3 > gpurun_out/ncu_$1.log 2>&1; echo "$1 rc=$?"
  ncu -i /tmp/ncu/r02b_$1.ncu-rep --page raw --csv > gpurun_out/r02b_$1.raw.csv 2>/dev/null
  ncu -i /tmp/ncu/r02b_$1.ncu-rep --page source --csv --print-source=sass > gpurun_out/r02b_$1.sass.csv 2>/dev/null
  ncu -i /tmp/ncu/r02b_$1.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/r02b_$1.src.csv 2>/dev/null
}
cap c4_cli_fast k_sweep_cpipe ""
cap c4_cli_exact k_sweep_cpipe "--math exact"
cap c4_sbb_fast k_sweep_cpipe "--scheme SBB"
cap c2_fast k_sweep_cpipe "--config C2"
cap c3_fast k_sweep_cpipe "--config C3"
cap c5_fast k_sweep_pipe "--config C5"
cp /tmp/ncu/r02b_c4_cli_fast.ncu-rep gpurun_out/
python -c "import paper_1507_06565_b200 as pg; print(pg.build_info())" > gpurun_out/r02b_build_info.txt
du -sh gpurun_out
