# round 2 (fourth session) profiles: launch list of the default bench + ncu --set full of the hot
# kernel per workload (units sweep k_sweep_units on the fluid-only layout; the chunk sweep on C4 and
# the dense layout's k_sweep_pipe on C5 for comparison); reports exported to CSV on the box (raw metrics + SASS source page); only the
# headline workload's .ncu-rep is kept (gpurun_out/ travels back only up to 64 MiB)
#   CAPS="c4_cli_fast c3_fast" bash tools/gpu_r2c_profiles.sh     (default: all)
mkdir -p gpurun_out /tmp/ncu
P=${PREFIX:-r02c}
B="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config"
CAPS=${CAPS:-launches c4_cli_fast c4_cli_exact c4_sbb_fast c2_fast c3_fast c5_fast c5_fast_dense c4_cli_fast_cpipe}
cap() {  # name regex args [env]
  timeout 900 env $4 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o /tmp/ncu/${P}_$1 -f python bench.py $B $3 > gpurun_out/ncu_$1.log 2>&1; echo "$1 rc=$?"
  ncu -i /tmp/ncu/${P}_$1.ncu-rep --page raw --csv > gpurun_out/${P}_$1.raw.csv 2>/dev/null
  ncu -i /tmp/ncu/${P}_$1.ncu-rep --page source --csv --print-source=sass > gpurun_out/${P}_$1.sass.csv 2>/dev/null
  ncu -i /tmp/ncu/${P}_$1.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/${P}_$1.src.csv 2>/dev/null
}
for c in $CAPS; do case $c in
  launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches_c4.csv python bench.py $B > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?";;
  c4_cli_fast) cap c4_cli_fast k_sweep_units "";;
  c4_cli_exact) cap c4_cli_exact k_sweep_units "--math exact";;
  c4_sbb_fast) cap c4_sbb_fast k_sweep_units "--scheme SBB";;
  c2_fast) cap c2_fast k_sweep_units "--config C2";;
  c3_fast) cap c3_fast k_sweep_units "--config C3";;
  c5_fast) cap c5_fast k_sweep_units "--config C5";;
  c5_fast_dense) cap c5_fast_dense k_sweep_pipe "--config C5" PGPU_LAYOUT=dense;;
  c4_cli_fast_cpipe) cap c4_cli_fast_cpipe k_sweep_cpipe "" PGPU_SWEEP=cpipe;;
esac; done
[ -f /tmp/ncu/${P}_c4_cli_fast.ncu-rep ] && cp /tmp/ncu/${P}_c4_cli_fast.ncu-rep gpurun_out/
python -c "import paper_1507_06565_b200 as pg; print(pg.build_info())" > gpurun_out/${P}_build_info.txt
du -sh gpurun_out
