# compute-sanitizer memcheck / racecheck / initcheck on small runs of both layouts
mkdir -p gpurun_out
for tool in memcheck racecheck initcheck; do
  for l in compact dense; do
    PGPU_LAYOUT=$l timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${tool}_$l.log 2>&1
    echo "$tool $l rc=$? $(grep -c 'ERROR SUMMARY: 0 errors' gpurun_out/san_${tool}_$l.log) $(tail -1 gpurun_out/san_${tool}_$l.log)"
  done
done
