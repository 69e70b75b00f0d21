mkdir -p gpurun_out
for c in C4 C2; do
for v in product sbb1s4 sbb2s4; do
  if [ $v = product ]; then unset PGPU_LIB; else export PGPU_LIB=paper_1507_06565_b200/_variants/$v/libporolb_cuda.so; fi
  st=200; [ $c != C4 ] && st=2000
  for rep in 1 2 3; do
    if [ $c = C4 ]; then a="--scheme SBB"; else a="--config $c"; fi
    python bench.py $a --steps $st --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$c'-SBB '$v'", round(d["value"]), round(d["roofline"]["frac"],3))'
  done
done
done
