# GPU suite on the bounds-checking build (device traps on any out-of-range compact address)
mkdir -p gpurun_out
PGPU_LIB=paper_1507_06565_b200/_variants/bounds/libporolb_cuda.so timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_bounds.log 2>&1; echo rc=$? >> gpurun_out/t_bounds.log; tail -3 gpurun_out/t_bounds.log
PGPU_LIB=paper_1507_06565_b200/_variants/bounds/libporolb_cuda.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-120
PGPU_LIB=paper_1507_06565_b200/_variants/bounds/libporolb_cuda.so timeout 300 python bench.py --force-slab --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-120
