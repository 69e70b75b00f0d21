# Full GPU suite on the bounds-checking build with the fluid-only layout forced everywhere.
mkdir -p gpurun_out
PGPU_LAYOUT=compact PGPU_LIB=paper_1507_06565_b200/_variants/bounds/libporolb_cuda.so timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/t_bounds_all.log 2>&1; echo rc=$? >> gpurun_out/t_bounds_all.log
tail -12 gpurun_out/t_bounds_all.log
