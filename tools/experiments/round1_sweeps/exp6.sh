# ncu DRAM traffic of K1 on the C4 geometry (SBB) vs z-chunk depth and bounce loads
V=paper_1507_06565_b200/_variants
prof() { local tag=$1; shift; env "$@" ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_sweep_pipe -s 2 -c 1 --csv python bench.py --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram__bytes|duration|hit_rate" | awk -F'","' -v t=$tag '{print t, $(NF-2), $(NF-1), $NF}'; }
python bench.py --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && echo plain-ok
for zp in 1 4 8 32 128; do prof "zper=$zp" PGPU_ZPER=$zp; done
prof "nobounce" PGPU_LIB=$V/nobounce/libporolb_cuda.so PGPU_ZPER=8
