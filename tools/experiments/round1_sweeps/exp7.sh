prof() { local tag=$1; shift; env "$@" ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sweep_pipe -s 2 -c 1 --csv python bench.py --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram__bytes|duration" | awk -F'","' -v t=$tag '{print t, $(NF-2), $(NF-1), $NF}'; }
run() { local envs="$1"; shift; timeout 300 env $envs python bench.py "$@" --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs $*', round(d['value']), 'MLUPS', round(d['roofline']['frac'],3), round(d['ms_per_step'],3),'ms')"; }
python bench.py --scheme SBB --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && echo plain-ok
python -c "
import ctypes; c=ctypes.CDLL('libcudart.so'); v=ctypes.c_size_t(); print('default L2 fetch granularity', c.cudaDeviceGetLimit(ctypes.byref(v), 0x13), v.value)" 2>&1 | tail -1
for g in 32 64 128; do prof "l2fetch=$g" PGPU_L2_FETCH=$g; done
for g in 32 64 128; do run "PGPU_L2_FETCH=$g" --scheme SBB; run "PGPU_L2_FETCH=$g" --scheme CLI; done
