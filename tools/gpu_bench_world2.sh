# the N>1 bench path on ONE B200: 2 ranks as processes on cuda:0, gloo for the
# host-side collectives, the IPC halo transport (correctness of the flow and
# --verify parity; the timing of two time-sliced ranks on one GPU means nothing)
mkdir -p gpurun_out
for sc in strong weak; do
PGPU_BENCH_ONE_DEVICE=1 PGPU_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 2 --steps 10 --warmup 3 --scaling $sc --verify --transport ipc --no-cpu-baseline > gpurun_out/w2_$sc.json 2> gpurun_out/w2_$sc.err; echo "$sc rc=$?"
python -c "
import json; L=[l for l in open('gpurun_out/w2_$sc.json') if l.startswith('{')]; d=json.loads(L[-1]); print('$sc', d['n_gpus'], d['config']['workload'], d['config']['parallelism'], round(d['value']), d.get('parity'), round(d['e2e']['value']), d['halo_transport'])" || tail -20 gpurun_out/w2_$sc.err
done
