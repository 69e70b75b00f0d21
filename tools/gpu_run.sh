# generic: bash tools/gpu_run.sh '<command>'  (runs it with gpurun_out/ present)
mkdir -p gpurun_out
eval "$1"
