# usage: bash tools/gpu_ab.sh "C4 C3" variant...   (A/B of the product build vs variants)
mkdir -p gpurun_out
bash tools/ab_bench.sh "$@" 2>&1 | tee gpurun_out/ab.log
