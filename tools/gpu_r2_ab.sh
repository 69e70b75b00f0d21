mkdir -p gpurun_out
bash tools/ab_variants.sh "C4" "fast exact" "product minb5 minb6" 2
bash tools/ab_variants.sh "C4" "fast" "product minb5 minb6" 2 "--scheme SBB"
bash tools/ab_variants.sh "C3 C2" "fast" "product minb5 minb6" 1
