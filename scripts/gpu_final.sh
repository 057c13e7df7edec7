# end-of-round evidence: suite + bench lines + ncu launch lists and full captures
mkdir -p gpurun_out
bash scripts/gpu_full_bench2.sh
bash scripts/gpu_prof_tf32bf16.sh
