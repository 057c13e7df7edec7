# ncu --set full of the 3xFP16 preparation kernels at 32768^3 (B split pass, A pass, B max).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for k in prep16_b_kernel prep16_a_kernel prep16_bmax_kernel; do
SHAPES="32768,32768,32768" TERMS=4 REPS=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k python scripts/shortk_probe.py > gpurun_out/ncu_$k.log 2>&1; echo ${k}_rc=$?
python scripts/ncu_summary.py gpurun_out/prof_$k.ncu-rep > gpurun_out/prof_${k}_summary.json 2>&1
grep -E "duration|dram__bytes_(read|write)|per_second\"" gpurun_out/prof_${k}_summary.json
done
