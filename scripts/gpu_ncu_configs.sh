# ncu --set full of the product GEMM launch at every BASELINE config (after the epilogue fix):
# DRAM traffic per launch for bench.py's roofline.traffic, tensor-pipe %, clocks.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "c2 4096,4096,4096" "c3 16384,16384,16384" "c4 262144,1024,1024" "c5 32768,32768,32768"; do
  set -- $cfg
  SHAPES="$2" TERMS=4 REPS=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_$1_pow2 python scripts/shortk_probe.py > gpurun_out/ncu_$1.log 2>&1; echo ncu_$1_rc=$?
  python scripts/ncu_summary.py gpurun_out/prof_$1_pow2.ncu-rep > gpurun_out/prof_$1_pow2_summary.json 2>&1
  grep -E "duration|dram__bytes_(read|write)|tensor_cycles|per_second\"" gpurun_out/prof_$1_pow2_summary.json
done
