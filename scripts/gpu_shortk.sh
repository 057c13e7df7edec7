# Where short-K 3xFP16 launches lose time: event times per scheme, the launch list of one
# K = 1024 chunk shape and of c4, and one ncu --set full capture of the K = 1024 GEMM.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python scripts/shortk_probe.py > gpurun_out/shortk_probe.log 2>&1; echo probe_rc=$?; cat gpurun_out/shortk_probe.log | tail -14
SHAPES="16384,32768,1024" TERMS=4 REPS=1 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shortk_16k32k1k.csv python scripts/shortk_probe.py > /dev/null 2>&1; echo l1_rc=$?
SHAPES="262144,1024,1024" TERMS=4 REPS=1 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shortk_c4.csv python scripts/shortk_probe.py > /dev/null 2>&1; echo l2_rc=$?
SHAPES="16384,32768,1024" TERMS=4 REPS=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_shortk python scripts/shortk_probe.py > gpurun_out/ncu_shortk.log 2>&1; echo ncu_rc=$?
