# launch lists (ncu, serialised) of 3xFP16 at the shapes where it loses to 3xTF32
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for sh in 262144x1024x1024 4096x4096x4096 16384x32768x1024; do
PROBE_ACC=0 PROBE_TERMS=4,3 PROBE_SHAPES=$sh timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix" -c 16 --csv --log-file gpurun_out/launches_$sh.csv python scripts/fp16_probe.py > /dev/null 2>&1; echo ncu_rc=$?
done
PROBE_ACC=0 PROBE_TERMS=4,3 PROBE_SHAPES=262144x1024x1024,4096x4096x4096,16384x32768x1024,16384x16384x16384 python scripts/fp16_probe.py
