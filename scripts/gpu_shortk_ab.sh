mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export SHAPES="16384,32768,1024;262144,1024,1024;16384,32768,4096;32768,32768,32768" TERMS=4 REPS=3
for v in "X=1" "GIGA_WAVE_SYNC=0" "GIGA_PROMOTE_KBLOCKS=16" "GIGA_GROUP_M=16" "GIGA_GROUP_M=4"; do
  echo "== $v"; env $v timeout -s KILL 600 python scripts/shortk_probe.py 2>&1 | tail -4
done
