mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
: > gpurun_out/compute_sanitizer.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool python scripts/sanitize_small.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?: $(grep -E 'sanitize script ok' gpurun_out/san_$tool.log | head -1)" >> gpurun_out/compute_sanitizer.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error:|access at" gpurun_out/san_$tool.log | sed "s/^/$tool: /" | head -8 >> gpurun_out/compute_sanitizer.txt
done
for pre in "GIGA_A_PRE=0" "GIGA_B_PRE=0"; do
  for tool in memcheck racecheck synccheck; do
    env $pre timeout -s KILL 600 compute-sanitizer --tool $tool python scripts/sanitize_t2_onchip.py > gpurun_out/san_t2.log 2>&1
    echo "t2 $pre $tool rc=$?: $(grep -E 'sanitize script ok' gpurun_out/san_t2.log | head -1)" >> gpurun_out/compute_sanitizer.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error:|access at" gpurun_out/san_t2.log | sed "s/^/t2 $pre $tool: /" | head -6 >> gpurun_out/compute_sanitizer.txt
  done
done
timeout -s KILL 300 compute-sanitizer --tool racecheck python scripts/racecheck_pair_alloc.py > gpurun_out/san_pair.log 2>&1
echo "racecheck pair-alloc-only kernel rc=$?" >> gpurun_out/compute_sanitizer.txt
grep -E "pair alloc|RACECHECK SUMMARY|Error:|access at" gpurun_out/san_pair.log | sed "s/^/pair_alloc: /" | head -8 >> gpurun_out/compute_sanitizer.txt
cat gpurun_out/compute_sanitizer.txt
