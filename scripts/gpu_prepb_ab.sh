# prep16_b_kernel variants (rows in flight / blocks per SM): ncu launch times at 32768^3.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 0 1 2 3; do
GIGA_PREP_B_VARIANT=$v SHAPES="16384,32768,16384" TERMS=4 REPS=6 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:prep16_b_kernel --csv --log-file gpurun_out/prepb_v$v.csv python scripts/shortk_probe.py > /dev/null 2>&1
echo "v$v: $(grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/prepb_v$v.csv | tr '\n' ' ')"
done
