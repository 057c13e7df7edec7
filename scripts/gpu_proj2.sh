# N > 1 per-GPU compute projection after the 3xFP16 epilogue fix and the refitted chunk model.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1500 python scripts/project_scaling.py c3_16384 c5_32768 c4_tall c2_4096 > gpurun_out/proj_pow2scale.jsonl 2> gpurun_out/proj.err; echo proj_rc=$?
cat gpurun_out/proj_pow2scale.jsonl
