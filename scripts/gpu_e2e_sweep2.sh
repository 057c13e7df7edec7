# Host-buffer e2e at 32768^3 under forced host plans vs the planner's choice (after the
# epilogue fix and the refitted host model).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
E2E_PLANS="auto;16384,16,16;12288,16,16;20480,16,16;16384,8,16;16384,16,8;14336,16,16;18432,16,16;16384,12,16" timeout -s KILL 1500 python scripts/e2e_plan_sweep.py > gpurun_out/e2e_plan_sweep2.jsonl 2>&1; echo rc=$?
cat gpurun_out/e2e_plan_sweep2.jsonl
