# Per-GPU compute projection for both transports (NCCL pipeline on 140 SMs with row-chunked last
# K-chunk; p2p on all SMs, one launch per K-chunk), after the late round-2 changes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1200 python scripts/project_scaling.py c3_16384 c5_32768 > gpurun_out/proj_nccl_final.jsonl 2> gpurun_out/proj.err; echo nccl_rc=$?
GIGA_TRANSPORT=p2p timeout -s KILL 1200 python scripts/project_scaling.py c3_16384 c5_32768 > gpurun_out/proj_p2p_final.jsonl 2>> gpurun_out/proj.err; echo p2p_rc=$?
python - <<'PY'
import json
for t in ("nccl", "p2p"):
    for l in open(f"gpurun_out/proj_{t}_final.jsonl"):
        d = json.loads(l)
        print(t, d["config"], {w: (d[w]["compute_ms"], d[w].get("compute_speedup_vs_1")) for w in ("1", "2", "4", "8")})
PY
timeout -s KILL 900 python -m pytest tests/test_gpu_vec.py -q -p no:cacheprovider > gpurun_out/pytest_vec.log 2>&1; echo vec_rc=$?; tail -2 gpurun_out/pytest_vec.log
