set -x
python -c "from paper_2504_01266_b200 import build as b; b.build()"
python scripts/project_scaling.py c3_16384 c5_32768 > gpurun_out/proj_new.jsonl
GIGA_BCAST_CHUNKS=6 python scripts/project_scaling.py c3_16384 > gpurun_out/proj_b6.jsonl
GIGA_BCAST_CHUNKS=2 python scripts/project_scaling.py c3_16384 > gpurun_out/proj_b2.jsonl
cat gpurun_out/proj_*.jsonl
