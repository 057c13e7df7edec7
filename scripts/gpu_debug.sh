mkdir -p gpurun_out
python -c "from paper_2504_01266_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 120 python scripts/debug_umma.py 2>&1 | tail -30
