mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu.py -q -x > gpurun_out/pytest_lo.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_lo.log
run() { timeout -s KILL 300 python bench.py --config $2 --steps 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['gpu_launches'])"; }
for c in c3_16384 c5_32768 c2_4096 c4_tall; do
GIGA_LO_PRESPLIT=0 run smem $c
done
GIGA_LO_PRESPLIT=1 run presplit c3_16384
GIGA_CTA_GROUP=1 run cg1_smem c3_16384
