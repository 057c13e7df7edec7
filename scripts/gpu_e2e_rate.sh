# e2e (host buffers) at c5 / c3 with the host-plan GEMM rate model at its default and at 270
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for cfg in c5_32768 c3_16384; do
  for rate in "" 270; do
    GIGA_HOST_GEMM_TFLOPS=$rate timeout -s KILL 600 python bench.py --config $cfg --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', 'rate=${rate:-default}', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
  done
done
