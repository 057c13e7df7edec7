# 3xFP16 operand preparation: its parity tests and the launch list of the preparation kernels at c5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_fp16.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_fp16i.log 2>&1; echo fp16_rc=$?; tail -1 gpurun_out/pytest_fp16i.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep|compact|fix" -c 12 --csv --log-file gpurun_out/launches_prep_c5d.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_prep_c5d.csv')))
hdr=None; tot={}
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); k=d['Kernel Name'].split('(')[0]
        tot.setdefault(k,[]).append(float(d['Metric Value']))
for k,v in tot.items(): print(k, len(v), round(sum(v)/len(v)/1e3,1), 'us')
PY
