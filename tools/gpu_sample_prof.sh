#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/sample_bench.py 100000000 5
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sample_launches.csv \
   python tools/sample_bench.py 100000000 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/sample_launches.csv')))
hdr=None; seq=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            seq.append((d['Kernel Name'][:40], float(d['Metric Value'])))
for k,v in seq[-60:]: print(f"{v/1000:9.1f} us  {k}")
PY
