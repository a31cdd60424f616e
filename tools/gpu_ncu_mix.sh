#!/bin/bash
# k_hist per-level DRAM bytes / time (metric list) + one kernel's --set full capture ($KFULL)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:k_hist -s 8 -c 8 --csv --log-file gpurun_out/hist_metrics.csv python bench.py --profile-only --steps 1 --warmup 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/hist_metrics.csv')) if len(r)>10]
h=rows[0]; i_id=h.index('ID'); i_m=h.index('Metric Name'); i_v=h.index('Metric Value'); i_u=h.index('Metric Unit')
d={}
for r in rows[1:]:
    d.setdefault(r[i_id],{})[r[i_m]]=(r[i_v],r[i_u])
for k in sorted(d,key=int):
    print(k, {m.split('.')[0][:28]:v for m,v in d[k].items()})
PY
if [ -n "$KFULL" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KFULL -s ${KSKIP:-8} -c ${KCOUNT:-2} -o gpurun_out/prof_$KFULL -f python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
fi
