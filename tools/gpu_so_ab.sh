#!/bin/bash
# same-box A/B of two prebuilt libraries: the current liboocgb.so (B) and liboocgb_base.so.ab (A)
mkdir -p gpurun_out
L=paper_2005_09148_b200/liboocgb.so
cp $L /tmp/lib_new.so
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-link --steps 20 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('[$1]', round(d['value']*1e3,4),'ms', {k:round(v,4) for k,v in d['phases_ms_per_round'].items() if k in ('hist_ms','eval_ms','partition_ms')})" || tail -3 gpurun_out/ab.err
}
for k in 1 2; do
  cp /tmp/lib_new.so $L; run new
  cp paper_2005_09148_b200/liboocgb_base.so.ab $L; run base
done
cp /tmp/lib_new.so $L
