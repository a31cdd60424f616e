#!/bin/bash
# default build: parity + bench + launch list; then bench per extra-flag variant ($@)
bash tools/gpu_iter2.sh
for V in "$@"; do
  OOCGB_EXTRA_NVCC="$V" python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "BUILD FAIL $V"
  timeout 300 python bench.py --no-cpu-baseline --no-link > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$V', round(d['value']*1e3,4),'ms', {k:round(v,4) for k,v in d['phases_ms_per_round'].items() if k in ('hist_ms','eval_ms','partition_ms')})" || tail -3 gpurun_out/ab.err
done
python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
