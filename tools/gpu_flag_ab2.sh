#!/bin/bash
# A/B of compile-flag variants in one box: default twice (noise), then each variant ($@), 20 timed rounds each
mkdir -p gpurun_out
run() {
  OOCGB_EXTRA_NVCC="$1" python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "BUILD FAIL $1"
  timeout 300 python bench.py --no-cpu-baseline --no-link --steps 20 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('[$1]', round(d['value']*1e3,4),'ms', {k:round(v,4) for k,v in d['phases_ms_per_round'].items() if k in ('hist_ms','eval_ms','partition_ms')})" || tail -3 gpurun_out/ab.err
}
run ""
for V in "$@"; do run "$V"; done
run ""
python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
