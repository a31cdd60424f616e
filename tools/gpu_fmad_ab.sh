#!/bin/bash
# A/B: device FMA contraction off (-fmad=false, r01 default) vs on; GPU parity of the trees at each
mkdir -p gpurun_out
for F in 0 1; do
  OOCGB_FMAD=$F python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)" > gpurun_out/build_fmad$F.log 2>&1
  python -c "import oracle; oracle.build()" > /dev/null 2>&1
  timeout 900 python -m pytest tests -m gpu -q -x --tb=line -k "tree_bit_exact or sample_bit_exact or goss or depth8 or quant_bits or streamed" 2>&1 | tail -2
  for i in 1 2; do
    python bench.py --no-cpu-baseline --no-link > gpurun_out/bench_fmad$F.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/bench_fmad$F.json'));print('fmad=$F',round(d['value']*1e3,4),'ms', {k: round(v,4) for k,v in d['phases_ms_per_round'].items()})"
  done
done
