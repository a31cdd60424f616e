#!/bin/bash
# A/B of k_hist block shapes for the deep levels: parity + bench at the default, then variants.
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/bench_a.json 2>gpurun_out/bench_a.err
python -c "import json;d=json.load(open('gpurun_out/bench_a.json'));print('default',d['value']*1e3,'ms', d['phases_ms_per_round'])"
for V in "$@"; do
  OOCGB_EXTRA_NVCC="$V" python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)"
  python bench.py --no-cpu-baseline > gpurun_out/bench_v.json 2>gpurun_out/bench_v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_v.json'));print('$V',d['value']*1e3,'ms', d['phases_ms_per_round'])"
done
