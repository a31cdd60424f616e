#!/bin/bash
# A/B of build-time variants: GPU parity at the default, then config-2 bench per variant
# (usage: bash tools/gpu_ab.sh "" "-DMACRO=1" ...; "" = the default build)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for V in "$@"; do
  OOCGB_EXTRA_NVCC="$V" python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)"
  python bench.py --no-cpu-baseline > gpurun_out/bench_v.json 2>gpurun_out/bench_v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_v.json'));print('[$V]',round(d['value']*1e3,4),'ms', {k: round(v,4) for k,v in d['phases_ms_per_round'].items()})"
done
