#!/bin/bash
# A/B of k_eval_narrow occupancy targets: parity + bench at the default, then bench at MINB=8.
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench_a.json 2>gpurun_out/bench_a.err
python -c "import json;d=json.load(open('gpurun_out/bench_a.json'));print('A',d['value']*1e3,'ms', d['phases_ms_per_round'])"
OOCGB_EXTRA_NVCC="-DOOCGB_EVAL_NARROW_MINB=8" python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)"
python bench.py --no-cpu-baseline > gpurun_out/bench_b.json 2>gpurun_out/bench_b.err
python -c "import json;d=json.load(open('gpurun_out/bench_b.json'));print('B',d['value']*1e3,'ms', d['phases_ms_per_round'])"
