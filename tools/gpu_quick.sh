#!/bin/bash
# quick loop: build, GPU parity (+multirank), bench, per-kernel durations of one round (ncu)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; tail -1 gpurun_out/bench_q.err
python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print('VALUE',d['value']*1e3,'ms', d['phases_ms_per_round'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX:-k_}" --csv --log-file gpurun_out/quick_launches.csv python bench.py --profile-only --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/quick_launches.csv
