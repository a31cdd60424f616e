#!/bin/bash
# round-end style check: build, the whole GPU suite, smoke, the driver's default bench line, ncu launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 2400 python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -8 > gpurun_out/final_tests.log; tail -3 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.err
python -c "import json;d=json.load(open('gpurun_out/final_bench.json'));print('VALUE',d['value']*1e3,'e2e',d['e2e']['value']*1e3,'frac',d['roofline']['frac'],'link',d['link']['busy_frac_of_peak'],'cpu',d['cpu_baseline']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
   python bench.py --profile-only --steps 2 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/final_launches.csv 3 | head -16
