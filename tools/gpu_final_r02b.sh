#!/bin/bash
# r02 final evidence: build, whole GPU suite, smoke, the driver's default bench line, the ncu launch
# list of the same bench, one --set full capture of the 8 k_hist launches of a round
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 2400 python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -8 > gpurun_out/final_tests.log; tail -3 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.err
python -c "import json;d=json.load(open('gpurun_out/final_bench.json'));print('VALUE',d['value']*1e3,'e2e',d['e2e']['value']*1e3,'frac',d['roofline']['frac'],'link',d['link']['busy_frac_of_peak'],'cpu',d['cpu_baseline']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
   python bench.py --profile-only --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist -s 8 -c 8 -o gpurun_out/final_hist -f \
   python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/final_ncu.log 2>&1; tail -1 gpurun_out/final_ncu.log
python tools/launch_summary.py gpurun_out/final_launches.csv 3 | head -14
