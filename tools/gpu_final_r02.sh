#!/bin/bash
# r02 evidence run: build, default bench line (the driver's command), ncu launch list of the same
# bench, one --set full capture of the 8 k_hist launches of a round, sanitizers on the final code.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -2 gpurun_out/final_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
   python bench.py --profile-only --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist -s 8 -c 8 -o gpurun_out/final_hist -f \
   python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/final_ncu.log 2>&1; tail -1 gpurun_out/final_ncu.log
if [ -z "$SKIP_SAN" ]; then bash tools/gpu_sanitize.sh; fi
ls -la gpurun_out | tail -20
