#!/bin/bash
# One gpurun call: build, parity tests, smoke, bench JSON, ncu launch list, ncu full capture of k_hist.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -q -m gpu --tb=short --timeout 300 ${PYARGS} 2>&1 | tail -40 > gpurun_out/parity.log
  tail -5 gpurun_out/parity.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --profile-only --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist -s 8 -c ${HIST_COUNT:-8} -o gpurun_out/prof_hist -f \
     python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
fi
ls -la gpurun_out
