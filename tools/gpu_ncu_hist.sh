#!/bin/bash
# ncu full capture of k_hist (root level + level 1 of the 2nd round) and the launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist -s 8 -c ${NCOUNT:-2} -o gpurun_out/prof_hist${TAG} -f \
   python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches${TAG}.csv \
     python bench.py --profile-only --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
fi
