#!/bin/bash
# ncu --set full of k_eval_narrow at the deepest levels (launches 6, 7 of the 2nd round) with source
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_narrow -s 14 -c 2 -o gpurun_out/prof_narrow -f \
   python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_narrow.log 2>&1; tail -2 gpurun_out/ncu_narrow.log
