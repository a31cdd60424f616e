#!/bin/bash
# ncu --set full of the 8 k_eval_narrow and 8 k_part_fused launches of one config-2 round
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_eval_narrow|k_part_fused" -s 16 -c 16 -o gpurun_out/prof_evalpart -f \
   python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_evalpart.log 2>&1; tail -1 gpurun_out/ncu_evalpart.log
