#!/bin/bash
# --set full captures of one round's evaluation (k_eval / k_eval_narrow, 16 launches) and
# finalize + partition (16 launches), round 2 of a --profile-only run (config 2)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 16 -c 16 -o gpurun_out/prof_eval -f python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_eval.log 2>&1; tail -2 gpurun_out/ncu_eval.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_finalize|k_part_fused" -s 16 -c 16 -o gpurun_out/prof_fp -f python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_fp.log 2>&1; tail -2 gpurun_out/ncu_fp.log
