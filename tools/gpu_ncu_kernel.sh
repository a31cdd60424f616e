#!/bin/bash
# ncu full capture of kernels matching $KREGEX (skip $NSKIP, capture $NCOUNT) on a short bench run.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${NSKIP:-8} -c ${NCOUNT:-8} -o gpurun_out/prof_${TAG} -f \
   python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}.log 2>&1; tail -2 gpurun_out/ncu_${TAG}.log
