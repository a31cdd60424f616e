#!/bin/bash
mkdir -p gpurun_out
OOCGB_EXTRA_NVCC="-DOOCGB_PLAN_TRACE" python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
timeout 300 python bench.py --no-cpu-baseline --no-link --steps 2 --warmup 1 2>&1 | grep PLANTRACE | tail -16
python -c "from paper_2005_09148_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
