#!/bin/bash
# One gpurun call: build, GPU parity tests (output under gpurun_out/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_2005_09148_b200.build as b; b.build()" 2>&1 | tail -3
timeout ${T:-1200} python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=short --timeout 300 ${PYARGS} 2>&1 | tail -120 > gpurun_out/parity.log
cat gpurun_out/parity.log
