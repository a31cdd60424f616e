#!/bin/bash
# iteration: build, GPU tests ($PYT files, default parity), bench (no CPU leg), launch list of one round
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest ${PYT:-tests/test_gpu_parity.py} -m gpu -q -x --tb=short ${PYK:+-k "$PYK"} 2>&1 | tail -30 > gpurun_out/iter_tests.log; tail -30 gpurun_out/iter_tests.log
if [ -z "$SKIP_BENCH" ]; then
timeout 600 python bench.py --no-cpu-baseline --no-link ${BENCH_ARGS} > gpurun_out/iter_bench.json 2> gpurun_out/iter_bench.err; tail -2 gpurun_out/iter_bench.err
python -c "import json;d=json.load(open('gpurun_out/iter_bench.json'));print('VALUE',round(d['value']*1e3,4),'ms', {k:round(v,4) for k,v in d['phases_ms_per_round'].items()}, 'hist frac', round(d['roofline']['frac'],3), 'part', round(d['partition']['frac_of_hbm'],3))"
fi
if [ -z "$SKIP_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX:-k_}" --csv --log-file gpurun_out/iter_launches.csv python bench.py --profile-only --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/iter_launches.csv 2
fi
