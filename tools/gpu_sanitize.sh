#!/bin/bash
# compute-sanitizer over the whole hot path (tools/sanitize_run.py), logs to gpurun_out/sanitize_*.log
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for T in memcheck racecheck synccheck initcheck; do
  ARGS=""; W=""
  [ "$T" = "racecheck" ] && ARGS="--racecheck-report all" && W=small
  [ "$T" = "initcheck" ] && W=small
  timeout 1500 compute-sanitizer --tool $T $ARGS --print-limit 50 python tools/sanitize_run.py $W > gpurun_out/sanitize_$T.log 2>&1
  echo "== $T rc=$?"; tail -4 gpurun_out/sanitize_$T.log
done
