#!/bin/bash
# ncu evidence for the bench's dominant kernel (run under gpurun, 1 GPU).
# Only launches inside bench.py's NVTX range "timed" are profiled.
set -x
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r1}
STEPS=${STEPS:-3}
WARM=${WARM:-3}
EXTRA=${EXTRA:-}
# 1) launch list of the timed region (every kernel, device time)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps $STEPS --warmup $WARM --no-full-run --no-cpu-baseline $EXTRA \
  > $OUT/launches_$TAG.stdout 2>&1
# 2) full section set of one timed k_run launch
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:k_run -c 1 \
  -o $OUT/prof_$TAG -f python bench.py --steps $STEPS --warmup $WARM --no-full-run --no-cpu-baseline $EXTRA \
  > $OUT/prof_$TAG.stdout 2>&1
ls -la $OUT
