#!/bin/bash
# ncu evidence for the bench's dominant kernel (run under gpurun, 1 GPU).
# Launch count before the timed region: ffwd steps / sort period (k_run chunks) + warm-up steps.
set -x
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r1}
STEPS=${STEPS:-3}
WARM=${WARM:-3}
SKIP=$(( 57600 / 16 + WARM ))
# 1) launch list of the timed region (every kernel, device time)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $SKIP -c 200 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps $STEPS --warmup $WARM --no-full-run --no-cpu-baseline \
  > $OUT/launches_$TAG.stdout 2>&1
# 2) full section set of one timed k_run launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_run -s $SKIP -c 1 \
  -o $OUT/prof_$TAG -f python bench.py --steps $STEPS --warmup $WARM --no-full-run --no-cpu-baseline \
  > $OUT/prof_$TAG.stdout 2>&1
ls -la $OUT
