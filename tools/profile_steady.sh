#!/bin/bash
# ncu --set full of one steady-state k_run launch (K steps in one lpsim_step call, no L2 flush)
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r1s}
STEPS=${STEPS:-16}
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "steady/" -k regex:k_run -c 1 \
  -o $OUT/prof_$TAG -f python bench.py --steps $STEPS --warmup 3 --no-full-run --no-cpu-baseline \
  > $OUT/prof_$TAG.stdout 2>&1
ls -la $OUT | grep $TAG
