#!/bin/bash
# A/B of library builds on one box, interleaved bench window runs (lean kernel).
# CFGS="name:lib[:exp_flags] ..." (lib under ab/, exp_flags for LPSIM_EXP builds); default: every ab/*.so
O=gpurun_out
R=${ROUNDS:-3}
if [ -z "$CFGS" ]; then for f in ab/*.so; do n=$(basename $f .so); CFGS="$CFGS $n:$n"; done; fi
for i in $(seq 1 $R); do
  for c in $CFGS; do
    IFS=: read n lib fl <<< "$c"
    LPSIM_EXP_FLAGS=$fl LPSIM_LIB=$PWD/ab/$lib.so timeout 300 python bench.py --no-full-run --no-cpu-baseline ${BENCH_ARGS} > $O/ab_${n}_$i.log 2>&1
    python - "$O/ab_${n}_$i.log" "$n" <<'PY'
import json, sys
try:
    l = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])
    print(sys.argv[2], "cold ms %.5f steady ms %.5f" % (l["ms_per_step"], l["steady_state"]["ms_per_step"]))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
  done
done
