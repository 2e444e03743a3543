#!/bin/bash
# K partitions in one process (pilot-balanced multilevel partition), variants under ab/
O=gpurun_out
for v in ${VARIANTS:-base}; do
  for k in ${KS:-1 2 4 8}; do
    LPSIM_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 20 --warmup 5 --no-full-run --no-cpu-baseline --parts $k \
      ${EXTRA} > $O/r4_parts_${v}_$k.json 2> $O/r4_parts_${v}_$k.err
    python - "$O/r4_parts_${v}_$k.json" "$v" "$k" <<'PY'
import json, sys
try:
    l = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])
    print(sys.argv[2], "K", sys.argv[3], "cold us %.2f steady us %.2f" % (1e3 * l["ms_per_step"], 1e3 * l["steady_state"]["ms_per_step"]))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "failed", e)
PY
  done
done
