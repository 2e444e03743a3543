#!/bin/bash
# one GPU round trip: parity tests, bench line, per-CTA phase times (run under gpurun)
T=${TAG:-chk}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 900 python bench.py ${BENCH_ARGS:---no-cpu-baseline} > $O/${T}_bench.log 2>&1
[ -n "$BLOCK" ] && timeout 600 python tools/block_times.py bay9m > $O/${T}_block_times.txt 2>&1
tail -n 3 $O/${T}_pytest.log; tail -c 600 $O/${T}_bench.log
