#!/bin/bash
# one GPU round trip: parity tests, bench line (+ a second window sample), per-CTA phase times (run under gpurun)
T=${TAG:-chk}
O=gpurun_out
if [ -z "$NOTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log; fi
timeout 900 python bench.py ${BENCH_ARGS:---no-cpu-baseline} > $O/${T}_bench.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-full-run > $O/${T}_bench2.log 2>&1
[ -n "$BLOCK" ] && timeout 600 python tools/block_times.py bay9m > $O/${T}_block_times.txt 2>&1
tail -n 3 $O/${T}_pytest.log; tail -c 600 $O/${T}_bench.log
