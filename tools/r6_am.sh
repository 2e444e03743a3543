#!/bin/bash
# migrants materialised by the first admit CTA: GPU parity, then K-partition A/B against the previous build
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r6_am_test.log 2>&1; echo "gputest rc=$?"; tail -4 $O/r6_am_test.log
for k in 8 4 2; do ROUNDS=2 BENCH_ARGS="--parts $k --steps 20 --warmup 5" bash tools/ab.sh 2>&1 | sed "s/^/K=$k /"; done | tee $O/r6_am_ab.txt
