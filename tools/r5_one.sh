#!/bin/bash
# the one-barrier step (not kept): GPU parity, then an A/B against the two-barrier build
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/r5_one_test.log 2>&1; echo "gputest rc=$?"; tail -15 $O/r5_one_test.log
ROUNDS=2 CFGS="cur:cur one:one" bash tools/ab.sh 2>&1 | tee $O/r5_one_ab.txt
