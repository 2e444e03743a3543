#!/bin/bash
# current build: GPU tests, then the K-partition bench lines
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r4_check_test.log 2>&1; echo "gputest rc=$?"; tail -3 $O/r4_check_test.log
VARIANTS=cur KS="${KS:-1 2 4 8}" bash tools/r4_parts.sh 2>&1 | tee $O/r4_check_parts.txt
