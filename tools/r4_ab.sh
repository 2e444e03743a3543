#!/bin/bash
# A/B of ab/*.so variants (tools/ab.sh) + GPU parity of the variant named by $TESTLIB
O=gpurun_out
ROUNDS=${ROUNDS:-3} bash tools/ab.sh 2>&1 | tee $O/r4_ab.txt
if [ -n "$TESTLIB" ]; then
  LPSIM_LIB=$PWD/ab/$TESTLIB.so timeout 900 python -m pytest tests -m gpu -x -q > $O/r4_abtest.log 2>&1; echo "test $TESTLIB rc=$?"; tail -3 $O/r4_abtest.log
fi
