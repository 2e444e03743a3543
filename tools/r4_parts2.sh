#!/bin/bash
# A/B of the deferred migrant prefix and the admit-CTA threshold (K partitions in one process), then GPU parity of defer32
O=gpurun_out
for r in 1 2; do VARIANTS="nadmin32 defer32 defer" KS="1 4 8" bash tools/r4_parts.sh; done 2>&1 | tee $O/r4_parts2.txt
LPSIM_LIB=$PWD/ab/defer32.so timeout 900 python -m pytest tests -m gpu -x -q > $O/r4_defer_test.log 2>&1; echo "test defer32 rc=$?"; tail -3 $O/r4_defer_test.log
