#!/bin/bash
# occupancy experiment: rebuild with a different CTAs-per-SM register budget, bench window only
for mb in ${MBS:-4 3}; do
  LPSIM_NVCC_EXTRA="-DLPSIM_MINB=$mb" python -c "from paper_2406_08496_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-full-run --no-cpu-baseline > gpurun_out/exp_minb$mb.log 2>&1
done
