#!/bin/bash
# CTA-size experiment: rebuild with LPSIM_BS / LPSIM_MINB, bench window only
for cfg in ${CFGS:-"768 1" "384 2" "256 3"}; do
  set -- $cfg
  LPSIM_NVCC_EXTRA="-DLPSIM_BS=$1 -DLPSIM_MINB=$2" python -c "from paper_2406_08496_b200 import build; build.build(force=True)" > gpurun_out/exp_bs_build_$1.log 2>&1
  timeout 600 python bench.py --no-full-run --no-cpu-baseline > gpurun_out/exp_bs$1.log 2>&1
done
