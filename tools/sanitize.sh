#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the step kernel on C1b (run on the GPU box).
# LPSIM_MAX_BLOCKS=8: a few CTAs, so the kernel runs several chunk rounds per CTA (HBM claim records).
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
export LPSIM_MAX_BLOCKS=8
for tool in memcheck synccheck racecheck; do
  steps=200; [ "$tool" = racecheck ] && steps=60
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $steps > "$out/$tool.txt" 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|digests' "$out/$tool.txt" | tr '\n' ' ')"
done
