#!/bin/bash
# round-2 session-2 measurement (run under gpurun, 1 GPU): tests, the driver's bench command,
# K partitions in one process, ncu of a cold step and of a steady 127-step launch
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/r3_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 $O/r3_gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/r3_bench.json 2> $O/r3_bench.err; echo "bench rc=$?"
for k in 2 4 8; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-full-run --no-cpu-baseline --parts $k > $O/r3_bench_parts$k.json 2> $O/r3_bench_parts$k.err; echo "parts $k rc=$?"
done
TAG=r3 STEPS=3 WARM=3 bash tools/profile.sh > $O/r3_profile.log 2>&1; echo "profile rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "steady/" -k regex:k_run -s 1 -c 1 \
  -o $O/prof_r3s -f python bench.py --steps 4 --warmup 3 --no-full-run --no-cpu-baseline > $O/prof_r3s.stdout 2>&1; echo "steady profile rc=$?"
