#!/bin/bash
# round-2 session-3 evidence (1 GPU): GPU tests, the driver's bench command, the reference arm,
# K partitions in one process, ncu launch list + a cold step + a steady launch
O=gpurun_out
T=${TAG:-r4}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 $O/${T}_gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_bench_reference.json 2> $O/${T}_bench_reference.err; echo "reference rc=$?"
for k in 2 4 8; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-full-run --no-cpu-baseline --parts $k > $O/${T}_bench_parts$k.json 2> $O/${T}_bench_parts$k.err; echo "parts $k rc=$?"
done
TAG=$T STEPS=3 WARM=3 bash tools/profile.sh > $O/${T}_profile.log 2>&1; echo "profile rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "steady/" -k regex:k_run -s 1 -c 1 \
  -o $O/prof_${T}s -f python bench.py --steps 4 --warmup 3 --no-full-run --no-cpu-baseline > $O/prof_${T}s.stdout 2>&1; echo "steady profile rc=$?"
ls -la $O | grep $T
