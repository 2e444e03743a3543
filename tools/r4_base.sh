#!/bin/bash
# round-2 session-3 baseline (1 GPU): build, GPU tests, the driver's bench command
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r4_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 $O/r4_gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/r4_bench.json 2> $O/r4_bench.err; echo "bench rc=$?"; tail -c 600 $O/r4_bench.json
