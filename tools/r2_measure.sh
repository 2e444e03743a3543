#!/bin/bash
# r2 measurement round (run under gpurun, 1 GPU): the driver's bench command, the a9 ablation, ncu
O=gpurun_out
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/r2_bench.json 2> $O/r2_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 --no-full-run --no-cpu-baseline --ablation nosort > $O/r2_bench_nosort.json 2> $O/r2_bench_nosort.err; echo "nosort rc=$?"
TAG=r2 STEPS=3 WARM=3 bash tools/profile.sh > $O/r2_profile.log 2>&1; echo "profile rc=$?"
TAG=r2ns STEPS=3 WARM=3 EXTRA="--ablation nosort" bash tools/profile.sh > $O/r2ns_profile.log 2>&1; echo "profile ns rc=$?"
