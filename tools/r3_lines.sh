#!/bin/bash
# load-stage times on C4; bench lines for C3 (paper's single-GPU case) and C5 (24M trips) on one GPU
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
LPSIM_LOAD_TIMES=1 REPS=2 timeout 900 python tools/load_times.py bay9m > $O/r3_load_times.txt 2>&1; echo "load times rc=$?"
timeout 1200 python bench.py --workload bay --steps 20 --warmup 5 > $O/r3_bench_c3.json 2> $O/r3_bench_c3.err; echo "c3 rc=$?"
timeout 2400 python bench.py --workload bay24m --steps 20 --warmup 5 > $O/r3_bench_c5.json 2> $O/r3_bench_c5.err; echo "c5 rc=$?"
