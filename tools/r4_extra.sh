#!/bin/bash
# round-2 session-3 extra lines (1 GPU): the driver's bench command on the final build, C3 and C5 bench
# lines, and a 4-rank bench through CUDA IPC with every rank on device 0 (time-sliced: exercises the
# multi-process path; its times are not multi-GPU times)
O=gpurun_out
T=${TAG:-r5}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --workload bay --steps 20 --warmup 5 > $O/${T}_bench_c3_bay.json 2> $O/${T}_bench_c3.err; echo "c3 rc=$?"
timeout 2400 python bench.py --workload bay24m --steps 20 --warmup 5 > $O/${T}_bench_c5_bay24m.json 2> $O/${T}_bench_c5.err; echo "c5 rc=$?"
LPSIM_BENCH_SAME_GPU=1 LPSIM_MAX_BLOCKS=148 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 10 --warmup 3 --no-full-run \
  > $O/${T}_bench_4rank_same_gpu.json 2> $O/${T}_bench_4rank.err; echo "4rank rc=$?"
tail -c 300 $O/${T}_bench_4rank.err
