#!/bin/bash
# One GPU-box pass: GPU tests, the bench line, a 2-rank functional run of the N>1 bench path
# (gloo, both ranks on cuda:0), the ncu launch list and one ncu --set full capture of the
# search kernel. Usage: scripts/gpu_round.sh <tag>
tag=${1:-run}
o=gpurun_out
mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/gpu_tests_$tag.log 2>&1; echo "rc=$?" >> $o/gpu_tests_$tag.log
timeout 600 python bench.py --steps 5 --warmup 3 > $o/bench_$tag.log 2>&1; echo "rc=$?" >> $o/bench_$tag.log
CUBICS_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --no-cpu \
  > $o/bench2_$tag.log 2>&1; echo "rc=$?" >> $o/bench2_$tag.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_$tag.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > $o/ncu_launch_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 \
  -o $o/prof_nq14_$tag -f python bench.py --steps 1 --warmup 3 --no-extras --no-cpu > $o/ncu_full_$tag.log 2>&1
echo done
