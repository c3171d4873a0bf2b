#!/bin/bash
# bench pass: the default line (nq14), the B&B and first-solution workloads at N=1 and N=2
# (self-spawned ranks; gloo on a 1-GPU box), and the reference arm for each
o=gpurun_out; mkdir -p $o; tag=${1:-b}
timeout 900 python bench.py --steps 5 --warmup 3 > $o/bench_${tag}_nq14.log 2>&1; echo "rc=$?" >> $o/bench_${tag}_nq14.log
for inst in golomb10 rcsp_1000; do
  timeout 600 python bench.py --instance $inst --steps 3 --warmup 3 --no-extras > $o/bench_${tag}_$inst.log 2>&1; echo "rc=$?" >> $o/bench_${tag}_$inst.log
  timeout 600 python bench.py --instance $inst --gpus 2 --steps 3 --warmup 3 --no-extras --no-cpu > $o/bench_${tag}_${inst}_n2.log 2>&1; echo "rc=$?" >> $o/bench_${tag}_${inst}_n2.log
  timeout 600 python bench.py --instance $inst --impl reference --steps 2 --warmup 1 > $o/bench_${tag}_${inst}_ref.log 2>&1; echo "rc=$?" >> $o/bench_${tag}_${inst}_ref.log
done
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --no-cpu > $o/bench_${tag}_nq14_n2.log 2>&1; echo "rc=$?" >> $o/bench_${tag}_nq14_n2.log
echo done
