#!/bin/bash
# round-2 first pass: GPU tests (incl. the new headline file), the bench line, self-spawned 2-rank bench
o=gpurun_out; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > $o/r2a_gpu_tests.log 2>&1; echo "rc=$?" >> $o/r2a_gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > $o/r2a_bench.log 2>&1; echo "rc=$?" >> $o/r2a_bench.log
timeout 300 python bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --no-cpu > $o/r2a_bench2.log 2>&1; echo "rc=$?" >> $o/r2a_bench2.log
echo done
