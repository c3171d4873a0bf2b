#!/bin/bash
# quick GPU pass: selected tests (args), then the full GPU suite and the default bench line
o=gpurun_out; mkdir -p $o; tag=${1:-q}; shift
timeout 900 python -m pytest -x -q -p no:cacheprovider --timeout 240 --timeout-method=thread "$@" > $o/quick_$tag.log 2>&1; echo "rc=$?" >> $o/quick_$tag.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method=thread --durations=15 > $o/gpu_tests_$tag.log 2>&1; echo "rc=$?" >> $o/gpu_tests_$tag.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu > $o/bench_$tag.log 2>&1; echo "rc=$?" >> $o/bench_$tag.log
echo done
