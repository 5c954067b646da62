#!/bin/bash
# One perf iteration on the GPU box: GPU parity tests (fast subset), C2 bench, ncu of the align kernel.
# usage (inside gpurun): bash tools/perf_iter.sh TAG [full]
TAG=${1:-x}
if [ "$2" == "full" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
else
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "random_short or edge or c1_full or subsets or tie" 2>&1 | tail -3
fi
python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('GCUPS', d['value'], 'kernel', d['roofline']['kernel_gcups'], d['stats_last_step'])"
ncu --set full --clock-control none --import-source on -k regex:align16 -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --pairs 20000 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
