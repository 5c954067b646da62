#!/bin/bash
# A/B kernel variants on the GPU box: each variants/*.so is swapped in as the library and
# timed on a bench config (default C2, device-resident), alternating the order over ROUNDS
# rounds.  usage (inside gpurun): bash tools/ab_bench.sh [ROUNDS] [extra bench args]
ROUNDS=${1:-2}; shift
LIB=paper_2403_06478_b200/libagatha.so
cp $LIB /tmp/agatha_default.so
for r in $(seq 1 $ROUNDS); do
  for v in variants/*.so; do
    cp $v $LIB
    python bench.py --no-cpu --no-e2e --steps 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$*', round(d['value'],1), round(d['roofline']['kernel_gcups'],1))"
  done
done
cp /tmp/agatha_default.so $LIB
