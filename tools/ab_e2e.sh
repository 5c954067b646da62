#!/bin/bash
# A/B of variants/*.so on the e2e (host buffers through the C ABI) number of bench.py.
# usage (inside gpurun): bash tools/ab_e2e.sh [ROUNDS] [extra bench args]
ROUNDS=${1:-2}; shift
LIB=paper_2403_06478_b200/libagatha.so
cp $LIB /tmp/agatha_default.so
for r in $(seq 1 $ROUNDS); do
  for v in variants/*.so; do
    cp $v $LIB
    python bench.py --no-cpu --steps 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['stats_last_step']['input_chunks'])"
  done
done
cp /tmp/agatha_default.so $LIB
