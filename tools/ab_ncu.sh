#!/bin/bash
# ncu (full set, source counters) of the align16 kernel for each variants/*.so (20000 C2 pairs)
LIB=paper_2403_06478_b200/libagatha.so
cp $LIB /tmp/agatha_default.so
for v in variants/*.so; do
  b=$(basename $v .so)
  cp $v $LIB
  ncu --set full --clock-control none --import-source on -k regex:align16 -s 3 -c 1 -o gpurun_out/ab_$b python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --pairs 20000 > gpurun_out/ab_$b.log 2>&1
  tail -1 gpurun_out/ab_$b.log
done
cp /tmp/agatha_default.so $LIB
