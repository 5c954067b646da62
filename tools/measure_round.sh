#!/bin/bash
# Round-end measurement set on the GPU box (writes gpurun_out/; copy the keepers to profiles/).
# usage (inside gpurun): bash tools/measure_round.sh TAG [bench|ncu|study]...
#   bench: default bench (C2, e2e + cpu_baseline), C1/C3/C4/C5, input-order ablations, reference arm
#   ncu:   launch list of the device-resident bench (ncu serialises launches, so the
#          e2e leg, whose kernel overlaps its own input copies, is left out), DRAM bytes
#          of the align kernel on the full C2 batch, and one `--set full` on 20k C2 pairs
#   study: the long/short study (tools/long_short_study.py)
TAG=${1:-r01}; shift
O=gpurun_out
for part in "${@:-bench ncu study}"; do for p in $part; do case $p in
bench)
  python bench.py > $O/bench_${TAG}_c2_full.json 2> $O/bench_${TAG}_c2_full.err
  for c in C1 C3 C4 C5; do
    python bench.py --config $c --no-cpu > $O/bench_${TAG}_$c.json 2> $O/bench_${TAG}_$c.err
  done
  python bench.py --config C3 --no-cpu --no-e2e --order input > $O/bench_${TAG}_C3_input.json 2>/dev/null
  python bench.py --config C4 --no-cpu --no-e2e --order input > $O/bench_${TAG}_C4_input.json 2>/dev/null
  python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_${TAG}_reference.json 2> $O/bench_${TAG}_reference.err
  ;;
ncu)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${TAG}.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launch_${TAG}.log 2>&1
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:align --csv --log-file $O/ncu_dram_${TAG}.csv \
      python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_dram_${TAG}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:align16 -s 3 -c 1 -o $O/prof_full_${TAG} \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --pairs 20000 > $O/ncu_full_${TAG}.log 2>&1
  ;;
study)
  python tools/long_short_study.py > $O/long_short_${TAG}.jsonl 2> $O/long_short_${TAG}.err
  ;;
esac; done; done
