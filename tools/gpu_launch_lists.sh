#!/bin/bash
# ncu launch lists (gpu__time_duration.sum, serialised, cold cache) of the bench step of
# configs 0, 1 and 3, each after the same command has exited 0 without ncu.
mkdir -p gpurun_out/ll
O=gpurun_out/ll
for c in 0 1 3; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c$c.json 2> $O/bench_c$c.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c$c.csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_c$c.log 2>&1
  python tools/launches.py $O/launches_c$c.csv > $O/launches_c$c.txt 2>&1
  head -12 $O/launches_c$c.txt
done
