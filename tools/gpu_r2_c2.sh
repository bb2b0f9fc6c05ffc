#!/bin/bash
mkdir -p gpurun_out/c2
O=gpurun_out/c2
python tools/prof_c2.py > $O/c2plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/prof_c2.py > $O/ncu_c2.log 2>&1
python tools/launches.py $O/launches_c2.csv > $O/launches_c2.txt 2>&1; head -20 $O/launches_c2.txt
python bench.py --config 2 --steps 5 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 1500 $O/bench_c2.json; tail -3 $O/bench_c2.err
python bench.py --config 2 --impl reference --steps 1 --warmup 0 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err; tail -c 600 $O/bench_ref_c2.json; tail -3 $O/bench_ref_c2.err
