#!/bin/bash
# one GPU call: tests, bench, launch list, full ncu capture of K1 and the propagation kernels
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
tail -c 600 gpurun_out/bench_r1.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1.json 2> gpurun_out/bench_ref_r1.err
python tools/prof_rsd.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_r1.csv python tools/prof_rsd.py > /dev/null 2>&1
python tools/prof_rsd.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_temporal_dft|k_p[abc]" -s 0 -c 4 -o gpurun_out/prof_r1_full python tools/prof_rsd.py > gpurun_out/ncu_full_r1.log 2>&1
tail -2 gpurun_out/ncu_full_r1.log
