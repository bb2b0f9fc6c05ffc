#!/bin/bash
# Round-2 first check: full GPU suite + default bench line + launch list.
mkdir -p gpurun_out/r2a
O=gpurun_out/r2a
nproc > $O/nproc.txt; lscpu | head -20 >> $O/nproc.txt; free -g >> $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; cat $O/bench_c4.json | head -c 600
