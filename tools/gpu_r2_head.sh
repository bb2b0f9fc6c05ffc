#!/bin/bash
# Health check of HEAD on a fresh box: smoke, the GPU suite, bench lines of configs 4/1/2/7,
# and the config-1 step launch list (the P = 140 propagation is the next target).
O=gpurun_out/head; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
PF_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; cut -c1-400 $O/bench_c4.json
for c in 1 2; do python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err; cut -c1-300 $O/bench_c$c.json; done
python bench.py --config 7 --steps 3 --warmup 3 > $O/bench_c7.json 2> $O/bench_c7.err; cut -c1-300 $O/bench_c7.json
PF_CFG=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/step_c1.csv python tools/prof_step.py > $O/step_c1.log 2>&1
ls $O
