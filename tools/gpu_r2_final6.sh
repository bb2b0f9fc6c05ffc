#!/bin/bash
# Record after the exponential-of-semicircle window: GPU suite (full-size parity), bench lines
# of the NUFFT configurations 1, 2, 5, 7 (ours) and step launch lists of 1, 2, 7.
O=gpurun_out/final11; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
PF_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for c in 1 2 5; do
  python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err
done
python bench.py --config 7 --steps 3 --warmup 3 > $O/bench_c7.json 2> $O/bench_c7.err
for c in 1 2 7; do
  PF_CFG=$c timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c$c.csv python tools/prof_step.py > $O/step_c$c.log 2>&1
  python tools/launches.py $O/step_c$c.csv > $O/step_c$c.txt
done
ls $O
