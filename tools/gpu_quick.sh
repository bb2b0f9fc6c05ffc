#!/bin/bash
# quick check: one test file (or -k expr) + launch lists of the given configs
# usage: tools/gpu_quick.sh "<pytest args>" "<configs>"
mkdir -p gpurun_out/q
O=gpurun_out/q
timeout 600 python -m pytest $1 -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in $2; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c$c.json 2> $O/bench_c$c.err
  python -c "import json; d=json.load(open('$O/bench_c$c.json')); print('c$c', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms'].items()}, 'k1 frac', round(d['roofline_other']['frac'] if d['roofline']['bound']=='fp32' else d['roofline']['frac'],3))" || tail -5 $O/bench_c$c.err
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c$c.csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_c$c.log 2>&1
  python tools/launches.py $O/launches_c$c.csv 2>&1 | grep -E "k_|bluestein" | grep -v probe | head -8
done
