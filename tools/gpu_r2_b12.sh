#!/bin/bash
# fused B1+B2 (k_pb12): smoke, GPU suite, config-4/0/3 bench with PF_B12=0/1, launch list
mkdir -p gpurun_out/b12
O=gpurun_out/b12
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for b in 0 1; do for c in 4 0 3; do
  PF_B12=$b python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c${c}_b$b.json 2> $O/bench_c${c}_b$b.err
  python -c "import json; d=json.load(open('$O/bench_c${c}_b$b.json')); print('b12=$b c$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['roofline']['frac'],3), d['roofline'].get('executed',{}).get('frac'))" || tail -3 $O/bench_c${c}_b$b.err
done; done
PF_NF=2 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      --log-file $O/launches_c4.csv python tools/prof_rsd.py > /dev/null 2>&1
python tools/launches.py $O/launches_c4.csv 2>&1 | head -12
