#!/bin/bash
# reference arms (measured bounded sub-workload)
O=gpurun_out/ref; mkdir -p $O
for c in 4 0 1 3; do
  t0=$(date +%s)
  python bench.py --config $c --impl reference --steps 3 --warmup 1 > $O/bench_ref_c$c.json 2> $O/bench_ref_c$c.err
  t1=$(date +%s)
  python -c "import json;d=json.load(open('$O/bench_ref_c$c.json'));print($c,'%.3g'%d['value'],round(d['ms_per_step']),d['config']['step'],'wall',$t1-$t0)"
done
