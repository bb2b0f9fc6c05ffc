#!/bin/bash
# the driver's round-end sequence at HEAD: smoke, default bench (N = 1), reference arm
O=gpurun_out/last; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
t0=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err; t1=$(date +%s)
python -c "import json;d=json.load(open('$O/bench.json'));print('ours',d['ms_per_step'],'%.4g'%d['value'],d['roofline']['frac'],d['roofline_other']['frac'],'%.4g'%d['e2e']['value'],d['gpu_launches'],d['clocks'],'wall',$t1-$t0)"
t0=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; t1=$(date +%s)
python -c "import json;d=json.load(open('$O/bench_ref.json'));print('ref','%.4g'%d['value'],d['ms_per_step'],d['config']['step'],'wall',$t1-$t0)"
