#!/bin/bash
# split type-2 passes: threads per CTA sweep (rows x cols) on config 2 and 7
O=gpurun_out/t2thr; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_spectral.py -m gpu -q -k type2_start > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for r in 128 256; do for cc in 128 256; do
for c in 2 7; do
  PF_T2_THREADS_ROWS=$r PF_T2_THREADS_COLS=$cc python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b.json 2> $O/b.err
  python -c "import json;d=json.load(open('$O/b.json'));print($c,'rows',$r,'cols',$cc,d['ms_per_step'],d['volume_sha256_16'])"
done; done; done
