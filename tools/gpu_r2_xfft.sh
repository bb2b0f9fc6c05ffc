#!/bin/bash
mkdir -p gpurun_out/xfft
O=gpurun_out/xfft
timeout 900 python -m pytest tests/test_gpu_rsd.py -q -x -k "fft_lines or fftn" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py > $O/pytest_all.log 2>&1; tail -3 $O/pytest_all.log
for x in 0 1; do for c in 1 2; do
PF_XFFT=$x python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/b_c${c}_x$x.json 2>/dev/null
python -c "import json; d=json.load(open('$O/b_c${c}_x$x.json')); print('xfft=$x c$c', round(d['ms_per_step'],3))"
done; done
python tools/prof_c2.py > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/prof_c2.py > /dev/null 2>&1
python tools/launches.py $O/launches_c2.csv | head -8
