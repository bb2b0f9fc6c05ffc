# iteration check: targeted GPU tests, config-4 bench (device leg), shard timings
mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_rsd.py tests/test_gpu_configs.py -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
python -c "import json; d=json.load(open('$O/bench_c4.json')); print('c4', round(d['ms_per_step'],3), d['stage_ms'], round(d['roofline']['frac'],3))" || tail -5 $O/bench_c4.err
timeout 600 python tools/chunk_prof.py > $O/chunk_prof.txt 2>&1; cat $O/chunk_prof.txt
