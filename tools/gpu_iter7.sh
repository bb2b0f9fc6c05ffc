mkdir -p gpurun_out/it7
O=gpurun_out/it7
timeout 900 python -m pytest tests/test_gpu_rsd.py tests/test_gpu_configs.py tests/test_gpu_algorithms.py -m gpu -q > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
for c in 4 3; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "import json; d=json.load(open('$O/bench_c$c.json')); print('c$c', round(d['ms_per_step'],3), d['stage_ms'], round(d['roofline']['frac'],3))" || tail -5 $O/bench_c$c.err
done
