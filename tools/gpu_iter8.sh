mkdir -p gpurun_out/it8
O=gpurun_out/it8
timeout 900 python -m pytest tests/test_gpu_rsd.py tests/test_gpu_configs.py tests/test_gpu_algorithms.py tests/test_gpu_acceptance.py tests/test_gpu_edge.py -m gpu -q > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
python bench.py --config 0 > $O/bench_c0.json 2> $O/bench_c0.err
python -c "import json; d=json.load(open('$O/bench_c0.json')); print('c0', round(d['ms_per_step'],4), d['stage_ms'], round(d['roofline']['frac'],3))" || tail -5 $O/bench_c0.err
