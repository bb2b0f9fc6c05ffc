# SRSD check: algorithm/config/acceptance GPU tests + config-3 bench (device leg)
mkdir -p gpurun_out/srsd
O=gpurun_out/srsd
timeout 900 python -m pytest tests/test_gpu_algorithms.py tests/test_gpu_configs.py tests/test_gpu_acceptance.py tests/test_gpu_spectral.py -m gpu -q > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
python -c "import json; d=json.load(open('$O/bench_c3.json')); print('c3', round(d['ms_per_step'],3), d['stage_ms'], round(d['roofline']['frac'],3))" || tail -5 $O/bench_c3.err
