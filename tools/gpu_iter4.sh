# NUFFT spread variants: spectral/algorithm/config GPU tests, configs 5 and 1 bench, config 2
mkdir -p gpurun_out/it4
O=gpurun_out/it4
timeout 900 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_algorithms.py tests/test_gpu_configs.py tests/test_gpu_acceptance.py tests/test_gpu_acceptance_physics.py tests/test_gpu_edge.py -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in 5 1; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "import json; d=json.load(open('$O/bench_c$c.json')); print('c$c', round(d['ms_per_step'],3), d['stage_ms'], round(d['roofline']['frac'],3))" || tail -5 $O/bench_c$c.err
done
timeout 600 python tools/run_config2.py > $O/config2.json 2> $O/config2.err; cat $O/config2.json
