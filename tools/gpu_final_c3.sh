mkdir -p gpurun_out/f3
O=gpurun_out/f3
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -n 1 $O/pytest_gpu.log
python bench.py --config 3 > $O/bench_c3.json 2> $O/bench_c3.err
PF_PARITY_LOG=$O/parity.jsonl timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q > $O/parity_pytest.log 2>&1; tail -n 1 $O/parity_pytest.log
