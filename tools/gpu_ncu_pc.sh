# bench (device leg) + ncu --set full with source of one k_pc and one k_pb2 launch (config 4)
mkdir -p gpurun_out/pc
O=gpurun_out/pc
timeout 600 python -m pytest tests/test_gpu_rsd.py -m gpu -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
python -c "import json; d=json.load(open('$O/bench_c4.json')); print('c4', round(d['ms_per_step'],3), d['stage_ms'], round(d['roofline']['frac'],3))" || tail -5 $O/bench_c4.err
PF_NF=2 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_pc|k_pb2|k_pa" -s 30 -c 3 -o $O/prof_pc python tools/prof_rsd.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
