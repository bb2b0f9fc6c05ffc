set -x
mkdir -p gpurun_out/v1
O=gpurun_out/v1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; head -c 600 $O/bench_c4.json
python tools/prof_c2.py > $O/c2plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/prof_c2.py > $O/ncu_c2.log 2>&1
python tools/launches.py $O/launches_c2.csv 2>&1 | head -20
