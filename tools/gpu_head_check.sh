# HEAD check: full GPU suite, smoke, default bench line
mkdir -p gpurun_out/head
O=gpurun_out/head
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(round(d['ms_per_step'],3), '%.3g'%d['value'], round(d['roofline']['frac'],3), '%.3g'%d['e2e']['value'], d['gpu_launches'], d['clocks'])" || tail -5 $O/bench.err
