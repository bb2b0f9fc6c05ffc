# smoke + the N=2 bench path (two gloo ranks on cuda:0, host-staged collectives) on the final code
mkdir -p gpurun_out/san
O=gpurun_out/san
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -n 2 $O/smoke.log
PF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu \
  > $O/b_n2_gloo.json 2> $O/b_n2_gloo.err
python -c "import json; d=json.load(open('$O/b_n2_gloo.json')); print('n2 gloo', d['n_gpus'], round(d['ms_per_step'],3), d['gpu_launches'], d['e2e']['value'] if d['e2e'] else None)" || tail -5 $O/b_n2_gloo.err
