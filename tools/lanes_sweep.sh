# config-4 device step for stream-lane / plane-batch variants (PF_LANES, PF_BATCH_CAP)
mkdir -p gpurun_out/lanes
O=gpurun_out/lanes
for c in "2 4" "3 4" "1 4" "2 2" "3 2" "1 8"; do
  set -- $c
  PF_LANES=$1 PF_BATCH_CAP=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/b_$1_$2.json 2> $O/b_$1_$2.err
  python -c "import json; d=json.load(open('$O/b_$1_$2.json')); print('lanes=$1 cap=$2', round(d['ms_per_step'],3), round(d['stage_ms']['propagation'],3))" || tail -3 $O/b_$1_$2.err
done
# N=2 bench path (two gloo ranks on cuda:0: host-staged collectives, no cross-rank kernel waits)
PF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu \
  > $O/b_n2_gloo.json 2> $O/b_n2_gloo.err
python -c "import json; d=json.load(open('$O/b_n2_gloo.json')); print('n2 gloo', d['n_gpus'], round(d['ms_per_step'],3), d['gpu_launches'], d['e2e']['value'] if d['e2e'] else None)" || tail -5 $O/b_n2_gloo.err
python -c "import json; d=json.load(open('$O/b_3_4.json')); print('launches c4', d['gpu_launches'])"
