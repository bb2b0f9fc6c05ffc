# per-rank propagation time of N-GPU shards of config 4 on one GPU (chunked and not),
# and lanes/batch-cap variants for the 32-plane shard
mkdir -p gpurun_out/shards
O=gpurun_out/shards
timeout 600 python tools/chunk_prof.py > $O/chunk_prof.txt 2>&1; cat $O/chunk_prof.txt
timeout 900 bash tools/shard_sweep.sh > $O/shard_sweep.txt 2>&1; cat $O/shard_sweep.txt
