#!/bin/bash
# One GPU call refreshing the round-2 record: GPU suite (incl. full-size parity), bench lines
# (ours + reference arm) for configs 4 (headline), 0, 1, 2, 3, 5, 6, the config-4 launch list,
# ncu --set full of K1 and the propagation kernels, steady-state traffic.
mkdir -p gpurun_out/final8
O=gpurun_out/final8
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
PF_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4.err
python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
for c in 0 1 2 3 5; do
  python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err
done
python bench.py --config 6 --steps 3 --warmup 3 > $O/bench_c6.json 2> $O/bench_c6.err
python bench.py --config 7 --steps 3 --warmup 3 > $O/bench_c7.json 2> $O/bench_c7.err
for c in 0 1 2 3; do
  python bench.py --config $c --impl reference --steps 3 --warmup 1 > $O/bench_ref_c$c.json 2> $O/bench_ref_c$c.err
done
PF_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_c4_gloo2.json 2> $O/bench_c4_gloo2.err
PF_PEER=0 PF_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_c4_gloo2_nccl_path.json 2> $O/bench_c4_gloo2_nccl_path.err
PF_NF=2 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      --log-file $O/launches_c4.csv python tools/prof_rsd.py > /dev/null 2>&1
PF_NF=2 PF_CFG=3 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      --log-file $O/launches_c3.csv python tools/prof_rsd.py > /dev/null 2>&1
PF_NF=2 ncu --set full --clock-control none --import-source on \
    -k regex:"k_pa|k_pb12|k_pc_h" -s 6 -c 3 -o $O/prof_full \
    python tools/prof_rsd.py > $O/ncu_full.log 2>&1
PF_NF=2 ncu --set full --clock-control none --import-source on \
    -k regex:"k_temporal_dft" -s 1 -c 1 -o $O/prof_k1 \
    python tools/prof_rsd.py > $O/ncu_k1.log 2>&1
PF_NF=2 timeout 1200 ncu --replay-mode application --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    -k regex:"k_" --csv --log-file $O/traffic_app.csv python tools/prof_rsd.py > $O/ncu_app.log 2>&1
timeout 600 python tools/chunk_prof.py > $O/chunk_prof.txt 2>&1; tail -5 $O/chunk_prof.txt
ls $O
