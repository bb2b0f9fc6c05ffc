#!/bin/bash
# One GPU call refreshing every round artefact: tests, bench lines (ours + reference arm)
# for configs 4 (headline), 0, 1, 3, 5, config 2 timing, the c4 launch list and one
# ncu --set full capture of K1 and the four propagation stages.
set -x
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
for c in 0 1 3 5; do
  python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err
done
for c in 0 1 3; do
  python bench.py --config $c --impl reference --steps 2 --warmup 1 > $O/bench_ref_c$c.json 2> $O/bench_ref_c$c.err
done
python tools/run_config2.py > $O/config2.json 2> $O/config2.err
PF_NF=2 python tools/prof_rsd.py > $O/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      --log-file $O/launches_c4.csv python tools/prof_rsd.py > /dev/null 2>&1
PF_NF=2 ncu --set full --clock-control none --import-source on \
    -k regex:"k_pa|k_pb1|k_pb2|k_pc" -s 4 -c 4 -o $O/prof_full \
    python tools/prof_rsd.py > $O/ncu_full.log 2>&1
PF_NF=2 ncu --set full --clock-control none --import-source on \
    -k regex:"k_temporal_dft" -s 1 -c 1 -o $O/prof_k1 \
    python tools/prof_rsd.py > $O/ncu_k1.log 2>&1
tail -n 2 $O/ncu_full.log $O/ncu_k1.log
timeout 600 python tools/chunk_prof.py > $O/chunk_prof.txt 2>&1; cat $O/chunk_prof.txt
PF_PARITY_LOG=$O/parity.jsonl timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q > $O/parity_pytest.log 2>&1; tail -n 2 $O/parity_pytest.log
