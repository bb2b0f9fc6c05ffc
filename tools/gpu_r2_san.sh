#!/bin/bash
mkdir -p gpurun_out/san
O=gpurun_out/san
python tools/san_case.py > $O/plain.log 2>&1; tail -1 $O/plain.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/san_case.py > $O/memcheck.log 2>&1; tail -4 $O/memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 50 python tools/san_case.py > $O/racecheck.log 2>&1; tail -4 $O/racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 50 python tools/san_case.py > $O/synccheck.log 2>&1; tail -4 $O/synccheck.log
