#!/bin/bash
# C-ABI whole-algorithm entry points on the GPU (pf_rsd / pf_srsd / pf_nursd1 / pf_nursd2).
mkdir -p gpurun_out/capi2
timeout 900 python -m pytest tests/test_capi.py -q -m gpu > gpurun_out/capi2/pytest.log 2>&1; tail -15 gpurun_out/capi2/pytest.log
