#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-mha}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs.py -x -q -k "staged or config4 or cache_case or sharded" > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
timeout 300 python tools/staged_bench.py --configs cfg4_b16_8k_d4m256_mha,d4m256_128k --kernels 2,0 2>&1 | tail -6
ANTKV_NO_MHA=1 timeout 300 python tools/staged_bench.py --configs cfg4_b16_8k_d4m256_mha --kernels 2 2>&1 | tail -1
