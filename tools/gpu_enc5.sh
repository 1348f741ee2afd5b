#!/bin/bash
# tcgen05 encoder iteration: parity tests, throughput (tc5 vs mma.sync A/B), under gpurun.
mkdir -p gpurun_out
TAG=${1:-enc5}
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core_encoder or assign_nearest or cache_case" > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
timeout 120 python tools/enc_bench.py d8m256 2>&1 | tail -1
ANTKV_NO_TC5_ENC=1 timeout 120 python tools/enc_bench.py d8m256 2>&1 | tail -1
