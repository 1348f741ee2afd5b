#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-enc5l}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core_encoder or staged or packed or sharded_decode" > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
timeout 200 python tools/enc_bench.py d32m4096 d16m4096 d16m256 2>&1 | tail -3 | cut -c1-160
ANTKV_NO_TC5_ENC=1 timeout 200 python tools/enc_bench.py d32m4096 d16m4096 2>&1 | tail -2 | cut -c1-160
