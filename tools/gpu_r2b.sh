#!/bin/bash
# Round-2: BASELINE-config parity tests + the observed-error table.
mkdir -p gpurun_out
TAG=${1:-r2b}
rm -f gpurun_out/parity_errors.jsonl
timeout 1500 python -m pytest tests/test_baseline_configs.py tests/test_gpu_parity.py -m gpu -q -x ${2:+-k "$2"} \
  --durations=15 > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -30 gpurun_out/pt_$TAG.log
cat gpurun_out/parity_errors.jsonl
