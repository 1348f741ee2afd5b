#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-fa}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs.py -x -q -k "tcgen05 or ckernels_shim or flash or config1 or 128k or cache_case or prefill" > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
timeout 600 python tools/prefill_bench.py 32768 131072 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"flash_tc|ans_tc" -c 2 python tools/flash_tc_once.py 32768 2>&1 | grep -E "flash|ans_tc|duration|tensor" | head -8
