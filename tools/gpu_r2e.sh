#!/bin/bash
# Round-2 perf iteration: bench (excl), PDL trace, quick fused-kernel parity.
mkdir -p gpurun_out
TAG=${1:-r2e}
timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 50 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1]);print('value',d['value'],'ms/step',d['ms_per_step'],'launch_ms',d['roofline']['launch_ms'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])"
tail -3 gpurun_out/bench_$TAG.err
timeout 300 python tools/trace_pdl.py --graph > gpurun_out/tpdl_$TAG.log 2>&1; tail -24 gpurun_out/tpdl_$TAG.log
timeout 600 python -m pytest tests/test_baseline_configs.py -q -x -k "config1 and (fused or staged)" > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
