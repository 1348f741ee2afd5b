#!/bin/bash
# Round-2 check: GPU parity suite, bench with / without the exclusive-stream
# early reads, CTA trace.  Run under gpurun.
mkdir -p gpurun_out
TAG=${1:-r2a}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pt_$TAG.log
for mode in excl shared; do
  extra=""; [ $mode = shared ] && extra="--shared-stream"
  timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 50 $extra > gpurun_out/bench_${TAG}_$mode.json 2> gpurun_out/bench_${TAG}_$mode.err; echo bench $mode rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_${TAG}_$mode.json').read().strip().splitlines()[-1]);print('$mode value',d['value'],'ms/step',d['ms_per_step'],'launch_ms',d['roofline']['launch_ms'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])"
done
ANTKV_TRACE=1 timeout 300 python tools/trace_cta.py > gpurun_out/trace_$TAG.log 2>&1; tail -16 gpurun_out/trace_$TAG.log
