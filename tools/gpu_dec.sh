#!/bin/bash
# Decode-kernel iteration: bench (exclusive / shared stream) + CTA trace.  Run under gpurun.
mkdir -p gpurun_out
TAG=${1:-dec}
for mode in excl shared; do
  extra=""; [ $mode = shared ] && extra="--shared-stream"
  timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 50 $extra > gpurun_out/bench_${TAG}_$mode.json 2> gpurun_out/bench_${TAG}_$mode.err; echo bench $mode rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_${TAG}_$mode.json').read().strip().splitlines()[-1]);print('$mode value',d['value'],'ms/step',d['ms_per_step'],'launch_ms',d['roofline']['launch_ms'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])" || tail -5 gpurun_out/bench_${TAG}_$mode.err
done
ANTKV_TRACE=1 timeout 300 python tools/trace_cta.py > gpurun_out/trace_$TAG.log 2>&1; tail -18 gpurun_out/trace_$TAG.log
if [ -n "$PYT" ]; then timeout 900 python -m pytest tests -m gpu -x -q $PYT > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log; fi
