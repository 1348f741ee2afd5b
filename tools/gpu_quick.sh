mkdir -p gpurun_out
TAG=$1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1]);print('value',d['value'],'ms/step',d['ms_per_step'],'launch_ms',d['roofline']['launch_ms'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])"
tail -3 gpurun_out/bench_$TAG.err
ANTKV_TRACE=1 timeout 300 python tools/trace_cta.py > gpurun_out/trace_$TAG.log 2>&1; tail -16 gpurun_out/trace_$TAG.log
