cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -x -q -k "${PTK:-fast or gqa or cache_case or pdl or one_split or sharded or peer}" > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 50 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1]);print('value',d['value'],'ms/step',d['ms_per_step'],'launch_ms',d['roofline']['launch_ms'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])"
done
ANTKV_TRACE=1 timeout 300 python tools/trace_cta.py > gpurun_out/trace_$TAG.log 2>&1; head -16 gpurun_out/trace_$TAG.log
